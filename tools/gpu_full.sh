# Round evidence: GPU tests, full bench (with cpu_baseline + e2e), the reference arm,
# the ncu launch list of the bench command, and an ncu --set full capture of one step's kernels.
# usage: bash tools/gpu_full.sh <tag>
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench exit $?" >> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 2 > gpurun_out/${TAG}_reference.json 2>&1
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:^k_" -s 40 -c 22 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
