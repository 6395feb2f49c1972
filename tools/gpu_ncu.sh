# usage: bash tools/gpu_ncu.sh <tag> [kernel-regex]
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01}
KRE=${2:-k_ransac_score|k_nearest|k_dense}
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:${KRE}" -s 0 -c 6 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
