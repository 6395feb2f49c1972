# ncu --set full with source correlation for the hot kernels of one C2 step (one GPU).
# usage: bash tools/gpu_ncu_src.sh <tag> [kernel-regex]
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r02}
KRE=${2:-k_match_ws|k_dense|k_score_tc}
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-c4 --no-graph"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:${KRE}" -s 14 -c 7 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
