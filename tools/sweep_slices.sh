# temporary tuning sweep: scoring slices x finish split
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BT_FIN_SPLIT=0 timeout 600 python -m pytest tests -m gpu -x -q -k "ransac or parity or graph" > gpurun_out/s2_pytest0.log 2>&1; echo "pytest exit $?" >> gpurun_out/s2_pytest0.log
for rep in 1 2; do
for sp in 0 1; do
for m in 1 2 3; do
  BT_FIN_SPLIT=$sp BT_SCORE_SLICES=$m timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/s2_b.json 2>/dev/null
  python -c "
import json,sys;d=json.loads(open('gpurun_out/s2_b.json').read().strip().splitlines()[-1])
print('split $sp slices x$m', round(d['ms_per_step'],4), round(d['ms_per_step_instrumented'],4), {k:round(v,4) for k,v in d['kernel_ms_per_step'].items() if 'ransac' in k}, d['kernels']['k_ransac_score']['standalone_ms_per_step'])" >> gpurun_out/s2_sweep.txt
done; done; done
