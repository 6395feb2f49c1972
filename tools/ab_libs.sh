# A/B timing of alternative builds of libbt.so (abtmp/<variant>/libbt.so, selected with BT_LIB):
# the bench step and the dominant kernel's standalone time.  usage: bash tools/ab_libs.sh tag v1 v2 ...
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=$1; shift
for rep in 1 2; do
for v in "$@"; do
  BT_LIB=abtmp/$v/libbt.so timeout 300 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_b.json 2>gpurun_out/${TAG}_b.err
  python -c "
import json;d=json.loads(open('gpurun_out/${TAG}_b.json').read().strip().splitlines()[-1])
print('$v', round(d['ms_per_step'],4), round(d['ms_per_step_instrumented'],4), {k:(round(v['standalone_ms_per_step'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})" >> gpurun_out/${TAG}_ab.txt 2>&1
done; done
