# A/B timing of builds x environment settings.  usage: bash tools/ab_env.sh tag "label:ENV=val ENV2=val" ...
# (BT_LIB=abtmp/<v>/libbt.so selects a build).  Two rounds, bench step + per-kernel standalone / frac.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=$1; shift
for rep in 1 2; do
for spec in "$@"; do
  lab=${spec%%:*}; envs=${spec#*:}
  env $envs timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-c4 > gpurun_out/${TAG}_b.json 2>gpurun_out/${TAG}_b.err
  python -c "
import json;d=json.loads(open('gpurun_out/${TAG}_b.json').read().strip().splitlines()[-1])
print('$lab', round(d['ms_per_step'],4), round(d['ms_per_step_instrumented'],4), {k:(round(v['standalone_ms_per_step'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})" >> gpurun_out/${TAG}_ab.txt 2>&1
done; done
