# Build alternative libbt.so variants for A/B timing: abtmp/<name>/libbt.so
# usage: bash tools/build_variants.sh "name:-DFLAG=1 -DOTHER=2" "name2:" ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  n=${v%%:*}; f=${v#*:}; mkdir -p abtmp/$n
  ( BT_NVCC_FLAGS="$f" python -c "
import sys; sys.path.insert(0, '.')
from paper_2108_00516_b200 import build as b
b.LIB = 'abtmp/$n/libbt.so'; b.build(force=True, verbose=False)" > abtmp/$n/build.log 2>&1 && echo "built $n" || { echo "FAILED $n"; grep -m5 error abtmp/$n/build.log; } ) &
done
wait
