"""Summarise an ncu source page (SASS view): top stall-sampled instructions of one kernel.
usage: python tools/ncu_hot.py <report.ncu-rep> <kernel-regex> [N]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = [x for x in r[2:] if len(x) == len(h)]
ia, iw, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
num = lambda s: int(s) if s.strip().isdigit() else 0
tot = sum(num(x[iw]) for x in rows)
tote = sum(num(x[ie]) for x in rows)
print(f"samples {tot}  warp-instructions executed {tote}")
for x in sorted(rows, key=lambda x: -num(x[iw]))[:n]:
    print(f"{num(x[iw]):7d} {100.0 * num(x[iw]) / max(tot, 1):5.1f}% {num(x[ie]):10d}  {x[0][-5:]} {x[ia].strip()[:80]}")
