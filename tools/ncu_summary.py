"""Summarise ncu evidence for profiles/: per-kernel metrics of a --set full report and the
share of each kernel in a launch list.  Writes <out>.md and (for the roofline `traffic`
field of bench.py) profiles/ncu_traffic.json.

usage: python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <out-prefix>"""
import collections
import csv
import json
import os
import re
import subprocess
import sys

rep, launches, out = sys.argv[1], sys.argv[2], sys.argv[3]

METRICS = [
    ("gpu__time_duration.sum", "duration (us)", 1e-3),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1),
    ("dram__bytes_write.sum", "DRAM write (MB)", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe inst %", 1),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles %", 1),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "FMA-heavy cycles % (elapsed)", 1),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %", 1),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %", 1),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", 1),
    ("launch__registers_per_thread", "registers", 1),
    ("launch__grid_size", "grid", 1),
    ("smsp__inst_executed.sum", "warp instructions", 1),
]


def short(name):
    m = re.search(r"::(k_[a-z_0-9]+)", name)
    return m.group(1) if m else name[:40]


raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
per = collections.defaultdict(list)
for r in rows[2:]:
    d = dict(zip(hdr, r))
    per[short(d.get("Kernel Name", "?"))].append(d)

lines = [f"# ncu --set full summary ({os.path.basename(rep)})", "",
         "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
         "(cold cache, serialised, replayed: compare shares, not absolutes).  'FMA pipe inst %' counts an "
         "FFMA2 (packed fp32x2) as one instruction; 'FMA pipe cycles %' / 'FMA-heavy "
         "cycles %' measure the pipe's occupancy (FFMA2 issues on the FMA-heavy pipe).", "",
         "| kernel | launches | " + " | ".join(m[1] for m in METRICS) + " |",
         "|---|---|" + "---|" * len(METRICS)]
traffic = {}
for k, ds in sorted(per.items()):
    vals = []
    for key, _, scale in METRICS:
        xs = []
        for d in ds:
            try:
                xs.append(float(d.get(key, "nan").replace(",", "")))
            except ValueError:
                pass
        v = sum(xs) / len(xs) if xs else float("nan")
        if key == "gpu__time_duration.sum":
            u = units[hdr.index(key)] if key in hdr else "ns"
            v = v * (1e-3 if u == "ns" else 1.0)
        vals.append(v)
    rd = vals[1] * (1e6 if units[hdr.index("dram__bytes_read.sum")].startswith("M") else 1)
    wr = vals[2] * (1e6 if units[hdr.index("dram__bytes_write.sum")].startswith("M") else 1)
    traffic[k] = rd + wr
    lines.append(f"| {k} | {len(ds)} | " + " | ".join(f"{v:.4g}" for v in vals) + " |")

# launch list shares
lst = list(csv.reader(open(launches).read().splitlines()))
hi = next(i for i, r in enumerate(lst) if "Kernel Name" in r)
h = lst[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = collections.Counter()
cnt = collections.Counter()
for r in lst[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1.0)
    tot[short(r[ki])] += v
    cnt[short(r[ki])] += 1
all_us = sum(tot.values())
lines += ["", f"## Launch list ({os.path.basename(launches)}): device time per kernel, serialised", "",
          "| kernel | launches | total us | share |", "|---|---|---|---|"]
for k, v in tot.most_common():
    lines.append(f"| {k} | {cnt[k]} | {v:.1f} | {100 * v / all_us:.1f}% |")
# the bt_register_pairs step alone (the bench command also runs standalone stage passes and the
# NEXT-row sections, which reuse the dense kernels): split the list into maximal runs of step
# kernels (the L2 flush between steps and every other kernel end a run) and keep the runs that
# hold whole steps (as many k_dense as scoring launches, at least one)
STEP = {"k_desc_prep", "k_desc_half", "k_match_tc", "k_match_ws", "k_fullscan", "k_rescore", "k_mutual", "k_ransac_hyp",
        "k_ransac_score", "k_corr_feat", "k_score_tc", "k_score_fix", "k_score_fix_rows", "k_ransac_finish",
        "k_edge_setup", "k_dense_mask", "k_dense_prep", "k_dense_scan", "k_dense", "k_dense_reduce"}
stot, scnt, n_steps = collections.Counter(), collections.Counter(), 0
run_t, run_c = collections.Counter(), collections.Counter()


def close_run():
    global n_steps
    ns = run_c["k_ransac_score"] + run_c["k_score_tc"]
    if ns and run_c["k_dense"] == ns:
        stot.update(run_t)
        scnt.update(run_c)
        n_steps += ns
    run_t.clear()
    run_c.clear()


for r in lst[hi + 1:]:
    if len(r) <= vi:
        continue
    k = short(r[ki])
    if k not in STEP:
        close_run()
        continue
    run_t[k] += float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1.0)
    run_c[k] += 1
close_run()
if n_steps:
    step_us = sum(stot.values())
    lines += ["", f"## The registration step only ({n_steps} whole steps in the list; serialised, cold cache)", "",
              "| kernel | launches / step | us / step | share of the step's kernels |", "|---|---|---|---|"]
    for k, v in stot.most_common():
        lines.append(f"| {k} | {scnt[k] / n_steps:g} | {v / n_steps:.1f} | {100 * v / step_us:.1f}% |")
    lines.append(f"| (sum) | | {step_us / n_steps:.1f} | 100% |")
open(out + ".md", "w").write("\n".join(lines) + "\n")
# per profiling bucket of libbt (bench.py's kernel names): the sum over the kernels the bucket
# launches once per step (each kernel's traffic averaged over its captured launches)
BUCKETS = {"k_ransac_score": ["k_corr_feat", "k_score_tc", "k_score_fix", "k_score_fix_rows", "k_ransac_score"],
           "k_match_tc": ["k_match_ws", "k_match_tc"],
           "k_dense_prep": ["k_edge_setup", "k_dense_mask", "k_dense_prep", "k_dense_scan"]}
out_t = dict(traffic)
for b, ks in BUCKETS.items():
    got = [traffic[k] for k in ks if k in traffic]
    if got:
        out_t[b] = sum(got)
json.dump(out_t, open(os.path.join(os.path.dirname(out), "ncu_traffic.json"), "w"), indent=1)
print("\n".join(lines))
