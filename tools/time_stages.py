"""Standalone per-stage / per-kernel device times on the bench workload (C2, rank 0): each C-ABI
entry (bt_match, bt_ransac, bt_dense_corr, bt_register_pairs) run alone, L2 flushed before every
call, kernels bracketed with the library's profiling events.  A development tool: the bench's
own per-kernel numbers come from inside the overlapped step.

usage: python tools/time_stages.py [reps]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2108_00516_b200 as bt  # noqa: E402
import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
sc, pairs, uids, poses = bench.workload(0)
P = len(pairs)
dev = torch.device("cuda", 0)
fb = bt.FrameBatch.from_scene(sc, dev)
t_pairs = torch.from_numpy(pairs).to(dev)
t_uid = torch.from_numpy(uids.view(np.int32)).to(dev)
t_pose = torch.from_numpy(poses).to(dev)
edges = torch.from_numpy(np.concatenate([pairs, pairs[:, ::-1]], 0).astype(np.int32).copy()).to(dev)
ctx = bt.Context(0)
ctx.reserve(P, bench.N_MAX, bench.N_HYP, bench.N_FRAMES, bench.W, bench.H)
rprm, eprm = bt.ransac_params(bench.N_HYP, synth.PHILOX_SEED), bt.edge_params()
rw = bt.record_words(bench.N_MAX)
rec = torch.zeros((P, rw), dtype=torch.int32, device=dev)
mt = torch.zeros((P, bench.N_MAX, 2), dtype=torch.int32, device=dev)
nm = torch.zeros(P, dtype=torch.int32, device=dev)
dout = torch.zeros((edges.shape[0], 32), dtype=torch.float32, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

stages = {
    "match": lambda: ctx.match(fb, t_pairs, mt, nm),
    "ransac": lambda: ctx.ransac(fb, t_pairs, t_uid, mt, nm, rprm, rec),
    "dense": lambda: ctx.dense_corr(fb, sc.K, t_pose, edges, eprm, dout),
    "register_pairs": lambda: ctx.register_pairs(fb, sc.K, t_pose, t_pairs, t_uid, rprm, eprm, rec),
}
out = {}
for name, fn in stages.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    evu = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evu:                                   # uninstrumented stage time
        flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    tu = sorted(a.elapsed_time(b) for a, b in evu)
    ctx.profile(True)
    ctx.profile_read()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    t = sorted(a.elapsed_time(b) for a, b in ev)
    out[name] = {"median_ms": tu[len(tu) // 2], "instrumented_median_ms": t[len(t) // 2], "min_ms": tu[0],
                 "kernels_us": {k: round(1e3 * v[0] / v[1], 2) for k, v in prof.items() if v[1]}}
print(json.dumps(out, indent=1))
