"""Standalone device time of bt_match on the first P pairs of the bench workload (C2 frames),
for a sweep of P: exposes the wave quantisation of the persistent matching kernel (items =
2 directions x P pairs x n_pad / 128 row tiles over 2 CTAs per SM).  A development tool.

usage: python tools/match_scan.py [P ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2108_00516_b200 as bt  # noqa: E402

Ps = [int(x) for x in sys.argv[1:]] or [37, 74, 100, 111, 112, 120, 148]
sc, pairs, uids, poses = bench.workload(0)
dev = torch.device("cuda", 0)
fb = bt.FrameBatch.from_scene(sc, dev)
ctx = bt.Context(0)
Pmax = len(pairs)
ctx.reserve(max(Ps + [Pmax]), bench.N_MAX, bench.N_HYP, bench.N_FRAMES, bench.W, bench.H)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
out = {}
for P in Ps:
    idx = np.arange(P) % Pmax
    t_pairs = torch.from_numpy(pairs[idx].copy()).to(dev)
    mt = torch.zeros((P, bench.N_MAX, 2), dtype=torch.int32, device=dev)
    nm = torch.zeros(P, dtype=torch.int32, device=dev)
    for _ in range(3):
        ctx.match(fb, t_pairs, mt, nm)
    torch.cuda.synchronize()
    ctx.profile(True)
    ctx.profile_read()
    reps = 30
    for _ in range(reps):
        flush.zero_()
        ctx.match(fb, t_pairs, mt, nm)
    torch.cuda.synchronize()
    prof = ctx.profile_read()
    ctx.profile(False)
    out[P] = {k: round(v[0] / reps * 1e3, 2) for k, v in prof.items() if v[1]}
    print(P, out[P], flush=True)
print(json.dumps(out))
