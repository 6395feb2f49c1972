"""k_ransac_score device time vs hypotheses per pair on the bench workload (wave-quantisation
check: CTAs = ceil(H / 512) * P).  usage: python tools/ransac_sweep.py"""
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

sc, pairs, uids, poses = bench.workload(0)
P = len(pairs)
dev = torch.device("cuda", 0)
fb = bt.FrameBatch.from_scene(sc, dev)
t_pairs = torch.from_numpy(pairs).to(dev)
t_uid = torch.from_numpy(uids.view(np.int32)).to(dev)
ctx = bt.Context(0)
ctx.reserve(P, bench.N_MAX, 8192, bench.N_FRAMES, bench.W, bench.H)
rec = torch.zeros((P, bt.record_words(bench.N_MAX)), dtype=torch.int32, device=dev)
mt = torch.zeros((P, bench.N_MAX, 2), dtype=torch.int32, device=dev)
nm = torch.zeros(P, dtype=torch.int32, device=dev)
ctx.match(fb, t_pairs, mt, nm)
torch.cuda.synchronize()
out = {}
for H in [int(x) for x in (sys.argv[1:] or [512, 1024, 2048, 2560, 3072, 3584, 4096, 4608, 5120, 6144, 8192])]:
    prm = bt.ransac_params(H, synth.PHILOX_SEED)
    for _ in range(3):
        ctx.ransac(fb, t_pairs, t_uid, mt, nm, prm, rec)
    torch.cuda.synchronize()
    ctx.profile(True)
    ctx.profile_read()
    for _ in range(20):
        ctx.ransac(fb, t_pairs, t_uid, mt, nm, prm, rec)
    torch.cuda.synchronize()
    pr = ctx.profile_read()
    ctx.profile(False)
    us = 1e3 * pr["k_ransac_score"][0] / pr["k_ransac_score"][1]
    out[H] = {"score_us": round(us, 2), "ns_per_hyp_pair": round(1e3 * us / (H * P), 4)}
print(json.dumps(out, indent=1))
