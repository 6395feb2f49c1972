"""Pose-graph step (NEXT-1) on the C2 graph, called `reps` times after one registration —
for an ncu launch list of k_graph_contrib / k_graph_assemble / k_graph_pcg.
usage: python tools/time_graph.py [reps] [max_iter] [precond]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2108_00516_b200 as bt  # noqa: E402
import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 200
precond = int(sys.argv[3]) if len(sys.argv) > 3 else 1
sc = synth.make_scene(16)
pairs = torch.from_numpy(synth.all_pairs(16)).cuda()
uid = torch.arange(120, dtype=torch.int32).cuda()
pose = torch.from_numpy(sc.perturbed_poses(1000)).cuda()
fb = bt.FrameBatch.from_scene(sc)
ctx = bt.Context(0)
ctx.reserve(120, 512, 4096, 16, 640, 480)
rec = torch.zeros((120, bt.record_words(512)), dtype=torch.int32, device="cuda")
ctx.register_pairs(fb, sc.K, pose, pairs, uid, bt.ransac_params(4096, synth.PHILOX_SEED), bt.edge_params(), rec)
new = torch.empty_like(pose)
st = torch.zeros(4, dtype=torch.float32, device="cuda")
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
for a, b in ev:
    a.record()
    ctx.pose_graph_step(pose, pairs, rec, 512, new, stats=st, max_iter=max_iter, precond=precond)
    b.record()
torch.cuda.synchronize()
print("ms per call", np.median([a.elapsed_time(b) for a, b in ev]), "stats", st.cpu().numpy())
ctx.close()
