"""How much of the C2 step the dense chain costs: the bench workload's bt_register_pairs captured
as a CUDA graph (as bench.py times it) with the dense edges (eprm) and without (eprm None: match
-> RANSAC -> refit only), L2 flushed before every step, CUDA events on the stream.  Also the
dense chain alone (bt_dense_corr).  A development tool.

usage: python tools/step_split.py [reps]"""
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

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
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
rprm = bt.ransac_params(bench.N_HYP, synth.PHILOX_SEED)
rec = torch.zeros((P, bt.record_words(bench.N_MAX)), dtype=torch.int32, device=dev)
dout = torch.zeros((edges.shape[0], 32), dtype=torch.float32, device=dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream(dev)
out = {}
for name, fn in {"full": lambda: ctx.register_pairs(fb, sc.K, t_pose, t_pairs, t_uid, rprm, bt.edge_params(), rec, stream=s),
                 "no_dense": lambda: ctx.register_pairs(fb, sc.K, t_pose, t_pairs, t_uid, rprm, None, rec, stream=s),
                 "dense_only": lambda: ctx.dense_corr(fb, sc.K, t_pose, edges, bt.edge_params(), dout, stream=s)}.items():
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    with torch.cuda.stream(s):
        for a, b in ev:
            flush.zero_()
            a.record(s)
            g.replay()
            b.record(s)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    out[name] = {"median_ms": t[len(t) // 2], "mean_ms": float(np.mean(t))}
    print(name, out[name], flush=True)
print(json.dumps(out))
