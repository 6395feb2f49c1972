"""One-GPU timing of BASELINE configs[4]'s shape (the stress config; the driver's bench line is
C2): 64 frames, n = 4096 keypoints (n_max 4096), all 2016 pairs, 16384 hypotheses per pair,
4032 directed dense edges at 640x480.  CUDA events around each bt_register_pairs (L2 flushed
before each, outside the events), median of `reps`.  Prints one JSON line.

usage: python tools/bench_c5.py [reps]"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2108_00516_b200 as bt  # noqa: E402
import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
F, N, H_ = 64, 4096, 16384
t0 = time.time()
sc = synth.make_scene(F, n=N, n_max=N, pool_size=14000, seed=5005, outlier_frac=0.16)
gen_s = time.time() - t0
pairs = synth.all_pairs(F)
P = len(pairs)
dev = torch.device("cuda", 0)
fb = bt.FrameBatch.from_scene(sc, dev)
t_pairs = torch.from_numpy(pairs).to(dev)
t_uid = torch.from_numpy(np.arange(P, dtype=np.int32)).to(dev)
t_pose = torch.from_numpy(sc.perturbed_poses(7)).to(dev)
ctx = bt.Context(0)
ctx.reserve(P, N, H_, F, 640, 480)
rec = torch.zeros((P, bt.record_words(N)), dtype=torch.int32, device=dev)
rprm, eprm = bt.ransac_params(H_, synth.PHILOX_SEED), bt.edge_params()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
ctx.register_pairs(fb, sc.K, t_pose, t_pairs, t_uid, rprm, eprm, rec)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
for a, b in ev:
    flush.zero_()
    a.record()
    ctx.register_pairs(fb, sc.K, t_pose, t_pairs, t_uid, rprm, eprm, rec)
    b.record()
torch.cuda.synchronize()
ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
ctx.profile(True)
ctx.profile_read()
flush.zero_()
ctx.register_pairs(fb, sc.K, t_pose, t_pairs, t_uid, rprm, eprm, rec)
torch.cuda.synchronize()
kern = {k: round(v[0], 3) for k, v in ctx.profile_read().items() if v[1]}
ctx.profile(False)
d = bt.decode_records(rec, N)
M = d["n_matches"].astype(np.int64)
out = {"workload": "C5 shape on 1 B200: 64 frames, n=4096, 2016 pairs, 16384 hypotheses/pair, 4032 dense "
                   "edges at 640x480", "ms_per_step": ms, "pairs_per_s": P / (ms * 1e-3),
       "hypotheses_per_s": P * H_ / (ms * 1e-3), "tests_per_s": float(M.sum()) * H_ / (ms * 1e-3),
       "mean_matches": float(M.mean()), "status_ok": int((d["status"] == 0).sum()), "reps": reps,
       "scene_generation_s": gen_s, "kernel_ms_instrumented_step": kern}
print(json.dumps(out))
ctx.close()
