"""One-GPU timing of BASELINE configs[3]'s shape: 64 concurrent tracks x 120 pairs (the C2
per-frame step of every track) registered as ONE bt_register_pairs batch of 7680 pairs over
1024 frames (64 x 16), 15360 directed dense edges at 640x480, 4096 hypotheses per pair.  This
is one rank's work at N = 1; under torchrun the same batch shards by pair (bench.py,
DESIGN.md §6).  Track t uses synthetic scene t mod S (S distinct renders, to bound the CPU
scene generation), its own node-pose perturbation and its own global pair uids t*120 + k, so
every pair's hypotheses differ.  CUDA events around each call (L2 flushed before each, outside
the events), median of `reps`; a sampled pair per distinct scene is checked bitwise against the
same pair registered alone in a C2-sized call (batch invariance).  Prints one JSON line.

usage: python tools/bench_c4.py [reps] [tracks] [distinct_scenes]"""
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

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
S = int(sys.argv[3]) if len(sys.argv) > 3 else 8
NF, N, NMAX, H_ = 16, 500, 512, 4096
dev = torch.device("cuda", 0)
t0 = time.time()
scenes = [synth.make_scene(NF, n=N, n_max=NMAX, seed=synth.DATA_SEED + s) for s in range(S)]
gen_s = time.time() - t0
K = scenes[0].K
base = synth.all_pairs(NF)
P1 = len(base)


def cat(field, dtype=None):
    parts = [torch.from_numpy(np.ascontiguousarray(getattr(scenes[t % S], field))).to(dev) for t in range(S)]
    return torch.cat([parts[t % S] for t in range(T)], 0).contiguous()


fb = bt.FrameBatch(cat("n_kp"), cat("desc"), cat("pts"), cat("nrm"), cat("depth"), cat("normal"), cat("mask"))
pairs = np.concatenate([base + NF * t for t in range(T)]).astype(np.int32)
uids = np.arange(T * P1, dtype=np.uint32)
poses = np.concatenate([scenes[t % S].perturbed_poses(seed=1000 + t) for t in range(T)])
P = len(pairs)
t_pairs = torch.from_numpy(pairs).to(dev)
t_uid = torch.from_numpy(uids.view(np.int32)).to(dev)
t_pose = torch.from_numpy(poses).to(dev)
ctx = bt.Context(0)
ctx.reserve(P, NMAX, H_, T * NF, 640, 480)
rec = torch.zeros((P, bt.record_words(NMAX)), dtype=torch.int32, device=dev)
rprm, eprm = bt.ransac_params(H_, synth.PHILOX_SEED), bt.edge_params()
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
ctx.register_pairs(fb, K, t_pose, t_pairs, t_uid, rprm, eprm, rec)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
for a, b in ev:
    flush.zero_()
    a.record()
    ctx.register_pairs(fb, K, t_pose, t_pairs, t_uid, rprm, eprm, rec)
    b.record()
torch.cuda.synchronize()
ms_all = [a.elapsed_time(b) for a, b in ev]
ms = float(np.median(ms_all))
ctx.profile(True)
ctx.profile_read()
flush.zero_()
ctx.register_pairs(fb, K, t_pose, t_pairs, t_uid, rprm, eprm, rec)
torch.cuda.synchronize()
kern = {k: round(v[0], 3) for k, v in ctx.profile_read().items() if v[1]}
ctx.profile(False)

# batch invariance: track t's pairs registered alone (frames of that track only) == the batch rows
inv_ok = True
for t in sorted({0, T - 1} | set(range(min(S, T)))):
    sc = scenes[t % S]
    fb1 = bt.FrameBatch.from_scene(sc, dev)
    r1 = torch.zeros((P1, rec.shape[1]), dtype=torch.int32, device=dev)
    ctx.register_pairs(fb1, K, t_pose[NF * t:NF * (t + 1)].contiguous(), torch.from_numpy(base).to(dev),
                       t_uid[P1 * t:P1 * (t + 1)].contiguous(), rprm, eprm, r1)
    torch.cuda.synchronize()
    inv_ok &= bool(torch.equal(r1, rec[P1 * t:P1 * (t + 1)]))
d = bt.decode_records(rec, NMAX)
M = d["n_matches"].astype(np.int64)
out = {"workload": f"C4 shape on 1 B200: {T} tracks x {P1} pairs = {P} pairs in one call ({T * NF} frames, "
                   f"{2 * P} dense edges at 640x480), {H_} hypotheses/pair; {S} distinct synthetic scenes",
       "ms_per_step": ms, "ms_all": ms_all, "pairs_per_s": P / (ms * 1e-3), "hypotheses_per_s": P * H_ / (ms * 1e-3),
       "tests_per_s": float(M.sum()) * H_ / (ms * 1e-3), "mean_matches": float(M.mean()),
       "status_ok": int((d["status"] == 0).sum()), "batch_invariant": inv_ok, "reps": reps,
       "l2": "flushed (512 MB write) before each call, outside the events",
       "scene_generation_s": gen_s, "kernel_ms_instrumented_step": kern}
print(json.dumps(out))
ctx.close()
