"""Per-frame latency over a 1000-frame synthetic replay (BASELINE configs[2]'s shape) on one
B200.  The pose graph holds the current frame + K = 15 keyframes in a ring of 16 frame slots
(keyframe selection — SURVEY §8(f) NEXT-2 — is not built: the keyframes are simply the 15
previous frames).  Per frame t, on one stream:

  1. the frame's keypoints + maps arrive in a staging buffer (H2D from pinned host memory in
     the e2e variant; a device-to-device copy from a pool of rendered frames otherwise), go to
     ring slot t mod 16, and its node pose starts at the previous frame's (coarse chaining);
  2. bt_register_pairs on the 15 NEW pairs (current x keyframes: matching, RANSAC, refit,
     Eq. (2) and Eq. (3) blocks); their records and match lists (bt_copy_matches) go into the
     120-pair tables (the other 105 pairs' C_ij are reused);
  3. G Gauss-Newton iterations of Eq. (1): bt_pose_graph_step over all 120 pairs (the oldest
     keyframe fixed), then bt_relinearize_matches (Eq. (2) at the new poses over the cached
     C_ij, Eq. (3) re-associated).

Steps 1 (from the staging buffer) to 3 are one CUDA graph per ring slot (eager launches are
reported too).  CUDA events bracket each frame (no L2 flush: a tracker's working set stays hot); reported as
p50 / p90 / p99 / max over the frames after the ring fills.  Frames cycle through a pool of
rendered views of one synthetic object (the data only shapes the work).  Prints one JSON line.

usage: python tools/bench_c3.py [frames] [gn_iters] [pool]"""
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

FRAMES = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
G = int(sys.argv[2]) if len(sys.argv) > 2 else 2
POOL = int(sys.argv[3]) if len(sys.argv) > 3 else 48
KF, NMAX, H_ = 15, 512, 4096
NS = KF + 1
dev = torch.device("cuda", 0)
t0 = time.time()
sc = synth.make_scene(POOL, n=500, n_max=NMAX, seed=synth.DATA_SEED + 3)
gen_s = time.time() - t0
pool_pose = sc.perturbed_poses(seed=77)
FIELDS = ("n_kp", "desc", "pts", "nrm", "depth", "normal", "mask")
pool_dev = {f: torch.from_numpy(np.ascontiguousarray(getattr(sc, f))).to(dev) for f in FIELDS}
pool_host = {f: torch.from_numpy(np.ascontiguousarray(getattr(sc, f))).pin_memory() for f in FIELDS}
slots = {f: torch.zeros((NS,) + tuple(v.shape[1:]), dtype=v.dtype, device=dev) for f, v in pool_dev.items()}
fb = bt.FrameBatch(*(slots[f] for f in FIELDS))
pose = torch.zeros((NS, 12), dtype=torch.float32, device=dev)
pose[:, [0, 4, 8]] = 1.0                               # identity until a slot is filled
new_pose = torch.empty_like(pose)
pairs120 = synth.all_pairs(NS)
t_pairs120 = torch.from_numpy(pairs120).to(dev)
rows_of = {s: np.nonzero((pairs120 == s).any(1))[0] for s in range(NS)}   # the 15 pairs touching slot s
t_rows = {s: torch.from_numpy(rows_of[s]).to(dev) for s in range(NS)}
t_new = {s: torch.from_numpy(pairs120[rows_of[s]]).to(dev) for s in range(NS)}
rw = bt.record_words(NMAX)
rec = torch.zeros((len(pairs120), rw), dtype=torch.int32, device=dev)
rec15 = torch.zeros((KF, rw), dtype=torch.int32, device=dev)
mt = torch.zeros((len(pairs120), NMAX, 2), dtype=torch.int32, device=dev)      # the C_ij cache
nm = torch.zeros(len(pairs120), dtype=torch.int32, device=dev)
mt15 = torch.zeros((KF, NMAX, 2), dtype=torch.int32, device=dev)
nm15 = torch.zeros(KF, dtype=torch.int32, device=dev)
uid = torch.empty(KF, dtype=torch.int32, device=dev)
ctx = bt.Context(0)
ctx.reserve(len(pairs120), NMAX, H_, NS, 640, 480)
rprm, eprm = bt.ransac_params(H_, synth.PHILOX_SEED), bt.edge_params()
host_uids = torch.arange((FRAMES + NS) * KF, dtype=torch.int32).view(FRAMES + NS, KF).pin_memory()


stage = {f: torch.zeros(tuple(v.shape[1:]), dtype=v.dtype, device=dev) for f, v in pool_dev.items()}
uid_stage = torch.empty(KF, dtype=torch.int32, device=dev)


def arrive(t, host):
    """The new frame lands in the staging buffers (H2D from pinned memory, or D2D from the pool)."""
    for f in FIELDS:
        stage[f].copy_((pool_host if host else pool_dev)[f][t % POOL], non_blocking=True)
    uid_stage.copy_(host_uids[t], non_blocking=True)


def body(s):
    """Everything after the arrival, for the frame in ring slot s (ring full: t >= 16)."""
    for f in FIELDS:
        slots[f][s].copy_(stage[f])
    pose[s].copy_(pose[(s - 1) % NS])                 # coarse chaining: previous frame's pose
    uid.copy_(uid_stage)
    ctx.register_pairs(fb, sc.K, pose, t_new[s], uid, rprm, eprm, rec15)
    ctx.copy_matches(mt15, nm15)
    rec.index_copy_(0, t_rows[s], rec15)
    mt.index_copy_(0, t_rows[s], mt15)
    nm.index_copy_(0, t_rows[s], nm15)
    for _ in range(G):
        ctx.pose_graph_step(pose, t_pairs120, rec, NMAX, new_pose, fixed_node=(s + 1) % NS)
        pose.copy_(new_pose)
        ctx.relinearize(fb, sc.K, pose, t_pairs120, eprm, rec, matches=mt, n_matches=nm)


def fill():
    """Ring filling (untimed): the first 16 frames start at their perturbed ground-truth poses."""
    for t in range(NS):
        arrive(t, False)
        pose[t].copy_(torch.from_numpy(pool_pose[t % POOL]).to(dev))
        body(t)
        pose[t].copy_(torch.from_numpy(pool_pose[t % POOL]).to(dev))


def replay(host, graphs=None):
    fill()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(FRAMES)]
    for t in range(NS, NS + FRAMES):
        a, b = ev[t - NS]
        a.record()
        arrive(t, host)
        if graphs is None:
            body(t % NS)
        else:
            graphs[t % NS].replay()
        b.record()
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(b) for a, b in ev])
    return {"p50_ms": float(np.percentile(ms, 50)), "p90_ms": float(np.percentile(ms, 90)),
            "p99_ms": float(np.percentile(ms, 99)), "max_ms": float(ms.max()), "mean_ms": float(ms.mean())}


replay(False)                                          # warm-up pass (also fills every record)
eager_dev = replay(False)
graphs = []
gs = torch.cuda.Stream()
for s_ in range(NS):                                   # one graph per ring slot
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        body(s_)
    graphs.append(g)
torch.cuda.synchronize()
graph_dev = replay(False, graphs)
graph_host = replay(True, graphs)
d = bt.decode_records(rec, NMAX)
frame_bytes = sum(int(v[0].numel() * v.element_size()) for v in pool_host.values())
out = {"workload": f"C3 shape on 1 B200: {FRAMES}-frame replay, K={KF} keyframes (ring of {NS} slots), per frame "
                   f"15 new pairs registered (4096 hypotheses, dense at 640x480) + {G} Gauss-Newton iterations "
                   f"over the 120-pair graph (step + re-linearization)",
       "latency_device_resident": graph_dev,
       "latency_with_frame_h2d": dict(graph_host, h2d_bytes_per_frame=frame_bytes),
       "latency_eager_launches": eager_dev,
       "launch": "one CUDA graph per ring slot (the frame's arrival copy outside it, inside the events)",
       "frames_per_s_p50": 1e3 / graph_dev["p50_ms"], "gn_iterations": G,
       "status_ok_last_graph": int((d["status"] == 0).sum()), "pool_frames": POOL,
       "scene_generation_s": gen_s, "l2": "not flushed (tracker working set stays hot)"}
print(json.dumps(out))
ctx.close()
