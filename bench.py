#!/usr/bin/env python
"""bench.py — throughput of the BundleTrack pairwise-registration hot path on B200.

One STEP = one bt_register_pairs call over the BundleTrack per-frame workload of
BASELINE.json configs[1] ("C2"): the current frame against K = 15 keyframes -> the 16-node
pose graph's 120 frame pairs, n = 500 keypoints (128-d), 640x480 depth / normal / mask maps,
4096 RANSAC hypotheses per pair: mutual-NN matching -> RANSAC -> refit -> Eq. (2) feature
blocks -> both directed Eq. (3) dense edges (240).  Under torchrun each rank runs its own
track (weak scaling) and the per-pair records are all-gathered over NCCL (the exchange the
pose-graph solve needs).

Beside the headline, the line carries SURVEY §8(e)'s sharded configurations, strong scaling
(fixed total work split over the N ranks, records all-gathered over NCCL, max over ranks):
`c4` = BASELINE configs[3], 64 tracks x 120 pairs track-major (default; --no-c4 skips it) and,
with --c5, `c5` = configs[4], 2016 pairs of n = 4096 keypoints in contiguous pair blocks.

Prints ONE JSON line (rank 0).  `--impl reference` times the CPU oracle (oracle/, plain C,
fp64) on a bounded sample of the same workload instead.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "frame-pairs registered/sec + RANSAC hypotheses/sec at 1/2/4/8 B200 vs roofline"
UNIT = "pairs/s"
N_FRAMES, N_KP, N_MAX, N_HYP, W, H = 16, 500, 512, 4096, 640, 480
# Algorithmic work per (hypothesis, correspondence) test = SURVEY §8(d)'s per-unit figure:
# 24 FMA-pipe instructions = 43 flop (distance gate |R a + t - b|^2 < delta^2: 9 FFMA + 3 FADD
# + 3 FFMA; normal gate <R, n_b n_a^T> > cos(alpha): 9 FFMA).  The short-circuit lower bound
# (27 flop per test + 18 only where the distance passes) is reported beside it.
FLOPS_TEST = 43
FLOPS_DIST, FLOPS_NORMAL = 27, 18
SM_COUNT, FP32_LANES = 148, 128


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--e2e-warmup-s", type=float, default=1.0,
                    help="seconds of untimed calls before each e2e measurement (the host link's "
                         "throughput ramps up over the first ~second of transfers)")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the step's kernels one by one instead of replaying it as a CUDA graph")
    ap.add_argument("--no-kernel-events", action="store_true",
                    help="time the step without the per-kernel CUDA-event brackets (overhead check)")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 multi-track block")
    ap.add_argument("--c4-steps", type=int, default=10)
    ap.add_argument("--c4-scenes", type=int, default=8,
                    help="distinct synthetic scenes the 64 tracks cycle through (bounds CPU scene generation)")
    ap.add_argument("--c5", action="store_true", help="add the C5 stress block (n=4096, 2016 pairs; slow to generate)")
    ap.add_argument("--c5-steps", type=int, default=3)
    ap.add_argument("--exchange", default="nccl", choices=["fused", "nccl"],
                    help="N > 1 record exchange: NCCL all_gather_into_tensor (default, measured path) or the fused "
                         "producer stores into symmetric-memory gather buffers (NEXT-3; tested on one GPU only)")
    return ap.parse_args()


def workload(rank: int):
    """Rank r's track: the C2 scene with seed DATA_SEED + r, node poses perturbed by <= 5 deg /
    2 cm (the state a pose-graph iteration linearizes at), global pair uids r*120 + k."""
    sc = synth.make_scene(N_FRAMES, n=N_KP, n_max=N_MAX, width=W, height=H, seed=synth.DATA_SEED + rank)
    pairs = synth.all_pairs(N_FRAMES)
    uids = (rank * len(pairs) + np.arange(len(pairs))).astype(np.uint32)
    poses = sc.perturbed_poses(seed=1000 + rank)
    return sc, pairs, uids, poses


C4_TRACKS = 64


def multi_block(kind, args, bt, parallel, torch, dist, world, rank, local, dev, flush):
    """SURVEY §8(e)'s sharded configurations, timed like the headline (L2 flushed before each
    step outside the events, CUDA events on the launching stream, barrier + synchronize on both
    sides, max over ranks), each step = this rank's bt_register_pairs + the NCCL
    all_gather_into_tensor of the records (the exchange the pose-graph solve needs).  Strong
    scaling: the total work is fixed, each rank takes its share.
      c4: BASELINE configs[3] — 64 tracks x 120 pairs (the C2 step of every track), track-major:
          rank r holds only its 64/N tracks' frames (no input replication);
      c5: BASELINE configs[4] — 64 frames, n = 4096, 2016 pairs, 16384 hypotheses, pair blocks:
          frames replicated, rank r registers the contiguous block shard_range(2016, N, r)."""
    t0 = time.perf_counter()
    if kind == "c4":
        S = max(1, args.c4_scenes)
        tp = synth.all_pairs(N_FRAMES)
        plan = parallel.track_plan(C4_TRACKS, N_FRAMES, tp, world, rank)
        t_lo, t_hi = plan.frame_lo // N_FRAMES, plan.frame_hi // N_FRAMES
        need = sorted({t % S for t in range(t_lo, t_hi)})
        scenes = {s_: synth.make_scene(N_FRAMES, n=N_KP, n_max=N_MAX, width=W, height=H, seed=synth.DATA_SEED + 100 + s_)
                  for s_ in need}
        tsc = [scenes[t % S] for t in range(t_lo, t_hi)]
        poses = np.concatenate([tsc[t - t_lo].perturbed_poses(seed=2000 + t) for t in range(t_lo, t_hi)])
        n_max, n_hyp, steps, K = N_MAX, N_HYP, args.c4_steps, tsc[0].K
        workload_ = (f"C4: {C4_TRACKS} tracks x {len(tp)} pairs = {C4_TRACKS * len(tp)} pairs per step "
                     f"({C4_TRACKS * N_FRAMES} frames, {2 * C4_TRACKS * len(tp)} dense edges, 640x480, n=500, "
                     f"{N_HYP} hypotheses/pair), track-major: {t_hi - t_lo} tracks on this rank; tracks cycle "
                     f"through {S} distinct synthetic scenes, each with its own node poses and global pair uids")

        def field(f):
            return torch.cat([torch.from_numpy(np.ascontiguousarray(getattr(x, f))).to(dev) for x in tsc], 0)
    else:
        sc = synth.make_scene(64, n=4096, n_max=4096, pool_size=14000, seed=5005, outlier_frac=0.16)
        pairs_all = synth.all_pairs(64)
        plan = parallel.pair_block_plan(pairs_all, 64, world, rank)
        poses = sc.perturbed_poses(7)
        n_max, n_hyp, steps, K = 4096, 16384, args.c5_steps, sc.K
        workload_ = (f"C5: 64 frames, n=4096, {len(pairs_all)} pairs ({2 * len(pairs_all)} dense edges at 640x480), "
                     f"16384 hypotheses/pair; pair blocks: pairs [{plan.row_lo}, {plan.row_lo + len(plan.pairs)}) on "
                     "this rank, frames replicated")

        def field(f):
            return torch.from_numpy(np.ascontiguousarray(getattr(sc, f))).to(dev)
    gen_s = time.perf_counter() - t0
    fb = bt.FrameBatch(*(field(f) for f in ("n_kp", "desc", "pts", "nrm", "depth", "normal", "mask")))
    P_r = len(plan.pairs)
    n_total = int(sum(plan.rows))
    t_pairs = torch.from_numpy(plan.pairs).to(dev)
    t_uid = torch.from_numpy(plan.uids.view(np.int32)).to(dev)
    t_pose = torch.from_numpy(np.ascontiguousarray(poses)).to(dev)
    rec = torch.zeros((P_r, bt.record_words(n_max)), dtype=torch.int32, device=dev)
    ctx = bt.Context(local)
    ctx.reserve(max(P_r, 1), n_max, n_hyp, int(fb.desc.shape[0]), W, H)
    rprm, eprm = bt.ransac_params(n_hyp, synth.PHILOX_SEED), bt.edge_params()
    stream = torch.cuda.current_stream(dev)
    gathered = [None]
    # the exchange: NEXT-3's fused record stores into every rank's symmetric-memory gather buffer
    # (one barrier), else one NCCL all_gather_into_tensor of the records
    fused = None
    if world > 1 and args.exchange == "fused" and parallel.FusedRecordExchange.available():
        try:
            fused = parallel.FusedRecordExchange(ctx, plan.rows, bt.record_words(n_max), device=dev)
        except Exception as e:                                   # no peer access: NCCL all-gather
            print(f"[bench] fused record exchange unavailable ({type(e).__name__}: {e}); NCCL all-gather",
                  file=sys.stderr)
            fused = None
    exchange_kind = ("fused: producer kernels store each record word into every rank's symmetric-memory "
                     "gather buffer (bt_set_record_peers), one barrier" if fused is not None else
                     f"one all_gather_into_tensor of the fixed-stride records over NCCL")

    def exchange():
        if world > 1:
            gathered[0] = fused.finish() if fused is not None else parallel.all_gather_rows(rec, plan.rows)

    def one():
        if P_r:
            ctx.register_pairs(fb, K, t_pose, t_pairs, t_uid, rprm, eprm, rec, stream=stream)
        exchange()
    for _ in range(2):
        one()
    torch.cuda.synchronize()
    launches = ctx.last_launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    gx = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(steps):
            flush.zero_()
            ev[k][0].record(stream)
            if P_r:
                ctx.register_pairs(fb, K, t_pose, t_pairs, t_uid, rprm, eprm, rec, stream=stream)
            gx[k][0].record(stream)
            exchange()
            gx[k][1].record(stream)
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = float(sum(a.elapsed_time(b) for a, b in ev))
    gms = float(sum(a.elapsed_time(b) for a, b in gx))
    t_ = torch.tensor([ms, gms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
    ms_max, gms_max = float(t_[0].item()), float(t_[1].item())
    d = bt.decode_records(rec, n_max)
    ok = torch.tensor([int((d["status"] == 0).sum()), int(d["n_matches"].astype(np.int64).sum())],
                      dtype=torch.int64, device=dev)
    same = None
    if world > 1:
        dist.all_reduce(ok)
        assert gathered[0].shape[0] == n_total
        # the exchange is exact: this rank's rows of the gathered table are its own records
        same = bool(torch.equal(gathered[0][plan.row_lo: plan.row_lo + P_r], rec))
    if fused is not None:
        fused.close()
    ctx.close()
    del fb, rec
    torch.cuda.empty_cache()
    sec = ms_max / 1e3
    return {"workload": workload_, "pairs_per_step": n_total, "value": n_total * steps / sec, "unit": UNIT,
            "hypotheses_per_s": n_total * n_hyp * steps / sec, "tests_per_s": float(ok[1].item()) * n_hyp * steps / sec,
            "ms_per_step": ms_max / steps, "exchange_ms_per_step": gms_max / steps, "steps": steps, "warmup": 2,
            "scaling": "strong", "n_gpus": world, "pairs_this_rank": P_r, "status_ok": int(ok[0].item()),
            "gpu_launches": launches * steps, "clocks": clk.summary(), "scene_generation_s": gen_s,
            "exchange": (f"{exchange_kind} ({4 * bt.record_words(n_max)} B per pair, {n_total} pairs)"
                         if world > 1 else "none (one rank)"),
            "exchange_rows_match_local": same,
            "l2": "flushed (512 MiB memset) before each step, outside the events",
            "launch": "eager (the step is ms-long; launch overhead is negligible)"}


def dense_params():
    return dict(dist_gate=0.02, cos_gate=float(np.cos(np.deg2rad(45.0))), huber_delta=0.005, stride=1)


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampler of SM clock and clock-event reasons during the timed region."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index: int, period_s: float = 0.001):
        self.samples, self.reasons = [], set()
        self.period = period_s
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
            self.max_mhz = None
        self._stop = threading.Event()

    def _sample(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        try:
            self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            r = get_r(self.h)
            for bit, name in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        # every ~1 ms while the timed region runs (a 20-step C2 region is ~6 ms of GPU time)
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------- the oracle arm
def oracle_pairs_per_s(sc, pairs, uids, poses, sample_pairs):
    """The CPU oracle as it stands (single thread) on `sample_pairs` of the workload."""
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    for p in sample_pairs:
        a, b = pairs[p]
        oracle.register_pair(sc, int(a), int(b), int(uids[p]), N_HYP, synth.PHILOX_SEED, node_poses=poses,
                             dense=dense_params())
    dt = time.perf_counter() - t0
    return len(sample_pairs) / dt, dt


_ORC = None


def _oracle_one(p):
    sc, pairs, uids, poses = _ORC
    import oracle
    a, b = pairs[p]
    oracle.register_pair(sc, int(a), int(b), int(uids[p]), N_HYP, synth.PHILOX_SEED, node_poses=poses,
                         dense=dense_params())
    return p


def oracle_all_cores(sc, pairs, uids, poses, sample_pairs, reps=3):
    """The same oracle, unchanged (each pair's registration stays plain and serial), over all
    host cores: a process per core, pairs handed out one at a time ("all cores
    with OpenMP parallel for over pairs/edges" — processes instead of threads, same partition).
    Returns (pairs/s, cores, seconds of the timed reps)."""
    import multiprocessing as mp
    global _ORC
    import oracle
    oracle.build()
    oracle.lib()
    _ORC = (sc, pairs, uids, poses)
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_oracle_one, list(sample_pairs)[:cores], chunksize=1)        # warm the workers
        t0 = time.perf_counter()
        for _ in range(reps):
            pool.map(_oracle_one, list(sample_pairs), chunksize=1)
        dt = time.perf_counter() - t0
    _ORC = None
    return reps * len(sample_pairs) / dt, cores, dt


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sc, pairs, uids, poses = workload(0)
    # each step: one frame pair of the C2 workload (round robin), full per-pair work
    for s in range(args.warmup):
        oracle_pairs_per_s(sc, pairs, uids, poses, [s % len(pairs)])
    t0 = time.perf_counter()
    for s in range(args.steps):
        oracle_pairs_per_s(sc, pairs, uids, poses, [(args.warmup + s) % len(pairs)])
    dt = time.perf_counter() - t0
    value = args.steps / dt
    sample = (f"1 of the 120 C2 frame pairs per step (round robin): matching + {N_HYP}-hypothesis RANSAC + "
              f"refit + Eq.(2) blocks + both dense edges at {W}x{H}")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_block(),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                             "cpu": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_block():
    return {"workload": "C2: BundleTrack per-frame step, current frame vs K=15 keyframes (120 pairs, 240 "
                        "directed dense edges), n=500 keypoints, 128-d descriptors, 640x480 maps, 4096 "
                        "hypotheses/pair",
            "pairs_per_step": 120, "n": N_KP, "n_max": N_MAX, "hypotheses_per_pair": N_HYP, "frames": N_FRAMES,
            "height": H, "width": W, "l2": "flushed between timed steps (512 MiB memset, outside the events)"}


# --------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2108_00516_b200 as bt
    from paper_2108_00516_b200 import parallel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    sc, pairs, uids, poses = workload(rank)
    P = len(pairs)
    fb = bt.FrameBatch.from_scene(sc, dev)
    t_pairs = torch.from_numpy(pairs).to(dev)
    t_uid = torch.from_numpy(uids.view(np.int32)).to(dev)
    t_pose = torch.from_numpy(poses).to(dev)
    rw = bt.record_words(N_MAX)
    rec = torch.zeros((P, rw), dtype=torch.int32, device=dev)
    ctx = bt.Context(local)
    ctx.reserve(P, N_MAX, N_HYP, N_FRAMES, W, H)
    rprm = bt.ransac_params(N_HYP, synth.PHILOX_SEED)
    eprm = bt.edge_params()
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step():
        ctx.register_pairs(fb, sc.K, t_pose, t_pairs, t_uid, rprm, eprm, rec, stream=stream)
        if world > 1:                                    # the pose-graph exchange
            parallel.all_gather_records(rec, world * P)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = ctx.last_launches
    dec = bt.decode_records(rec, N_MAX)
    M = dec["n_matches"].astype(np.int64)
    tests = int(M.sum()) * N_HYP
    # sum of per-hypothesis inlier counts (a lower bound on the distance-gate passes), from one
    # bt_match + bt_ransac call with per-hypothesis counts, outside the timed region
    mt_ = torch.zeros((P, N_MAX, 2), dtype=torch.int32, device=dev)
    nm_ = torch.zeros(P, dtype=torch.int32, device=dev)
    hc_ = torch.zeros((P, N_HYP), dtype=torch.int32, device=dev)
    rec_ = torch.zeros_like(rec)
    ctx.match(fb, t_pairs, mt_, nm_, stream=stream)
    ctx.ransac(fb, t_pairs, t_uid, mt_, nm_, rprm, rec_, hc_, stream=stream)
    torch.cuda.synchronize()
    sum_counts = int(hc_.clamp(min=0).sum().item())
    n_assoc = float(dec["dense_ij"][:, 28].sum() + dec["dense_ji"][:, 28].sum())

    # standalone per-kernel device times (each C-ABI stage alone, outside the timed region): in
    # the step the dense chain runs on a low-priority stream beside matching / RANSAC, so its
    # in-step brackets include time it waits for SMs; the dominant kernel is chosen on these
    edges_t = torch.from_numpy(np.concatenate([pairs, pairs[:, ::-1]], 0).astype(np.int32).copy()).to(dev)
    dout_ = torch.zeros((edges_t.shape[0], 32), dtype=torch.float32, device=dev)
    ctx.profile(True)
    ctx.profile_read()
    for _ in range(5):
        flush.zero_()
        ctx.match(fb, t_pairs, mt_, nm_, stream=stream)
        ctx.ransac(fb, t_pairs, t_uid, mt_, nm_, rprm, rec_, stream=stream)
        ctx.dense_corr(fb, sc.K, t_pose, edges_t, eprm, dout_, stream=stream)
    torch.cuda.synchronize()
    solo = {k: v for k, v in ctx.profile_read().items() if v[1]}
    ctx.profile(False)
    del mt_, nm_, hc_, rec_, dout_

    graph_exec = None
    if not args.no_graph:
        # the step's bt_register_pairs call (fork to the dense stream, match -> RANSAC, join)
        # captured once as a CUDA graph and replayed every step (the C ABI only enqueues
        # stream-ordered work; tests/test_gpu_parity.py checks replay == eager bitwise)
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(stream)
        graph_exec = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_exec, stream=gs):
            ctx.register_pairs(fb, sc.K, t_pose, t_pairs, t_uid, rprm, eprm, rec, stream=gs)
        stream.wait_stream(gs)
        torch.cuda.synchronize()

    def run_step(instrumented):
        if graph_exec is not None and not instrumented:
            graph_exec.replay()
            if world > 1:                                # the pose-graph exchange, after the replay
                parallel.all_gather_records(rec, world * P)
        else:
            step()

    def timed_region(instrumented: bool, only=None):
        """K steps, L2 flushed before each (outside the events), CUDA events around each step on
        the launching stream, barrier + synchronize on both sides, max over ranks."""
        ctx.profile(instrumented, only=only)
        ctx.profile_read()
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        stops = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk_:
            for k in range(args.steps):
                flush.zero_()                            # evict L2 (outside the events)
                starts[k].record(stream)
                run_step(instrumented)
                stops[k].record(stream)
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms_ = float(sum(a.elapsed_time(b) for a, b in zip(starts, stops)))
        t_ = torch.tensor([ms_], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        prof_ = ctx.profile_read() if instrumented else {}
        ctx.profile(False)
        return ms_, float(t_.item()), clk_, prof_

    # the headline: the step WITHOUT per-kernel instrumentation (the per-kernel event pairs
    # cost ~12 % of the step); then the same K steps again with every kernel bracketed by
    # CUDA events on its stream, for the per-kernel durations of the roofline block
    ms, ms_max, clk, _ = timed_region(False)
    prof_dom, ms_d = {}, None
    if args.no_kernel_events:
        ms_i, prof = ms, {}
    else:
        ms_i, _, _, prof = timed_region(True)
        # the dominant stage alone bracketed (every other kernel unbracketed, as in the headline
        # region): its in-step duration with the streams' overlap perturbed least
        ms_d, _, _, prof_dom = timed_region(True, only="k_ransac_score")
    sec = ms_max / 1e3
    value = world * P * args.steps / sec
    hyp_per_s = world * P * N_HYP * args.steps / sec

    # ---- per-kernel roofline (algorithmic work / measured launch duration) ----------
    mhz_max = 1965.0
    fp32_peak_tflops = SM_COUNT * FP32_LANES * 2 * mhz_max * 1e6 / 1e12
    import json as _j
    peaks = _j.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    npx = W * H
    kern = {}

    def add(name, bound, work_per_step, unit, peak, note):
        tot, n = prof.get(name, (0.0, 0))
        if n == 0:
            return
        step_ms = tot / args.steps                      # this kernel's device time per step
        ach = work_per_step / (step_ms / 1e3) / (1e12 if unit == "TFLOP/s" else 1e9)
        st, sn = solo.get(name, (0.0, 0))
        solo_ms = st / 5 if sn else None
        kern[name] = {"bound": bound, "achieved": ach, "peak": peak, "unit": unit, "frac": ach / peak,
                      "avg_launch_ms": tot / n, "launches_per_step": n / args.steps,
                      "share_of_step": tot / ms_i if ms_i else None,
                      "standalone_ms_per_step": solo_ms,
                      # the same work over the stage's time when it runs alone (no dense stream beside it)
                      "frac_standalone": (work_per_step / (solo_ms / 1e3) / (1e12 if unit == "TFLOP/s" else 1e9) / peak)
                      if solo_ms else None, "work": note}
    pair_sizes = float(sum(int(sc.n_kp[a]) * int(sc.n_kp[b]) for a, b in pairs))
    tc_peak = float(peaks.get("bf16_tflops", 1614.4))     # fp16 kind::f16 = bf16 rate (guide ratio 1:1)
    add("k_match_tc", "tensor", 2 * pair_sizes * 128, "TFLOP/s", tc_peak,
        "2 n_a n_b 128 flop per pair (the Gram contraction, counted once)")
    add("k_ransac_score", "alu", tests * FLOPS_TEST, "TFLOP/s", fp32_peak_tflops,
        f"{FLOPS_TEST} flop per (hypothesis, correspondence) test (SURVEY 8(d)); {tests} tests; measured on "
        "the scoring stage as launched: k_corr_feat + k_score_tc (tcgen05 fp16 hi/lo contractions + "
        "FMA/ALU epilogue, DESIGN.md R27) + k_score_fix, or the FFMA2 kernel with "
        "BT_SCORE_FMA=1; peak = the FP32 FMA pipe of the direct formulation")
    if "k_ransac_score" in kern and not os.environ.get("BT_SCORE_FMA") == "1":
        # the same stage seen as tensor work: 6 MMAs x 16 K x 2 flop per (hypothesis row,
        # correspondence column) of every computed 128 x 64 tile, padding columns included
        cols = float(sum(((int(c) + 63) // 64) * 64 for c in M if c >= 3))
        tc_flop = cols * ((N_HYP + 127) // 128) * 128 * 6 * 16 * 2
        t = kern["k_ransac_score"]
        t["tensor_view"] = {"flop": tc_flop, "achieved_tflops": tc_flop / (t["avg_launch_ms"] * t["launches_per_step"] / 1e3) / 1e12,
                            "peak_tflops": tc_peak}
    if "k_match_tc" in kern:
        # the matching kernel is bound by its epilogue, not the tensor pipe (ncu: ALU pipe ~56 %,
        # tensor ~22 %): the same launches seen as the top-3 selection's work — 4
        # integer min/max per (row, column) element and direction (two keys per step: min, max,
        # 3 max + 3 min-of-3 into the running top-3), on the ALU pipe's 64 lanes/clk/SM
        t = kern["k_match_tc"]
        sel_ops = 2 * pair_sizes * 4
        alu_peak = SM_COUNT * 64 * mhz_max * 1e6 / 1e12          # T lane-ops/s
        sec = t["avg_launch_ms"] * t["launches_per_step"] / 1e3
        t["alu_view"] = {"ops": sel_ops, "achieved_tops": sel_ops / sec / 1e12, "peak_tops": alu_peak,
                         "frac": sel_ops / sec / 1e12 / alu_peak,
                         "frac_standalone": (sel_ops / (t["standalone_ms_per_step"] / 1e3) / 1e12 / alu_peak
                                             if t.get("standalone_ms_per_step") else None),
                         "work": "4 integer min/max per element per direction (2 n_a n_b per pair), "
                                 "ALU pipe 64 lanes/clk/SM"}
    if "k_ransac_score" in kern:                       # the short-circuit lower bound, for reference
        lb = tests * FLOPS_DIST + sum_counts * FLOPS_NORMAL
        kern["k_ransac_score"]["frac_short_circuit_lower_bound"] = kern["k_ransac_score"]["frac"] * lb / (
            tests * FLOPS_TEST)
        kern["k_ransac_score"]["short_circuit_work"] = (
            f"{FLOPS_DIST} flop per test + {FLOPS_NORMAL} per inlier ({sum_counts} inliers)")
    valid_per_frame = np.array([float(((sc.mask[f] > 0) & (sc.depth[f] > 0)).sum()) for f in range(N_FRAMES)])
    src_px_edges = float(sum(valid_per_frame[a] + valid_per_frame[b] for a, b in pairs))
    add("k_dense", "alu", 30 * src_px_edges + 160 * n_assoc, "TFLOP/s", fp32_peak_tflops,
        "30 flop per (valid source pixel, edge) + 160 flop per associated (pixel, edge)")
    # prep: must-read bytes = every mask byte + depth & normal of valid pixels; writes 32 B per entry
    add("k_dense_prep", "hbm", N_FRAMES * npx * 1 + valid_per_frame.sum() * (16 + 32), "GB/s", hbm_peak,
        "mask of every pixel + depth/normal of valid pixels + 32-B entry per valid pixel")
    # DRAM bytes per step of each stage's launches (ncu --set full, profiles/ncu_traffic.json:
    # dram__bytes_read.sum + dram__bytes_write.sum per launch), beside the algorithmic bytes of
    # the HBM-bound stage — traffic well above them would be re-reads
    tf_all = {}
    tf_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf_path):
        tf_all = _j.load(open(tf_path))
    members = {"k_match_tc": ["k_match_ws"], "k_ransac_score": ["k_corr_feat", "k_score_tc", "k_score_fix"],
               "k_dense": ["k_dense"], "k_dense_prep": ["k_edge_setup", "k_dense_mask", "k_dense_prep", "k_dense_scan"]}
    for name, ks in members.items():
        if name in kern and all(k in tf_all for k in ks):
            kern[name]["traffic_per_step"] = float(sum(tf_all[k] for k in ks))
    if "k_dense_prep" in kern:
        alg = N_FRAMES * npx * 1 + valid_per_frame.sum() * (16 + 32)
        kern["k_dense_prep"]["algorithmic_bytes_per_step"] = float(alg)
        if "traffic_per_step" in kern["k_dense_prep"]:
            kern["k_dense_prep"]["traffic_over_algorithmic"] = kern["k_dense_prep"]["traffic_per_step"] / alg
    # dominant = the largest standalone device time per step (agrees with the serialised ncu
    # launch list); `achieved` stays the in-step CUDA-event duration, overlap included
    dom = max(kern, key=lambda k: kern[k]["standalone_ms_per_step"] or 0) if kern else None
    step_ms_by_kernel = {k: v[0] / args.steps for k, v in prof.items() if v[1]}
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if dom and os.path.exists(tf):
        traffic = _j.load(open(tf)).get(dom)
    roof = dict(kern[dom]) if dom else None
    if roof and dom == "k_ransac_score" and prof_dom.get(dom, (0.0, 0))[1]:
        # `achieved` from the region where only this stage is bracketed (the others unbracketed,
        # as in the headline): bracketing every kernel perturbs the streams' overlap, which
        # stretches this stage in step — that figure stays as frac_all_bracketed
        tot_d, n_d = prof_dom[dom]
        work = roof["achieved"] * (roof["avg_launch_ms"] * roof["launches_per_step"] / 1e3)
        roof["frac_all_bracketed"] = roof["frac"]
        roof["avg_launch_ms"] = tot_d / n_d
        roof["achieved"] = work / (tot_d / args.steps / 1e3)
        roof["frac"] = roof["achieved"] / roof["peak"]
        roof["share_of_step"] = tot_d / ms_d if ms_d else None
        if "tensor_view" in roof:
            tv = dict(roof["tensor_view"])
            tv["achieved_tflops"] = tv["flop"] / (tot_d / args.steps / 1e3) / 1e12
            roof["tensor_view"] = tv
        roof["in_step_region"] = ("only this stage's launches bracketed by CUDA events (on its stream) over K "
                                  "steps; ms_per_step of that region " + f"{ms_d / args.steps:.4f}")
    if roof:
        roof["kernel"] = dom
        roof["traffic"] = traffic
        roof["peak_note"] = ("FP32 FMA pipe: 148 SMs x 128 lanes x 2 flop x 1965 MHz (derived, B200_PROFILING "
                             "unit counts)" if roof["bound"] == "alu" else "MEASURED_PEAKS.json hbm_gbs")

    # ---- NEXT-1: one pose-graph Gauss-Newton step on this step's records -----
    # assemble (fp64, fixed order) + Jacobi-PCG + exp update, 16 nodes / 120 pairs; CUDA
    # events on the stream, outside the headline timed region
    graph = None
    if world == 1:
        new_pose = torch.zeros_like(t_pose)
        gst = torch.zeros(4, dtype=torch.float32, device=dev)
        for _ in range(3):
            ctx.pose_graph_step(t_pose, t_pairs, rec, N_MAX, new_pose, stats=gst, stream=stream)
        torch.cuda.synchronize()
        ctx.profile(True)
        ctx.profile_read()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 100
        g0.record(stream)
        for _ in range(reps):
            ctx.pose_graph_step(t_pose, t_pairs, rec, N_MAX, new_pose, stats=gst, stream=stream)
        g1.record(stream)
        torch.cuda.synchronize()
        gprof = ctx.profile_read().get("k_graph", (0.0, 0))
        ctx.profile(False)
        st = gst.cpu().numpy()
        jac = torch.zeros(4, dtype=torch.float32, device=dev)   # the diagonal (Jacobi) preconditioner
        ctx.pose_graph_step(t_pose, t_pairs, rec, N_MAX, new_pose, stats=jac, precond=0, stream=stream)
        j0, j1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        j0.record(stream)
        for _ in range(10):
            ctx.pose_graph_step(t_pose, t_pairs, rec, N_MAX, new_pose, stats=jac, precond=0, stream=stream)
        j1.record(stream)
        torch.cuda.synchronize()
        jac = jac.cpu().numpy()
        # one full Gauss-Newton iteration of the per-frame optimisation: re-linearize the Eq. (2)
        # / Eq. (3) blocks at the current poses (C_ij reused, dense re-associated) + the step
        rec_gn = rec.clone()
        pose_a, pose_b = t_pose.clone(), torch.zeros_like(t_pose)
        for _ in range(2):
            ctx.relinearize(fb, sc.K, pose_a, t_pairs, eprm, rec_gn, stream=stream)
            ctx.pose_graph_step(pose_a, t_pairs, rec_gn, N_MAX, pose_b, stream=stream)
        n0, n1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gn_reps = 20
        n0.record(stream)
        for _ in range(gn_reps):
            ctx.relinearize(fb, sc.K, pose_a, t_pairs, eprm, rec_gn, stream=stream)
            ctx.pose_graph_step(pose_a, t_pairs, rec_gn, N_MAX, pose_b, stream=stream)
            pose_a, pose_b = pose_b, pose_a
        n1.record(stream)
        torch.cuda.synchronize()
        graph = {"api": "bt_pose_graph_step", "precond": "block-Jacobi (6x6 node blocks, reading R23)",
                 "ms_per_call": g0.elapsed_time(g1) / reps, "nodes": N_FRAMES,
                 "pairs": P, "unknowns": 6 * N_FRAMES, "launches_per_call": 3,
                 "kernel_ms_per_call": gprof[0] / max(1, gprof[1]) * 3, "pcg_iterations": float(st[2]),
                 "pcg_rel_residual": float(st[3]), "energy_feat": float(st[0]), "energy_dense": float(st[1]),
                 "bound": "latency (96 x 96 fp64 system; single-CTA PCG)",
                 "jacobi": {"ms_per_call": j0.elapsed_time(j1) / 10, "pcg_iterations": float(jac[2]),
                            "pcg_rel_residual": float(jac[3])},
                 "gn_iteration_ms": n0.elapsed_time(n1) / gn_reps,
                 "gn_iteration": "bt_relinearize (Eq. (2) from cached C_ij + 240 dense edges re-associated) + "
                                 "bt_pose_graph_step, L2 warm"}

    # ---- NEXT-4: normal maps from depth for the 16 frames (bt_estimate_normals) ----------
    # algorithmic bytes 4 (depth read) + 12 (normal written) per pixel; before each call,
    # outside its events, L2 is flushed AND cleaned (a 256 MiB read after the memset), so the
    # kernel does not pay for writing back the flush's dirty lines
    prep = None
    if world == 1:
        nrm_out = torch.empty((N_FRAMES, H, W, 3), dtype=torch.float32, device=dev)
        clean = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
        for _ in range(3):
            ctx.estimate_normals(fb.depth, sc.K, nrm_out, stream=stream)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for a_, b_ in ev:
            flush.zero_()
            clean.sum()
            a_.record(stream)
            ctx.estimate_normals(fb.depth, sc.K, nrm_out, stream=stream)
            b_.record(stream)
        torch.cuda.synchronize()
        t_ms = float(np.median([a_.elapsed_time(b_) for a_, b_ in ev]))
        nbytes = N_FRAMES * H * W * 16
        prep = {"api": "bt_estimate_normals", "frames": N_FRAMES, "width": W, "height": H,
                "ms_per_call": t_ms, "bound": "hbm", "bytes_per_call": nbytes,
                "achieved_gbs": nbytes / (t_ms * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                "frac": nbytes / (t_ms * 1e-3) / 1e9 / hbm_peak, "l2": "flushed + cleaned before each call"}
        # keypoint lifting (bt_lift_keypoints): the detector's 2-D keypoints (each keypoint's
        # projection, sub-pixel) + descriptors + the maps -> the registration inputs
        p_ = sc.pts.astype(np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            uv_ = np.stack([sc.K.fx * p_[..., 0] / p_[..., 2] + sc.K.cx, sc.K.fy * p_[..., 1] / p_[..., 2] + sc.K.cy], -1)
        uv_t = torch.from_numpy(np.nan_to_num(uv_, nan=-10.0).astype(np.float32)).to(dev)
        lo_ = bt.FrameBatch(torch.zeros_like(fb.n_kp), torch.empty_like(fb.desc), torch.empty_like(fb.pts),
                            torch.empty_like(fb.nrm))
        for _ in range(3):
            ctx.lift_keypoints(uv_t, fb.desc, fb.n_kp, fb, sc.K, lo_, stream=stream)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for a_, b_ in ev:
            flush.zero_()
            clean.sum()
            a_.record(stream)
            ctx.lift_keypoints(uv_t, fb.desc, fb.n_kp, fb, sc.K, lo_, stream=stream)
            b_.record(stream)
        torch.cuda.synchronize()
        l_ms = float(np.median([a_.elapsed_time(b_) for a_, b_ in ev]))
        nk = int(sc.n_kp.sum())
        lbytes = nk * (8 + 512 + 512 + 24 + 17)
        prep["lift"] = {"api": "bt_lift_keypoints", "keypoints": nk, "kept": int(lo_.n_kp.sum().item()),
                        "ms_per_call": l_ms, "bound": "latency (one CTA per frame; ~9 MB)",
                        "bytes_per_call": lbytes, "achieved_gbs": lbytes / (l_ms * 1e-3) / 1e9}
        del clean

    # ---- the sharded multi-track / stress configurations ---------------------
    c4 = None if args.no_c4 else multi_block("c4", args, bt, parallel, torch, dist, world, rank, local, dev, flush)
    c5 = multi_block("c5", args, bt, parallel, torch, dist, world, rank, local, dev, flush) if args.c5 else None

    # ---- end to end through the C ABI with pinned HOST buffers -------------------------
    # Primary: bt_register_raw_host from the RAW per-frame inputs — depth, mask and the keypoint
    # detector's output (2-D pixels + descriptors); normals and the keypoints' 3-D points are
    # derived on the device (NEXT-4), so only those bytes cross PCIe.  Also the older entry
    # bt_register_pairs_host with precomputed normal maps and 3-D keypoints (e2e_precomputed_maps).
    e2e = None
    e2e_blocking = None
    e2e_u16 = None
    e2e_pre = None
    if not args.no_e2e:
        def warm(fn):
            # untimed calls for >= e2e_warmup_s (and >= 3): pinned-host -> device copies run at
            # a fraction of the link's rate for the first ~second of traffic
            # (a fixed count under torchrun: the blocking step holds a collective, so every rank
            # must make the same number of calls)
            t0, k = time.time(), 0
            while k < 3 or (time.time() - t0 < args.e2e_warmup_s if world == 1 else k < 200):
                fn(k)
                k += 1
                if k % 8 == 0:
                    torch.cuda.synchronize()
            torch.cuda.synchronize()

        def timed(step, n):
            warm(lambda k: step())
            e_s = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
            e_e = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            for k in range(n):
                e_s[k].record(stream)
                step()
                e_e[k].record(stream)
            torch.cuda.synchronize()
            e_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in zip(e_s, e_e))], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
            return world * P * n / (float(e_ms.item()) / 1e3)

        h_pairs = torch.from_numpy(pairs).pin_memory()
        h_uid = torch.from_numpy(uids.view(np.int32)).pin_memory()
        h_pose = torch.from_numpy(poses).pin_memory()
        h_rec = torch.zeros((P, rw), dtype=torch.int32).pin_memory()
        small = sum(x.numel() * x.element_size() for x in (h_pairs, h_uid, h_pose))
        d2h = h_rec.numel() * 4
        xh2d, xd2h = (h_rec.numel() * 4, world * h_rec.numel() * 4) if world > 1 else (0, 0)

        def exchange_host():
            if world > 1:                                # records back to HBM for the exchange
                g = parallel.all_gather_records(h_rec.to(dev, non_blocking=True), world * P)
                g.cpu()
        # raw inputs: the detector's output = each keypoint's projection (sub-pixel) + descriptor
        Kc = sc.K
        uv = np.zeros(sc.desc.shape[:2] + (2,), np.float32)
        for f in range(sc.desc.shape[0]):
            n_ = int(sc.n_kp[f])
            p_ = sc.pts[f, :n_].astype(np.float64)
            uv[f, :n_, 0] = Kc.fx * p_[:, 0] / p_[:, 2] + Kc.cx
            uv[f, :n_, 1] = Kc.fy * p_[:, 1] / p_[:, 2] + Kc.cy
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        h_depth, h_mask, h_uv, h_desc, h_nin = pin(sc.depth), pin(sc.mask), pin(uv), pin(sc.desc), pin(sc.n_kp)
        h2d_raw = small + sum(x.numel() * x.element_size() for x in (h_depth, h_mask, h_uv, h_desc, h_nin))

        def raw_step():
            ctx.register_raw(h_depth, h_mask, h_uv, h_desc, h_nin, sc.K, h_pose, h_pairs, h_uid, rprm, eprm, h_rec,
                             stream=stream)
            exchange_host()
        v_raw = timed(raw_step, args.e2e_steps)
        d_raw = bt.decode_records(h_rec, N_MAX)
        e2e_blocking = {"value": v_raw, "unit": UNIT, "h2d_bytes_per_step": int(h2d_raw + xh2d),
                        "d2h_bytes_per_step": int(d2h + xd2h),
                        "api": "bt_register_raw_host: pinned host depth, mask, 2-D keypoints + descriptors in, "
                               "records out (normal map and keypoint lifting on the device; copies + sync inside "
                               "the call)", "pairs_ok": int((d_raw["status"] == 0).sum())}
        e2e = e2e_blocking
        if world == 1:
            # the streaming form: bt_register_raw_host_async per step (each step still copies its
            # inputs in and its records out), one synchronisation at the end — the copies of step
            # t + 1 run on the copy engine while the kernels of step t run.  One event pair on the
            # caller's stream around the K calls (the device is idle when the first is recorded,
            # so no copy of the first call can precede it).
            h_recs = [torch.zeros_like(h_rec).pin_memory() for _ in range(2)]

            def raw_async(k):
                ctx.register_raw(h_depth, h_mask, h_uv, h_desc, h_nin, sc.K, h_pose, h_pairs, h_uid, rprm, eprm,
                                 h_recs[k & 1], stream=stream, blocking=False)
            warm(raw_async)
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record(stream)
            for k in range(args.e2e_steps):
                raw_async(k)
            eb.record(stream)
            torch.cuda.synchronize()
            v_pipe = P * args.e2e_steps / (ea.elapsed_time(eb) / 1e3)
            assert all(np.array_equal(r.numpy(), h_rec.numpy()) for r in h_recs), "async records differ"
            e2e = {"value": v_pipe, "unit": UNIT, "h2d_bytes_per_step": int(h2d_raw), "d2h_bytes_per_step": int(d2h),
                   "api": "bt_register_raw_host_async per step: pinned host depth, mask, 2-D keypoints + "
                          "descriptors in, records out to pinned host memory (normal map and keypoint lifting on "
                          "the device); two staging slots, so the host->device copies of step t + 1 overlap the "
                          "kernels of step t; one synchronisation after the K steps",
                   "pairs_ok": int((d_raw["status"] == 0).sum()), "blocking_value": v_raw}
            # the same streaming entry with the depth maps as the sensor / the paper's datasets
            # store them: uint16 millimetres (half the depth bytes over PCIe).  The workload is
            # the C2 scene with its depth quantised to 1 mm; its records are checked against the
            # blocking f32 call on the same (dequantised) values.
            d_mm = np.where(sc.depth > 0, np.rint(sc.depth * 1000.0), 0).clip(0, 65535).astype(np.uint16)
            h_dmm = pin(d_mm)
            h_rq = torch.zeros_like(h_rec).pin_memory()
            ctx.register_raw(pin(d_mm.astype(np.float32) * np.float32(1e-3)), h_mask, h_uv, h_desc, h_nin, sc.K,
                             h_pose, h_pairs, h_uid, rprm, eprm, h_rq, stream=stream)

            def raw_u16(k):
                ctx.register_raw(h_dmm, h_mask, h_uv, h_desc, h_nin, sc.K, h_pose, h_pairs, h_uid, rprm, eprm,
                                 h_recs[k & 1], stream=stream, blocking=False, depth_scale=1e-3)
            warm(raw_u16)
            ea.record(stream)
            for k in range(args.e2e_steps):
                raw_u16(k)
            eb.record(stream)
            torch.cuda.synchronize()
            assert all(np.array_equal(r.numpy(), h_rq.numpy()) for r in h_recs), "u16 depth records differ"
            h2d_u16 = h2d_raw - h_depth.numel() * 4 + h_dmm.numel() * 2
            e2e_u16 = {"value": P * args.e2e_steps / (ea.elapsed_time(eb) / 1e3), "unit": UNIT,
                       "h2d_bytes_per_step": int(h2d_u16), "d2h_bytes_per_step": int(d2h),
                       "api": "bt_register_raw_host_async with uint16 depth (mm, depth_scale 1e-3) instead of "
                              "f32 metres; otherwise as e2e",
                       "pairs_ok": int((bt.decode_records(h_rq, N_MAX)["status"] == 0).sum())}
            # ... and the mask as packed bits (LSB first, unpacked on the device): the sensor /
            # segmentation formats, 1 + 2 bytes per pixel become 1/8 + 2
            h_bits = pin(np.packbits(sc.mask != 0, axis=-1, bitorder="little"))

            def raw_compact(k):
                ctx.register_raw(h_dmm, h_bits, h_uv, h_desc, h_nin, sc.K, h_pose, h_pairs, h_uid, rprm, eprm,
                                 h_recs[k & 1], stream=stream, blocking=False, depth_scale=1e-3, mask_bits=True)
            warm(raw_compact)
            ea.record(stream)
            for k in range(args.e2e_steps):
                raw_compact(k)
            eb.record(stream)
            torch.cuda.synchronize()
            assert all(np.array_equal(r.numpy(), h_rq.numpy()) for r in h_recs), "packed-mask records differ"
            h2d_c = h2d_u16 - h_mask.numel() + h_bits.numel()
            e2e_u16["compact_mask_bits"] = {
                "value": P * args.e2e_steps / (ea.elapsed_time(eb) / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(h2d_c), "d2h_bytes_per_step": int(d2h),
                "api": "as e2e_depth_u16 with the mask as packed bits (mask_bits)"}
        hb = bt.FrameBatch.from_scene(sc, device="cpu", pin=True)
        h2d_pre = small + sum(x.numel() * x.element_size() for x in (hb.n_kp, hb.desc, hb.pts, hb.nrm, hb.depth,
                                                                   hb.normal, hb.mask))

        def pre_step():
            ctx.register_pairs(hb, sc.K, h_pose, h_pairs, h_uid, rprm, eprm, h_rec, stream=stream, host=True)
            exchange_host()
        v_pre = timed(pre_step, args.e2e_steps)
        e2e_pre = {"value": v_pre, "unit": UNIT, "h2d_bytes_per_step": int(h2d_pre + xh2d),
                   "d2h_bytes_per_step": int(d2h + xd2h),
                   "api": "bt_register_pairs_host (precomputed normal maps and 3-D keypoints; pinned host buffers)"}
        assert np.array_equal(h_rec.numpy(), rec.cpu().numpy()), "host-buffer path disagrees with device path"

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = list(range(0, P, 1))
        v, dt = oracle_pairs_per_s(sc, pairs, uids, poses, sample)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu": cpu_model(),
               "sample": f"the full C2 step ({len(sample)} pairs: matching, {N_HYP}-hypothesis RANSAC, refit, "
                         f"Eq.(2) blocks, 240 dense edges), single-threaded C fp64, {dt:.1f} s"}
        try:
            va, cores, dta = oracle_all_cores(sc, pairs, uids, poses, sample)
            cpu["all_cores"] = {"value": va, "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": f"the full C2 step x 3, one process per core, pairs handed out one at a "
                                          f"time (the per-pair oracle unchanged), {dta:.1f} s"}
        except Exception as e:                         # pragma: no cover (host without fork)
            cpu["all_cores"] = {"unavailable": str(e)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded analytic ellipsoid scene, synth/)", "config": config_block(),
                "hypotheses_per_s": hyp_per_s, "tests_per_s": world * tests * args.steps / sec,
                "ms_per_step_instrumented": ms_i / args.steps,
                "launch": "CUDA graph replay of bt_register_pairs" if graph_exec is not None else "eager launches",
                "kernel_timing": "per-kernel CUDA-event brackets on each kernel's stream, over a second timed "
                                 "region of the same K steps (the headline region runs uninstrumented)",
                "parallelism": f"dp{world} (one track per rank, records all-gathered over NCCL)" if world > 1
                else "single GPU",
                "clocks": clk.summary(), "gpu_launches": launches_per_step * args.steps,
                "roofline": roof, "kernels": kern, "kernel_ms_per_step": step_ms_by_kernel,
                "e2e": e2e, "e2e_blocking": e2e_blocking, "e2e_depth_u16": e2e_u16, "e2e_precomputed_maps": e2e_pre, "cpu_baseline": cpu, "next_pose_graph": graph,
                "next_input_prep": prep, "c4": c4, "c5": c5}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
