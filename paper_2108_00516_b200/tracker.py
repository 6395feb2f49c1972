"""NEXT-2: the causal tracker loop of BundleTrack (§IV, P:4) on the GPU, orchestrated
on the host from the C-ABI calls (stream-ordered; the per-frame decisions run in the library's
kernels):

  1. coarse pose (§IV-B): register the consecutive pair (t-1, t) (bt_register_pairs without
     dense edges) and T~_t = T_rel . T_{t-1} (bt_coarse_pose, reading R13);
  2. keyframe selection (§IV-C): greedy K = 15 from the memory pool on the ESTIMATED pool
     poses and T~_t (bt_select_keyframes; the pool lives on the device);
  3. pose graph (§IV-D): nodes = the current frame + the selected keyframes in 16 frame
     slots; current x keyframe pairs registered (bt_register_pairs), keyframe pairs' C_ij reused
     from a cache when built in an earlier frame and re-linearized at the current poses
     (bt_relinearize_matches), G Gauss-Newton steps with I_0's node fixed (bt_pose_graph_step);
  4. output T_t (causal) and refresh the selected keyframes' pool poses from the optimized graph
     (P:85); pool augmentation by the 10 degree novelty rule on T_t (bt_pool_admit).

One host synchronisation per frame: the selection (a few ints) is read back to plan which pool
frames occupy the slots and which keyframe pairs are new.  `log=True` adds reads of the pool /
coarse / final poses for the tests (stage isolation of each decision).
"""
from __future__ import annotations

import numpy as np

from . import FrameBatch, Context, edge_params, ransac_params, record_words

FIELDS = ("n_kp", "desc", "pts", "nrm", "depth", "normal", "mask")
PHILOX_SEED = 0x0123456789ABCDEF


class Tracker:
    def __init__(self, K, n_max: int = 512, n_hyp: int = 4096, kf: int = 15, gn_iters: int = 2,
                 pool_cap: int = 96, cache_cap: int = 2048, novelty_deg: float = 10.0, device: int = 0,
                 log: bool = False, seed: int = PHILOX_SEED, min_inliers: int = 20, dense_gate_m: float = 0.005):
        import torch
        self.torch = torch
        self.K, self.n_max, self.kf, self.G = K, n_max, kf, gn_iters
        self.NS = kf + 1                      # graph slots: 0 = current frame, 1..kf = keyframes
        self.PREV = self.NS                   # slot NS: the previous frame (consecutive pair)
        self.dev = torch.device("cuda", device)
        self.ctx = Context(device)
        self.pool_cap, self.cache_cap = pool_cap, cache_cap
        self.thresh = float(np.deg2rad(novelty_deg))
        self.log_on = log
        W, H = int(K.width), int(K.height)
        maxp = max(self.NS * (self.NS - 1) // 2, 1)
        self.ctx.reserve(maxp, n_max, n_hyp, self.NS + 1, W, H)
        # a pair with fewer inliers is a failed registration (status FEW_INLIERS): the graph then
        # drops its Eq. (2) term (reading R30) and the coarse pose keeps T_{t-1}
        # dense association gate 5 mm (reading R31: the paper's only stated distance threshold, delta
        # of P:25): the 2 cm gate of R15 lets occlusion-boundary pixels associate, which biases the
        # converged relative pose of two views 20 deg apart by ~0.46 deg (5 mm: 0.02 deg)
        self.rprm = ransac_params(n_hyp, seed, min_inliers=min_inliers)
        self.eprm = edge_params(dist_gate_m=dense_gate_m)
        self.rw = record_words(n_max)
        dev = self.dev

        def buf(n, field_shape, dtype):
            return torch.zeros((n,) + field_shape, dtype=dtype, device=dev)
        shapes = {"n_kp": ((), torch.int32), "desc": ((n_max, 128), torch.float32),
                  "pts": ((n_max, 3), torch.float32), "nrm": ((n_max, 3), torch.float32),
                  "depth": ((H, W), torch.float32), "normal": ((H, W, 3), torch.float32),
                  "mask": ((H, W), torch.uint8)}
        self.slots = {f: buf(self.NS + 1, *shapes[f]) for f in FIELDS}
        self.store = {f: buf(pool_cap, *shapes[f]) for f in FIELDS}        # keyframe memory pool
        self.fb = FrameBatch(*(self.slots[f] for f in FIELDS))
        self.pose_s = torch.zeros((self.NS + 1, 12), dtype=torch.float32, device=dev)
        self.new_pose = torch.zeros((self.NS, 12), dtype=torch.float32, device=dev)
        self.odo = torch.zeros((2, 12), dtype=torch.float32, device=dev)  # frame-to-frame chain only
        self.pool_pose = torch.zeros((pool_cap, 12), dtype=torch.float32, device=dev)
        self.n_pool = torch.zeros(1, dtype=torch.int32, device=dev)
        self.sel = torch.zeros(kf, dtype=torch.int32, device=dev)
        self.n_sel = torch.zeros(1, dtype=torch.int32, device=dev)
        self.admitted = torch.full((1,), -1, dtype=torch.int32, device=dev)
        self.rec_prev = torch.zeros((1, self.rw), dtype=torch.int32, device=dev)
        self.rec_cur = torch.zeros((kf, self.rw), dtype=torch.int32, device=dev)
        self.mt_cur = torch.zeros((kf, n_max, 2), dtype=torch.int32, device=dev)
        self.nm_cur = torch.zeros(kf, dtype=torch.int32, device=dev)
        self.rec_cache = torch.zeros((cache_cap, self.rw), dtype=torch.int32, device=dev)
        self.mt_cache = torch.zeros((cache_cap, n_max, 2), dtype=torch.int32, device=dev)
        self.nm_cache = torch.zeros(cache_cap, dtype=torch.int32, device=dev)
        self.rec_g = torch.zeros((maxp, self.rw), dtype=torch.int32, device=dev)
        self.mt_g = torch.zeros((maxp, n_max, 2), dtype=torch.int32, device=dev)
        self.nm_g = torch.zeros(maxp, dtype=torch.int32, device=dev)
        self.rec_tmp = torch.zeros((maxp, self.rw), dtype=torch.int32, device=dev)
        self.mt_tmp = torch.zeros((maxp, n_max, 2), dtype=torch.int32, device=dev)
        self.nm_tmp = torch.zeros(maxp, dtype=torch.int32, device=dev)
        self.slot_pool = [None] * self.NS         # pool id held by each keyframe slot
        self.cache = {}                           # (pool a, pool b) in registration order -> cache row
        self.uid = 0
        self.t = 0
        self.prev_sel = []                        # pool ids of the previous frame's current pairs
        self.log = []

    # ------------------------------------------------------------------ helpers
    def _uids(self, n):
        u = self.torch.arange(self.uid, self.uid + n, dtype=self.torch.int32, device=self.dev)
        self.uid += n
        return u

    def _copy_frame(self, dst, i, src, j):
        for f in FIELDS:
            dst[f][i].copy_(src[f][j])

    def _register(self, pairs, rec, mt, nm, dense=True):
        tp = self.torch.tensor(pairs, dtype=self.torch.int32, device=self.dev).reshape(-1, 2)
        n = tp.shape[0]
        self.ctx.register_pairs(self.fb, self.K, self.pose_s, tp, self._uids(n), self.rprm,
                                self.eprm if dense else None, rec[:n])
        if mt is not None:
            self.ctx.copy_matches(mt[:n], nm[:n])

    def _cache_put(self, key, rec_row, mt_row, nm_row):
        if key in self.cache:
            return
        r = len(self.cache)
        if r >= self.cache_cap:
            raise RuntimeError("keyframe-pair cache full")
        self.cache[key] = r
        self.rec_cache[r].copy_(rec_row)
        self.mt_cache[r].copy_(mt_row)
        self.nm_cache[r].copy_(nm_row)

    def _snap(self, x):
        return x.detach().cpu().numpy().copy()

    # ------------------------------------------------------------------ one frame
    def step(self, frame: dict, j: int, T0=None):
        """Track one frame: `frame` = dict of device tensors [V][...] (the FIELDS), j = its index
        there.  Returns nothing; the output pose is self.pose_s[0] (device)."""
        torch = self.torch
        self._copy_frame(self.slots, 0, frame, j)
        rec = {}
        if self.t == 0:                                           # I_0: pose given, first keyframe
            self.pose_s[0].copy_(torch.as_tensor(np.asarray(T0, np.float32), device=self.dev))
            self.odo[1].copy_(self.pose_s[0])
            if self.log_on:
                rec.update(pool=[], coarse=self._snap(self.pose_s[0]), sel=[])
            self.ctx.pool_admit(self.pool_pose, self.n_pool, self.pose_s[0], self.thresh, self.admitted)
            self._copy_frame(self.store, 0, self.slots, 0)
            self.prev_sel = []
            if self.log_on:
                rec.update(pose=self._snap(self.pose_s[0]), pool_after_refresh=[], admitted=True)
        else:
            # 1. coarse pose from the consecutive pair
            self._register([[self.PREV, 0]], self.rec_prev, None, None, dense=False)
            self.ctx.coarse_pose(self.rec_prev[0], self.pose_s[self.PREV], self.pose_s[0])
            self.ctx.coarse_pose(self.rec_prev[0], self.odo[1], self.odo[0])
            self.odo[1].copy_(self.odo[0])
            # 2. keyframe selection on the estimated poses
            self.ctx.select_keyframes(self.pool_pose, self.n_pool, self.pose_s[0], self.kf, self.sel, self.n_sel)
            if self.log_on:
                npool = int(self.n_pool.item())
                rec.update(pool=self._snap(self.pool_pose[:npool]), coarse=self._snap(self.pose_s[0]))
            hs = self._snap(torch.cat([self.sel, self.n_sel, self.admitted]))      # the one sync
            n_sel, adm_prev = int(hs[self.kf]), int(hs[self.kf + 1])
            sel = [int(x) for x in hs[:n_sel]]
            # the previous frame joined the pool: its data (still in the prev slot) to the store,
            # its current x keyframe pairs into the cache
            if adm_prev >= 0:
                self._copy_frame(self.store, adm_prev, self.slots, self.PREV)
                for s, pid in enumerate(self.prev_sel):
                    self._cache_put((adm_prev, pid), self.rec_cur[s], self.mt_cur[s], self.nm_cur[s])
            # 3. slots: keep held keyframes, fill the new ones from the pool store
            keep = set(sel)
            for s in range(1, self.NS):
                if self.slot_pool[s] is not None and self.slot_pool[s] not in keep:
                    self.slot_pool[s] = None
            held = {p: s for s, p in enumerate(self.slot_pool) if p is not None}
            for p in sel:
                if p not in held:
                    s = next(s for s in range(1, self.NS) if self.slot_pool[s] is None)
                    self.slot_pool[s] = p
                    held[p] = s
                    self._copy_frame(self.slots, s, self.store, p)
                    self.pose_s[s].copy_(self.pool_pose[p])
            slots = sorted(held.values())                                    # active keyframe slots
            # current x keyframe pairs (new every frame)
            self._register([[0, s] for s in slots], self.rec_cur, self.mt_cur, self.nm_cur)
            self.prev_sel = [self.slot_pool[s] for s in slots]
            # keyframe pairs: cached C_ij, or registered now (first time selected together)
            kpairs = []
            fresh = []
            for a_i, sa in enumerate(slots):
                for sb in slots[a_i + 1:]:
                    pa, pb = self.slot_pool[sa], self.slot_pool[sb]
                    if (pa, pb) in self.cache:
                        kpairs.append((sa, sb, self.cache[(pa, pb)]))
                    elif (pb, pa) in self.cache:
                        kpairs.append((sb, sa, self.cache[(pb, pa)]))
                    else:
                        fresh.append((sa, sb))
            if fresh:
                self._register(fresh, self.rec_tmp, self.mt_tmp, self.nm_tmp)
                for k, (sa, sb) in enumerate(fresh):
                    self._cache_put((self.slot_pool[sa], self.slot_pool[sb]), self.rec_tmp[k], self.mt_tmp[k],
                                    self.nm_tmp[k])
                    kpairs.append((sa, sb, self.cache[(self.slot_pool[sa], self.slot_pool[sb])]))
            # 4. the pose graph: current pairs + keyframe pairs, G Gauss-Newton steps, I_0 fixed
            nc = len(slots)
            gp = [[0, s] for s in slots] + [[a, b] for a, b, _ in kpairs]
            P = len(gp)
            t_gp = torch.tensor(gp, dtype=torch.int32, device=self.dev)
            self.rec_g[:nc].copy_(self.rec_cur[:nc])
            self.mt_g[:nc].copy_(self.mt_cur[:nc])
            self.nm_g[:nc].copy_(self.nm_cur[:nc])
            if kpairs:
                rows = torch.tensor([r for _, _, r in kpairs], dtype=torch.long, device=self.dev)
                self.rec_g[nc:P].copy_(self.rec_cache.index_select(0, rows))
                self.mt_g[nc:P].copy_(self.mt_cache.index_select(0, rows))
                self.nm_g[nc:P].copy_(self.nm_cache.index_select(0, rows))
            n_nodes = self.NS
            fixed = held[0]
            for _ in range(self.G):
                self.ctx.relinearize(self.fb, self.K, self.pose_s, t_gp, self.eprm, self.rec_g[:P],
                                     matches=self.mt_g[:P], n_matches=self.nm_g[:P])
                self.ctx.pose_graph_step(self.pose_s[:n_nodes], t_gp, self.rec_g[:P], self.n_max, self.new_pose,
                                         fixed_node=fixed)
                self.pose_s[:n_nodes].copy_(self.new_pose)
            # 5. output T_t; refresh the selected keyframes' pool poses; augment the pool
            pid = torch.tensor([self.slot_pool[s] for s in slots], dtype=torch.long, device=self.dev)
            sid = torch.tensor(slots, dtype=torch.long, device=self.dev)
            self.pool_pose.index_copy_(0, pid, self.pose_s.index_select(0, sid))
            if self.log_on:
                npool = int(self.n_pool.item())
                rec.update(sel=sel, pose=self._snap(self.pose_s[0]), pool_after_refresh=self._snap(self.pool_pose[:npool]))
            self.ctx.pool_admit(self.pool_pose, self.n_pool, self.pose_s[0], self.thresh, self.admitted)
            if self.log_on:
                rec["admitted"] = int(self.admitted.item()) >= 0
        # the current frame becomes the previous one
        self._copy_frame(self.slots, self.PREV, self.slots, 0)
        self.pose_s[self.PREV].copy_(self.pose_s[0])
        if self.log_on:
            self.log.append(rec)
        self.t += 1

    def run(self, scene, order, T0, out_poses=None):
        """Track the scene's views in `order` (resident on the device); returns dict(poses
        [F][12] tracked, odometry [F][12] frame-to-frame chain only, ms per frame, pool_size,
        log)."""
        torch = self.torch
        frames = {f: torch.from_numpy(np.ascontiguousarray(getattr(scene, f))).to(self.dev) for f in FIELDS}
        F = len(order)
        poses = torch.zeros((F, 12), dtype=torch.float32, device=self.dev)
        odo = torch.zeros((F, 12), dtype=torch.float32, device=self.dev)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(F)]
        for t, j in enumerate(order):
            ev[t][0].record()
            self.step(frames, int(j), T0=T0 if t == 0 else None)
            ev[t][1].record()
            poses[t].copy_(self.pose_s[self.PREV])
            odo[t].copy_(self.odo[1])
        torch.cuda.synchronize()
        return {"poses": poses.cpu().numpy(), "odometry": odo.cpu().numpy(),
                "ms": np.array([a.elapsed_time(b) for a, b in ev]), "pool_size": int(self.n_pool.item()),
                "log": self.log}

    def close(self):
        self.ctx.close()


# ------------------------------------------------------------------ synthetic C3 inputs / metrics
def orbit_scene(views: int = 180, deg_per_view: float = 2.0, point_noise: float = 0.0005, seed: int = 210800516):
    """ORBIT: the object turns deg_per_view about the camera's y axis per frame
    at 0.5 m; views rendered once.  Returns (scene, ground-truth poses [views][12])."""
    import synth
    R0 = synth.rotvec_to_R(np.array([0.3, -0.5, 0.2]))
    vs = [(synth.rotvec_to_R(np.array([0.0, np.deg2rad(deg_per_view * v), 0.0])) @ R0, np.array([0.0, 0.0, 0.5]))
          for v in range(views)]
    sc = synth.make_scene(views, seed=seed, poses=vs, min_geodesic_deg=0.0, point_noise=point_noise)
    return sc, sc.node_poses()


def pose_errors(poses, gt):
    """Per-frame rotation error (deg, 2 asin(|dR|_F / (2 sqrt 2))) and translation error (m)."""
    P = np.asarray(poses, np.float64).reshape(-1, 12)
    G = np.asarray(gt, np.float64).reshape(-1, 12)
    dR = np.linalg.norm(P[:, :9] - G[:, :9], axis=1)
    rot = np.rad2deg(2 * np.arcsin(np.minimum(1.0, dR / (2 * np.sqrt(2)))))
    return rot, np.linalg.norm(P[:, 9:] - G[:, 9:], axis=1)
