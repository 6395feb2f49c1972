"""Diagnostics of the causal tracker: per frame the coarse-pose error, the error after the
pose graph, the pool size and selection, the status / inlier counts of the graph's pairs, for a
few Gauss-Newton settings.  Writes gpurun_out/track_diag.json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2108_00516_b200 as bt  # noqa: E402
from paper_2108_00516_b200 import tracker  # noqa: E402

F = int(sys.argv[1]) if len(sys.argv) > 1 else 60
scene, gt = tracker.orbit_scene(views=180, point_noise=0.0005)
order = list(range(F))
res = {}
for G in (0, 2, 6):
    tr = tracker.Tracker(scene.K, n_max=512, n_hyp=4096, gn_iters=G, log=True)
    out = tr.run(scene, order, T0=gt[0])
    rot, trans = tracker.pose_errors(out["poses"], [gt[v] for v in order])
    crot, ctrans = tracker.pose_errors(np.stack([fr["coarse"] for fr in out["log"]]), [gt[v] for v in order])
    d = bt.decode_records(tr.rec_g, 512)
    res[f"G{G}"] = {"rot": rot.tolist(), "trans_mm": (1e3 * trans).tolist(), "coarse_rot": crot.tolist(),
                    "coarse_mm": (1e3 * ctrans).tolist(), "sel": [fr["sel"] for fr in out["log"]],
                    "pool": out["pool_size"], "last_status": d["status"].tolist(),
                    "last_count": d["best_count"].tolist(), "last_dense_count": d["dense_ij"][:, 28].tolist()}
    tr.close()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/track_diag.json", "w"))
print("ok")
