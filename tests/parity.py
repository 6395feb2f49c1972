"""Comparison helpers shared by the GPU parity tests: band-aware integer comparisons and the
north-star tolerances (pose 1e-4 rad / 1e-5 m, J^T J 1e-4 relative), DESIGN.md §4."""
from __future__ import annotations

import numpy as np

import oracle

POSE_ROT_TOL = 1e-4      # rad
POSE_T_TOL = 1e-5        # m
H_REL_TOL = 1e-4


def rot_angle(Ra, Rb) -> float:
    """2 asin(|Ra - Rb|_F / (2 sqrt 2)): the rotation angle between Ra and Rb, computed
    without arccos' loss of resolution near 0 (exact for rotations)."""
    d = np.linalg.norm(np.asarray(Ra, float).reshape(3, 3) - np.asarray(Rb, float).reshape(3, 3))
    return float(2 * np.arcsin(min(1.0, d / (2 * np.sqrt(2)))))


def assert_pose_close(Tg, To, what=""):
    Tg = np.asarray(Tg, float)
    To = np.asarray(To, float)
    ang = rot_angle(Tg[:9], To[:9])
    dt = float(np.linalg.norm(Tg[9:] - To[9:]))
    assert ang <= POSE_ROT_TOL and dt <= POSE_T_TOL, f"{what}: rot {ang:.3g} rad, trans {dt:.3g} m"


def assert_H_close(Hg, Ho, what=""):
    Hg = np.asarray(Hg, float)
    Ho = np.asarray(Ho, float)
    err = np.linalg.norm(Hg - Ho)
    assert err <= H_REL_TOL * np.linalg.norm(Ho) + 1e-12, f"{what}: |dH| {err:.3g} vs |H| {np.linalg.norm(Ho):.3g}"


def assert_g_close(gg, go, scale, what=""):
    gg, go, scale = (np.asarray(x, float) for x in (gg, go, scale))
    bad = np.abs(gg - go) > H_REL_TOL * scale + 1e-9
    assert not bad.any(), f"{what}: g {gg[bad]} vs {go[bad]} (scale {scale[bad]})"


def assert_dense_close(g32, o48, what=""):
    """GPU dense row (32 f32) vs oracle row (48 f64): count within the borderline pixels;
    H and E within 1e-4 relative, g within 1e-4 of sum w|J_k r| — each plus the oracle's
    allowance for the borderline pixels (the largest contribution they can make)."""
    g32 = np.asarray(g32, float)
    o = np.asarray(o48, float)
    count_g, count_o, border = g32[28], o[28], o[29]
    assert abs(count_g - count_o) <= border, f"{what}: count {count_g} vs {count_o} (+-{border})"
    dH = np.linalg.norm(_sym(g32[:21]) - _sym(o[:21]))
    assert dH <= H_REL_TOL * np.linalg.norm(_sym(o[:21])) + o[45] + 1e-12, f"{what}: |dH| {dH:.3g}"
    gg, go = g32[21:27], o[21:27]
    bad = np.abs(gg - go) > H_REL_TOL * o[32:38] + o[38:44] + 1e-9
    assert not bad.any(), f"{what}: g {gg[bad]} vs {go[bad]} (scale {o[32:38][bad]}, allowance {o[38:44][bad]})"
    assert abs(g32[27] - o[27]) <= H_REL_TOL * abs(o[27]) + o[44] + 1e-12, f"{what}: E {g32[27]} vs {o[27]}"


def _sym(v21):
    H = np.zeros((6, 6))
    k = 0
    for a in range(6):
        for b in range(a, 6):
            H[a, b] = H[b, a] = v21[k]
            k += 1
    return H


def assert_feat_close(g96, o108, what=""):
    g96 = np.asarray(g96, float)
    assert_H_close(g96[:78], o108[:78], what + " H")
    assert_g_close(g96[78:90], o108[78:90], o108[96:108], what + " g")
    assert abs(g96[90] - o108[90]) <= H_REL_TOL * abs(o108[90]) + 1e-12, f"{what}: E {g96[90]} vs {o108[90]}"


def mask_bits(words, M):
    w = np.asarray(words, np.uint32)
    return np.array([(int(w[m // 32]) >> (m % 32)) & 1 for m in range(M)], bool)


def compare_matches(gpu_pairs, orc):
    """Mutual-NN match lists: identical outside rows / columns whose NN is ambiguous within
    the band.  Returns the number of excluded entries."""
    rb = np.nonzero(orc["row_border"])[0]
    cb = np.nonzero(orc["col_border"])[0]
    g = {tuple(x) for x in np.asarray(gpu_pairs).tolist()}
    o = {tuple(x) for x in orc["pairs"].tolist()}
    if len(rb) == 0 and len(cb) == 0:
        assert np.array_equal(np.asarray(gpu_pairs), orc["pairs"]), "match lists differ"
        return 0
    keep = lambda s: {(i, j) for i, j in s if i not in set(rb) and j not in set(cb)}
    assert keep(g) == keep(o), "match sets differ outside the borderline rows/columns"
    return len(g ^ o)


def ambiguous_best(cnt, lo, hi):
    """True iff another hypothesis' count interval can reach the oracle's best."""
    hs = int(np.argmax(cnt))
    for h in range(len(cnt)):
        if h == hs:
            continue
        if hi[h] > lo[hs] or (hi[h] == lo[hs] and h < hs):
            return True
    return False


def compare_ransac(gpu_counts, rec, orc_counts, pa, na, pb, nb, what=""):
    """Per-hypothesis counts inside the oracle's band interval; h*, count*, mask and T_best
    exact / within tolerance whenever the best is unambiguous."""
    cnt, lo, hi = orc_counts["cnt"], orc_counts["lo"], orc_counts["hi"]
    if gpu_counts is not None:
        g = np.asarray(gpu_counts)
        bad = (g < lo) | (g > hi)
        assert not bad.any(), f"{what}: counts outside band at h={np.nonzero(bad)[0][:8]} gpu={g[bad][:8]} lo={lo[bad][:8]} hi={hi[bad][:8]}"
    M = len(pa)
    fin = oracle.ransac_finish(pa, na, pb, nb, orc_counts)
    assert rec["n_matches"] == M
    if M < 3:
        assert rec["status"] == oracle.STATUS_FEW_MATCHES
        return fin
    if ambiguous_best(cnt, lo, hi):
        return None
    assert rec["best_hyp"] == fin["best_hyp"], f"{what}: h* {rec['best_hyp']} vs {fin['best_hyp']}"
    if fin["best_hyp"] < 0:
        assert rec["status"] == fin["status"]
        return fin
    assert rec["best_count"] == fin["best_count"] or lo[fin["best_hyp"]] <= rec["best_count"] <= hi[fin["best_hyp"]]
    assert_pose_close(rec["T_best"], fin["T_best"], what + " T_best")
    n, mo, border = oracle.inliers(fin["T_best"], pa, na, pb, nb)
    mg = mask_bits(rec["mask"], M)
    mo_b = mask_bits(mo, M)
    diff = (mg != mo_b) & ~border
    assert not diff.any(), f"{what}: inlier mask differs at {np.nonzero(diff)[0][:8]}"
    if rec["status"] == oracle.STATUS_OK and fin["status"] == oracle.STATUS_OK:
        if np.array_equal(mg, mo_b):
            assert_pose_close(rec["T_refit"], fin["T_refit"], what + " T_refit")
        else:      # stage isolation: refit the GPU's own inlier set in the oracle
            R, t, _ = oracle.arun(pa[mg], pb[mg])
            assert_pose_close(rec["T_refit"], np.concatenate([R.reshape(9), t]), what + " T_refit(gpu mask)")
    else:
        assert rec["status"] == fin["status"], f"{what}: status {rec['status']} vs {fin['status']}"
    return fin


# ------------------------------------------------- decision-level dense / feature parity
def dense_decisions(g32, assoc, o72, pix, border, allow, what=""):
    """Eq. (3) edge compared DECISION by decision, then element by element.

    assoc [H][W]: the GPU's association (bt_dense_assoc: target pixel index or -1); pix /
    border / allow: the oracle's (bto_dense_edge pix_out / pix_border / pix_allow).
    * every source pixel outside the band (reading R22) takes the oracle's decision, bit-exact:
      same target pixel, or rejected on both sides;
    * count = the number of associated pixels, exactly;
    * H element-wise within 1e-4 of the oracle's sum of absolute contributions
      sum w |J_a J_b| (out[48..68]: the magnitude fp summation error is relative to; on the
      diagonal it IS |H_aa|), g within 1e-4 of sum w |J_k r|, E within 1e-4 relative — plus,
      only for the borderline pixels whose decision actually differs, twice the largest
      contribution they can make (pix_allow; both sides may associate them, to different
      neighbours).
    Returns (pixels differing, max relative H error)."""
    g = np.asarray(g32, float)
    o = np.asarray(o72, float)
    assoc = np.asarray(assoc)
    pix = np.asarray(pix)
    diff = assoc != pix
    out_band = diff & ~border
    assert not out_band.any(), (f"{what}: {int(out_band.sum())} pixel decisions differ outside the band, e.g. "
                                f"{[(int(v), int(u), int(assoc[v, u]), int(pix[v, u])) for v, u in np.argwhere(out_band)[:5]]}")
    assert g[28] == float((assoc >= 0).sum()), f"{what}: count {g[28]} vs {(assoc >= 0).sum()} associated pixels"
    assert o[28] == float((pix >= 0).sum())
    fl = 2.0 * allow[diff].sum(axis=0) if diff.any() else np.zeros(8)
    dH = np.abs(g[:21] - o[:21])
    tolH = H_REL_TOL * o[48:69] + fl[0] + 1e-12
    bad = dH > tolH
    assert not bad.any(), f"{what}: H[{np.nonzero(bad)[0]}] |dH| {dH[bad]} > tol {tolH[bad]}"
    dg = np.abs(g[21:27] - o[21:27])
    tolg = H_REL_TOL * o[32:38] + fl[2:8] + 1e-12
    bad = dg > tolg
    assert not bad.any(), f"{what}: g[{np.nonzero(bad)[0]}] |dg| {dg[bad]} > tol {tolg[bad]}"
    assert abs(g[27] - o[27]) <= H_REL_TOL * abs(o[27]) + fl[1] + 1e-12, f"{what}: E {g[27]} vs {o[27]}"
    rel = float((dH / np.maximum(o[48:69], 1e-300)).max()) if o[28] > 0 else 0.0
    return int(diff.sum()), rel


def feat_elementwise(g96, o186, what=""):
    """Eq. (2) blocks element by element against the oracle evaluated on the SAME inlier
    set: H_ii / H_ij / H_jj within 1e-4 of the oracle's sum w |J_ra J_rb| (out[108..185]), g within
    1e-4 of sum w |J_k| |e| (out[96..107]), E within 1e-4 relative, count exact.  Returns the max
    relative H error."""
    g = np.asarray(g96, float)
    o = np.asarray(o186, float)
    assert g[91] == o[91], f"{what}: count {g[91]} vs {o[91]}"
    dH = np.abs(g[:78] - o[:78])
    tol = H_REL_TOL * o[108:186] + 1e-12
    bad = dH > tol
    assert not bad.any(), f"{what}: H[{np.nonzero(bad)[0][:8]}] |dH| {dH[bad][:8]} > tol {tol[bad][:8]}"
    dg = np.abs(g[78:90] - o[78:90])
    bad = dg > H_REL_TOL * o[96:108] + 1e-12
    assert not bad.any(), f"{what}: g {g[78:90][bad]} vs {o[78:90][bad]}"
    assert abs(g[90] - o[90]) <= H_REL_TOL * abs(o[90]) + 1e-12, f"{what}: E {g[90]} vs {o[90]}"
    return float((dH / np.maximum(o[108:186], 1e-300)).max())
