"""GPU parity of NEXT-1, the pose-graph Gauss-Newton step (bt_pose_graph_step, PAPER.md
P:76-83), through the C ABI.  Parity: the blocks come from the ORACLE (feature / dense edges
at perturbed poses), rounded to float32 exactly as a record stores them, and both sides solve
the same system — the GPU by Jacobi-PCG, the oracle by Cholesky.  At the C2 size (no oracle):
the fixed node stays put, results are bitwise reproducible, and re-registering at the new
poses lowers the Eq. (1) energy."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bt():
    import paper_2108_00516_b200 as m
    return m


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def records_from_blocks(bt, n_max, feat, dij, dji):
    """Host records [P][record_words] with the Eq. (2) / Eq. (3) words filled (float32)."""
    P = len(feat)
    rw = bt.record_words(n_max)
    rec = np.zeros((P, rw), np.uint32)
    mw = (n_max + 31) // 32
    o_ij = 28 + mw
    f = rec.view(np.float32)
    f[:, o_ij:o_ij + 32] = np.asarray(dij, np.float32)[:, :32]
    f[:, o_ij + 32:o_ij + 64] = np.asarray(dji, np.float32)[:, :32]
    f[:, o_ij + 64:o_ij + 160] = np.asarray(feat, np.float32)[:, :96]
    return rec


def oracle_blocks(sc, poses, pairs):
    feat, dij, dji = [], [], []
    for a, b in pairs:
        ids_a = {int(i): k for k, i in enumerate(sc.kp_pool[a][:sc.n_kp[a]])}
        pa, pb = [], []
        for k, i in enumerate(sc.kp_pool[b][:sc.n_kp[b]]):
            if int(i) in ids_a:
                pa.append(sc.pts[a][ids_a[int(i)]])
                pb.append(sc.pts[b][k])
        pa, pb = np.array(pa, np.float32), np.array(pb, np.float32)
        M = len(pa)
        mk = np.full((M + 31) // 32, 0xFFFFFFFF, np.uint32)
        if M % 32:
            mk[-1] = (1 << (M % 32)) - 1
        feat.append(oracle.feature_edge(pa, pb, mk, poses[a], poses[b])[:96])
        dij.append(oracle.dense_edge(sc.depth[a], sc.normal[a], sc.mask[a], sc.depth[b], sc.normal[b], sc.mask[b],
                                     sc.K, poses[a], poses[b])[:32])
        dji.append(oracle.dense_edge(sc.depth[b], sc.normal[b], sc.mask[b], sc.depth[a], sc.normal[a], sc.mask[a],
                                     sc.K, poses[b], poses[a])[:32])
    return np.stack(feat), np.stack(dij), np.stack(dji)


def gpu_step(bt, torch, ctx, poses, pairs, rec_host, n_max, **kw):
    dev = "cuda"
    P_ = torch.from_numpy(np.ascontiguousarray(poses, np.float32)).to(dev)
    pr = torch.from_numpy(np.ascontiguousarray(pairs, np.int32)).to(dev)
    rec = torch.from_numpy(rec_host.view(np.int32)).to(dev)
    out = torch.zeros_like(P_)
    delta = torch.zeros((len(poses), 6), dtype=torch.float64, device=dev)
    stats = torch.zeros(4, dtype=torch.float32, device=dev)
    ctx.pose_graph_step(P_, pr, rec, n_max, out, delta=delta, stats=stats, **kw)
    torch.cuda.synchronize()
    return delta.cpu().numpy(), out.cpu().numpy(), stats.cpu().numpy()


@pytest.fixture(scope="module")
def ctx(bt):
    c = bt.Context(0)
    c.reserve(256, 512, 4096, 16, 640, 480)
    yield c
    c.close()


@pytest.mark.parametrize("lf,lg,fixed,precond", [(1.0, 1.0, 0, 1), (1.0, 1.0, 0, 0), (1.0, 0.0, 2, 1), (0.3, 2.0, 1, 0)])
def test_graph_step_parity_with_oracle_blocks(bt, torch, ctx, lf, lg, fixed, precond):
    sc = synth.make_scene(5, n=300, seed=21)
    pairs = synth.all_pairs(5)
    poses = sc.perturbed_poses(3, rot_deg=2.0, trans_m=0.01, fixed=fixed)
    feat, dij, dji = oracle_blocks(sc, poses, pairs)
    rec = records_from_blocks(bt, 512, feat, dij, dji)
    f32 = rec.view(np.float32)
    o = 28 + 16
    # the oracle consumes the same float32 blocks the record holds
    d_o, p_o, (Ef, Eg) = oracle.graph_step(poses, pairs, f32[:, o + 64:o + 160].astype(np.float64),
                                           f32[:, o:o + 32].astype(np.float64), f32[:, o + 32:o + 64].astype(np.float64),
                                           lambda_f=lf, lambda_g=lg, fixed_node=fixed)
    d_g, p_g, st = gpu_step(bt, torch, ctx, poses, pairs, rec, 512, lambda_feat=lf, lambda_dense=lg,
                            fixed_node=fixed, max_iter=2000, rel_tol=1e-13, precond=precond)
    assert np.all(d_g[fixed] == 0) and np.array_equal(p_g[fixed], poses[fixed])
    scale = np.abs(d_o).max()
    assert np.abs(d_g - d_o).max() <= 1e-7 * scale + 1e-12, (np.abs(d_g - d_o).max(), scale)
    assert np.abs(p_g - p_o).max() <= 2e-6
    assert st[0] == pytest.approx(Ef, rel=1e-6) and st[1] == pytest.approx(Eg, rel=1e-6)
    assert 1 <= st[2] <= 2000 and st[3] <= 1e-12


def test_graph_step_unconstrained_node_and_skipped_pairs(bt, torch, ctx):
    sc = synth.make_scene(4, n=300, seed=22)
    pairs = np.array([(0, 1), (1, 2), (0, 2), (2, 2), (1, 9)], np.int32)    # (2,2), (1,9) skipped; node 3 free
    poses = sc.perturbed_poses(4, rot_deg=2.0, trans_m=0.01)
    feat, dij, dji = oracle_blocks(sc, poses, pairs[:3])
    z96, z32 = np.zeros((2, 96)), np.zeros((2, 32))
    rec = records_from_blocks(bt, 512, np.vstack([feat, z96]), np.vstack([dij, z32]), np.vstack([dji, z32]))
    d_g, p_g, st = gpu_step(bt, torch, ctx, poses, pairs, rec, 512, fixed_node=0, max_iter=400, rel_tol=1e-13)
    f32 = rec.view(np.float32)
    o = 28 + 16
    d_o, p_o, _ = oracle.graph_step(poses, pairs[:3], f32[:3, o + 64:o + 160].astype(np.float64),
                                    f32[:3, o:o + 32].astype(np.float64), f32[:3, o + 32:o + 64].astype(np.float64))
    assert np.all(d_g[3] == 0) and np.array_equal(p_g[3], poses[3])
    assert np.abs(d_g - d_o).max() <= 1e-7 * np.abs(d_o).max()


def test_graph_step_c2_full_size_descends(bt, torch, ctx):
    """BASELINE configs[1] size: register the 120 pairs at perturbed node poses, one graph
    step, re-register at the new poses: the Eq. (1) energy (lambda = 1) drops; I_0 is fixed;
    the step is bitwise reproducible."""
    sc = synth.make_scene(16)
    pairs = synth.all_pairs(16)
    uids = np.arange(len(pairs), dtype=np.uint32)
    fb = bt.FrameBatch.from_scene(sc)
    rw = bt.record_words(512)
    pr = torch.from_numpy(pairs).cuda()
    ud = torch.from_numpy(uids.view(np.int32)).cuda()
    rprm, eprm = bt.ransac_params(4096, synth.PHILOX_SEED), bt.edge_params()

    def register(P_):
        rec = torch.zeros((len(pairs), rw), dtype=torch.int32, device="cuda")
        ctx.register_pairs(fb, sc.K, P_, pr, ud, rprm, eprm, rec)
        torch.cuda.synchronize()
        return rec

    def energy(rec):
        d = bt.decode_records(rec, 512)
        return float(d["feat"][:, 90].sum() + d["dense_ij"][:, 27].sum() + d["dense_ji"][:, 27].sum())

    P0 = torch.from_numpy(sc.perturbed_poses(8, rot_deg=2.0, trans_m=0.01)).cuda()
    rec0 = register(P0)
    P1 = torch.zeros_like(P0)
    stats = torch.zeros(4, dtype=torch.float32, device="cuda")
    ctx.pose_graph_step(P0, pr, rec0, 512, P1, stats=stats)
    P1b = torch.zeros_like(P0)
    ctx.pose_graph_step(P0, pr, rec0, 512, P1b)
    torch.cuda.synchronize()
    assert torch.equal(P1, P1b)
    assert torch.equal(P1[0], P0[0])
    E0, E1 = energy(rec0), energy(register(P1))
    st = stats.cpu().numpy()
    assert st[0] + st[1] == pytest.approx(E0, rel=1e-4)
    assert E1 < 0.5 * E0, (E0, E1)


def test_graph_step_errors(bt, torch, ctx):
    P_ = torch.zeros((3, 12), dtype=torch.float32, device="cuda")
    pr = torch.zeros((1, 2), dtype=torch.int32, device="cuda")
    rec = torch.zeros((1, bt.record_words(512)), dtype=torch.int32, device="cuda")
    with pytest.raises(bt.BtError, match="EINVAL"):
        ctx.pose_graph_step(P_, pr, rec, 512, P_, fixed_node=3)
    with pytest.raises(bt.BtError, match="EINVAL"):
        ctx.pose_graph_step(P_, pr, rec, 512, P_, max_iter=0)
    with pytest.raises(bt.BtError, match="ECAPACITY"):
        big = torch.zeros((17, 12), dtype=torch.float32, device="cuda")
        ctx.pose_graph_step(big, pr, rec, 512, big)


def test_relinearize_equals_registration_and_gn_iterations_descend(bt, torch, ctx):
    """bt_relinearize (C_ij reused) at new poses writes exactly what bt_register_pairs
    writes there (matching / RANSAC do not depend on the node poses); iterating
    relinearize + graph step descends Eq. (1)."""
    sc = synth.make_scene(8, seed=31)
    pairs = synth.all_pairs(8)
    uids = np.arange(len(pairs), dtype=np.uint32)
    fb = bt.FrameBatch.from_scene(sc)
    rw = bt.record_words(512)
    pr = torch.from_numpy(pairs).cuda()
    ud = torch.from_numpy(uids.view(np.int32)).cuda()
    rprm, eprm = bt.ransac_params(2048, synth.PHILOX_SEED), bt.edge_params()

    def register(P_):
        rec = torch.zeros((len(pairs), rw), dtype=torch.int32, device="cuda")
        ctx.register_pairs(fb, sc.K, P_, pr, ud, rprm, eprm, rec)
        torch.cuda.synchronize()
        return rec

    def energy(rec):
        d = bt.decode_records(rec, 512)
        return float(d["feat"][:, 90].sum() + d["dense_ij"][:, 27].sum() + d["dense_ji"][:, 27].sum())

    P0 = torch.from_numpy(sc.perturbed_poses(12, rot_deg=2.0, trans_m=0.01)).cuda()
    rec = register(P0)
    P1 = torch.zeros_like(P0)
    ctx.pose_graph_step(P0, pr, rec, 512, P1)
    relin = rec.clone()
    ctx.relinearize(fb, sc.K, P1, pr, eprm, relin)
    torch.cuda.synchronize()
    fresh = register(P1)
    assert torch.equal(relin, fresh)
    # Gauss-Newton iterations: relinearize at the current poses, step
    E = [energy(rec)]
    P_ = P0.clone()
    for _ in range(3):
        ctx.relinearize(fb, sc.K, P_, pr, eprm, rec)
        Pn = torch.zeros_like(P_)
        ctx.pose_graph_step(P_, pr, rec, 512, Pn)
        P_ = Pn
        ctx.relinearize(fb, sc.K, P_, pr, eprm, rec)
        torch.cuda.synchronize()
        E.append(energy(rec))
    assert E[1] < 0.5 * E[0] and E[3] <= E[1] * 1.001, E
    with pytest.raises(bt.BtError, match="EINVAL"):
        ctx.relinearize(fb, sc.K, P_, pr[:5], eprm, rec[:5])


def test_relinearize_with_cached_matches_across_calls(bt, torch, ctx):
    """The C_ij cache across calls: pairs registered in two bt_register_pairs calls,
    their match lists kept by the caller (bt_copy_matches), re-linearized TOGETHER at new poses
    (bt_relinearize_matches) == one bt_register_pairs of all pairs at those poses, bitwise."""
    sc = synth.make_scene(8, seed=33)
    pairs = synth.all_pairs(8)
    P = len(pairs)
    uids = np.arange(100, 100 + P, dtype=np.uint32)
    fb = bt.FrameBatch.from_scene(sc)
    rw = bt.record_words(512)
    pr = torch.from_numpy(pairs).cuda()
    ud = torch.from_numpy(uids.view(np.int32)).cuda()
    rprm, eprm = bt.ransac_params(2048, synth.PHILOX_SEED), bt.edge_params()
    P0 = torch.from_numpy(sc.perturbed_poses(13, rot_deg=2.0, trans_m=0.01)).cuda()
    P1 = torch.from_numpy(sc.perturbed_poses(14, rot_deg=1.0, trans_m=0.005)).cuda()
    rec = torch.zeros((P, rw), dtype=torch.int32, device="cuda")
    mt = torch.full((P, 512, 2), -3, dtype=torch.int32, device="cuda")
    nm = torch.zeros(P, dtype=torch.int32, device="cuda")
    for lo, hi in ((0, 11), (11, P)):                              # two calls, like two frames
        r = torch.zeros((hi - lo, rw), dtype=torch.int32, device="cuda")
        ctx.register_pairs(fb, sc.K, P0, pr[lo:hi].contiguous(), ud[lo:hi].contiguous(), rprm, eprm, r)
        m_ = torch.empty((hi - lo, 512, 2), dtype=torch.int32, device="cuda")
        n_ = torch.empty(hi - lo, dtype=torch.int32, device="cuda")
        ctx.copy_matches(m_, n_)
        rec[lo:hi], mt[lo:hi], nm[lo:hi] = r, m_, n_
    with pytest.raises(bt.BtError, match="EINVAL"):                # the last call had P - 11 pairs
        ctx.copy_matches(mt[:11], nm[:11])
    ctx.relinearize(fb, sc.K, P1, pr, eprm, rec, matches=mt, n_matches=nm)
    fresh = torch.zeros_like(rec)
    ctx.register_pairs(fb, sc.K, P1, pr, ud, rprm, eprm, fresh)
    torch.cuda.synchronize()
    assert torch.equal(rec, fresh)
    d = bt.decode_records(fresh, 512)
    assert (d["status"] == 0).sum() >= P // 2
    with pytest.raises(bt.BtError, match="EINVAL"):
        ctx.relinearize(fb, sc.K, P1, pr, eprm, rec, matches=mt, n_matches=None)


def test_graph_step_failed_registrations_bring_no_feature_term(bt, torch, ctx):
    """Reading R30: a pair whose record says FEW_MATCHES / FEW_INLIERS contributes its dense edges
    but no Eq. (2) block — GPU and oracle (status array) agree; the same records with status OK
    give a different step."""
    sc = synth.make_scene(5, n=300, seed=23)
    pairs = synth.all_pairs(5)
    poses = sc.perturbed_poses(5, rot_deg=2.0, trans_m=0.01)
    feat, dij, dji = oracle_blocks(sc, poses, pairs)
    rec = records_from_blocks(bt, 512, feat, dij, dji)
    status = np.zeros(len(pairs), np.int32)
    status[[1, 4, 7]] = [2, 1, 2]
    rec[:, 0] = status
    f32 = rec.view(np.float32)
    o = 28 + 16
    args = (f32[:, o + 64:o + 160].astype(np.float64), f32[:, o:o + 32].astype(np.float64),
            f32[:, o + 32:o + 64].astype(np.float64))
    d_o, p_o, _ = oracle.graph_step(poses, pairs, *args, status=status)
    d_ok, _, _ = oracle.graph_step(poses, pairs, *args)
    d_g, p_g, _ = gpu_step(bt, torch, ctx, poses, pairs, rec, 512, max_iter=2000, rel_tol=1e-13)
    assert np.abs(d_g - d_o).max() <= 1e-7 * np.abs(d_o).max() + 1e-12
    assert np.abs(p_g - p_o).max() <= 2e-6
    assert np.abs(d_ok - d_o).max() > 1e-3 * np.abs(d_o).max()
