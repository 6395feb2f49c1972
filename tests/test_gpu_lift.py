"""NEXT-4 on the GPU: raw detector output (2-D keypoints + descriptors) and the depth / mask maps
are the only inputs.  bt_lift_keypoints (reading R29: pi_D^-1 at the keypoint with the nearest
pixel's depth; SPEC S:247 / S:262) against the oracle's bto_lift_keypoints — counts,
order, descriptors, points and normals bit for bit — and the whole raw-input chain
depth -> bt_estimate_normals -> bt_lift_keypoints -> bt_register_pairs against the oracle run
stage-isolated on the GPU's intermediate maps (the normal map's own parity: test_gpu_normals)."""
import dataclasses

import numpy as np
import pytest

import oracle
import parity
import synth

pytestmark = pytest.mark.gpu

SEED = synth.PHILOX_SEED
DENSE = dict(dist_gate=0.02, cos_gate=float(np.cos(np.deg2rad(45.0))), huber_delta=0.005, stride=1)


@pytest.fixture(scope="module")
def bt():
    import paper_2108_00516_b200 as m
    return m


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def detector_output(sc, seed=0, n_extra=24):
    """The scene's keypoints as a detector would report them: sub-pixel (u, v) of each keypoint
    (its projection) plus n_extra spurious ones per frame (background, off-frame, borders), at
    random positions in the list; descriptors alongside."""
    rng = np.random.default_rng(seed)
    F, n_max = sc.desc.shape[:2]
    K = sc.K
    uv = np.zeros((F, n_max, 2), np.float32)
    desc = np.zeros_like(sc.desc)
    n_in = np.zeros(F, np.int32)
    for f in range(F):
        n = int(sc.n_kp[f])
        p = sc.pts[f, :n].astype(np.float64)
        real = np.stack([K.fx * p[:, 0] / p[:, 2] + K.cx, K.fy * p[:, 1] / p[:, 2] + K.cy], 1)
        m = min(n_extra, n_max - n)
        extra = np.stack([rng.uniform(-3, K.width + 3, m), rng.uniform(-3, K.height + 3, m)], 1)
        allp = np.concatenate([real, extra])
        alld = np.concatenate([sc.desc[f, :n], rng.normal(size=(m, 128)).astype(np.float32)])
        order = rng.permutation(n + m)
        uv[f, :n + m] = allp[order]
        desc[f, :n + m] = alld[order]
        n_in[f] = n + m
    return uv, desc, n_in


def gpu_lift(bt, torch, ctx, uv, desc, n_in, maps_fb, K):
    F, n_max = desc.shape[:2]
    out = bt.FrameBatch(torch.zeros(F, dtype=torch.int32, device="cuda"),
                        torch.zeros((F, n_max, 128), dtype=torch.float32, device="cuda"),
                        torch.zeros((F, n_max, 3), dtype=torch.float32, device="cuda"),
                        torch.zeros((F, n_max, 3), dtype=torch.float32, device="cuda"),
                        maps_fb.depth, maps_fb.normal, maps_fb.mask)
    ctx.lift_keypoints(torch.from_numpy(uv).cuda(), torch.from_numpy(desc).cuda(), torch.from_numpy(n_in).cuda(),
                       maps_fb, K, out)
    torch.cuda.synchronize()
    return out


def _compare(out, ref):
    n = out.n_kp.cpu().numpy()
    assert np.array_equal(n, ref["n"])
    d, p, q = out.desc.cpu().numpy(), out.pts.cpu().numpy(), out.nrm.cpu().numpy()
    for f in range(len(n)):
        k = n[f]
        assert np.array_equal(d[f, :k], ref["desc"][f, :k])
        assert np.array_equal(p[f, :k], ref["pts"][f, :k]), f"frame {f}: points differ"
        assert np.array_equal(q[f, :k], ref["nrm"][f, :k])


def test_lift_parity_c2(bt, torch):
    sc = synth.make_scene(16)
    uv, desc, n_in = detector_output(sc)
    ctx = bt.Context(0)
    fb = bt.FrameBatch.from_scene(sc)
    out = gpu_lift(bt, torch, ctx, uv, desc, n_in, fb, sc.K)
    ref = oracle.lift_keypoints(uv, desc, n_in, sc.depth, sc.normal, sc.mask, sc.K)
    # borderline roundings (band rule) need no exclusion: both sides round the same float in the
    # same fp64 arithmetic, so every keypoint must agree exactly
    _compare(out, ref)
    assert (ref["n"] > 400).all() and (ref["n"] < n_in).all()          # spurious ones dropped
    ctx.close()


def test_lift_edge_cases(bt, torch):
    """Empty frames, n_in > n_max (clamped), keypoints exactly on the frame edge, all dropped."""
    sc = synth.make_scene(3, n=100, n_max=128, width=160, height=120, distance=0.9, seed=3)
    uv, desc, n_in = detector_output(sc, seed=5, n_extra=28)
    n_in[0] = 0
    n_in[2] = 1000                                                      # clamped to n_max
    uv[1, :4] = [[-0.5, 10.0], [159.49, 10.0], [-0.51, 10.0], [159.5, 10.0]]   # first two in frame
    ctx = bt.Context(0)
    fb = bt.FrameBatch.from_scene(sc)
    out = gpu_lift(bt, torch, ctx, uv, desc, n_in, fb, sc.K)
    ref = oracle.lift_keypoints(uv, desc, n_in, sc.depth, sc.normal, sc.mask, sc.K)
    _compare(out, ref)
    assert ref["n"][0] == 0
    ctx.close()


def test_raw_input_chain_depth_mask_keypoints_only(bt, torch):
    """C2 from raw inputs only: depth + mask -> bt_estimate_normals -> bt_lift_keypoints ->
    bt_register_pairs (120 pairs, 4096 hypotheses, 640x480).  The oracle, run on the GPU's
    normal map (stage isolation), lifts the same keypoints bit for bit, and registers sampled
    pairs equal to the GPU's records (band rule, tolerances of the north star)."""
    sc = synth.make_scene(16)
    uv, desc, n_in = detector_output(sc, seed=9)
    ctx = bt.Context(0)
    ctx.reserve(120, 512, 4096, 16, 640, 480)
    depth = torch.from_numpy(sc.depth).cuda()
    mask = torch.from_numpy(sc.mask).cuda()
    normal = torch.empty((16, 480, 640, 3), dtype=torch.float32, device="cuda")
    ctx.estimate_normals(depth, sc.K, normal)
    maps = bt.FrameBatch(None, None, None, None, depth, normal, mask)
    kp = gpu_lift(bt, torch, ctx, uv, desc, n_in, maps, sc.K)
    nrm_map = normal.cpu().numpy()
    ref = oracle.lift_keypoints(uv, desc, n_in, sc.depth, nrm_map, sc.mask, sc.K)
    _compare(kp, ref)
    pairs = synth.all_pairs(16)
    poses = sc.perturbed_poses(11)
    rec = torch.zeros((len(pairs), bt.record_words(512)), dtype=torch.int32, device="cuda")
    ctx.register_pairs(kp, sc.K, torch.from_numpy(poses).cuda(), torch.from_numpy(pairs).cuda(),
                       torch.arange(len(pairs), dtype=torch.int32, device="cuda"), bt.ransac_params(4096, SEED),
                       bt.edge_params(), rec)
    torch.cuda.synchronize()
    r_all = bt.decode_records(rec, 512)
    assert (r_all["status"] == 0).all()
    lifted = dataclasses.replace(sc, n_kp=ref["n"], desc=ref["desc"], pts=ref["pts"], nrm=ref["nrm"], normal=nrm_map)
    for p in (0, 33, 77, 119):
        a, b = pairs[p]
        o = oracle.register_pair(lifted, a, b, p, 4096, SEED, node_poses=poses, dense=DENSE, counts_out=True)
        r = {k: v[p] for k, v in r_all.items()}
        assert r["n_matches"] == o["n_matches"]
        P_ = o["match"]["pairs"]
        ia, ib = P_[:, 0], P_[:, 1]
        parity.compare_ransac(None, r, o["counts"], lifted.pts[a][ia], lifted.nrm[a][ia], lifted.pts[b][ib],
                              lifted.nrm[b][ib], what=f"raw pair {p}")
        parity.assert_dense_close(r["dense_ij"], o["dense_ij"], f"raw pair {p} ij")
        parity.assert_dense_close(r["dense_ji"], o["dense_ji"], f"raw pair {p} ji")
    ctx.close()


def test_raw_host_entry_equals_device_chain(bt, torch):
    """bt_register_raw_host (host depth / mask / 2-D keypoints / descriptors in, records out; the
    end-to-end entry bench.py times) equals the device chain bt_estimate_normals ->
    bt_lift_keypoints -> bt_register_pairs on the same inputs bit for bit — with and without the
    dense edges — and its capacity / argument errors."""
    sc = synth.make_scene(16)
    uv, desc, n_in = detector_output(sc, seed=13)
    pairs = synth.all_pairs(16)
    poses = sc.perturbed_poses(12)
    uid = np.arange(len(pairs), dtype=np.int32) + 7
    ctx = bt.Context(0)
    ctx.reserve(120, 512, 4096, 16, 640, 480)
    rprm = bt.ransac_params(4096, SEED)
    depth = torch.from_numpy(sc.depth).cuda()
    mask = torch.from_numpy(sc.mask).cuda()
    normal = torch.empty((16, 480, 640, 3), dtype=torch.float32, device="cuda")
    ctx.estimate_normals(depth, sc.K, normal, jump=0.05)           # the raw entry's jump_m default
    maps = bt.FrameBatch(None, None, None, None, depth, normal, mask)
    kp = gpu_lift(bt, torch, ctx, uv, desc, n_in, maps, sc.K)
    for eprm in (bt.edge_params(), None):
        dev_rec = torch.zeros((len(pairs), bt.record_words(512)), dtype=torch.int32, device="cuda")
        ctx.register_pairs(kp, sc.K, torch.from_numpy(poses).cuda(), torch.from_numpy(pairs).cuda(),
                           torch.from_numpy(uid).cuda(), rprm, eprm, dev_rec)
        torch.cuda.synchronize()
        host_rec = torch.zeros((len(pairs), bt.record_words(512)), dtype=torch.int32).pin_memory()
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        ctx.register_raw(pin(sc.depth), pin(sc.mask), pin(uv), pin(desc), pin(n_in), sc.K, pin(poses),
                         pin(pairs.astype(np.int32)), pin(uid), rprm, eprm, host_rec)
        got = host_rec.numpy()
        want = dev_rec.cpu().numpy()
        if eprm is None:                                          # dense / feature words are not written
            n_ransac = 28 + 512 // 32
            got, want = got[:, :n_ransac], want[:, :n_ransac]
        assert np.array_equal(got, want), "raw host entry differs from the device chain"
    # errors: dim != 128, frames beyond the staging, NULL buffers
    host_rec = np.zeros((len(pairs), bt.record_words(512)), np.int32)
    with pytest.raises(bt.BtError, match="EUNSUPPORTED"):
        ctx.register_raw(sc.depth, sc.mask, uv, desc[:, :, :64].copy(), n_in, sc.K, poses, pairs.astype(np.int32),
                         uid, rprm, None, host_rec)
    big = np.zeros((17, 480, 640), np.float32)
    with pytest.raises(bt.BtError, match="ECAPACITY"):
        ctx.register_raw(big, np.zeros((17, 480, 640), np.uint8), np.zeros((17, 512, 2), np.float32),
                         np.zeros((17, 512, 128), np.float32), np.zeros(17, np.int32), sc.K,
                         np.zeros((17, 12), np.float32), pairs.astype(np.int32), uid, rprm, None, host_rec)
    ctx.close()


def test_raw_host_async_pipelined_equals_blocking(bt, torch):
    """bt_register_raw_host_async: four calls in flight on one stream (two different frame
    batches A, B alternating, so the two staging slots hold different inputs while the copies
    of call t + 1 overlap the kernels of call t) give, after one synchronisation, the records
    of the blocking calls bit for bit."""
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    batches = []
    for seed in (21, 22):
        sc = synth.make_scene(16, seed=seed)
        uv, desc, n_in = detector_output(sc, seed=seed + 1)
        pairs = synth.all_pairs(16)
        batches.append((sc, [pin(sc.depth), pin(sc.mask), pin(uv), pin(desc), pin(n_in)],
                        pin(sc.perturbed_poses(seed)), pin(pairs.astype(np.int32)),
                        pin(np.arange(len(pairs), dtype=np.int32) + seed)))
    ctx = bt.Context(0)
    ctx.reserve(120, 512, 4096, 16, 640, 480)
    rprm, eprm = bt.ransac_params(4096, SEED), bt.edge_params()
    rw = bt.record_words(512)
    want = []
    for sc, inp, poses, pairs, uid in batches:
        r = torch.zeros((len(pairs), rw), dtype=torch.int32).pin_memory()
        ctx.register_raw(*inp, sc.K, poses, pairs, uid, rprm, eprm, r)
        want.append(r.numpy().copy())
    s = torch.cuda.Stream()
    outs = []
    for k in range(4):
        sc, inp, poses, pairs, uid = batches[k % 2]
        r = torch.zeros((len(pairs), rw), dtype=torch.int32).pin_memory()
        ctx.register_raw(*inp, sc.K, poses, pairs, uid, rprm, eprm, r, stream=s, blocking=False)
        outs.append(r)
    s.synchronize()
    for k, r in enumerate(outs):
        assert np.array_equal(r.numpy(), want[k % 2]), f"async call {k} differs from the blocking call"
    assert not np.array_equal(want[0], want[1])
    ctx.close()


def test_raw_host_depth_u16_equals_f32(bt, torch):
    """A uint16 depth map (the sensor / dataset format, 0 = invalid) with depth_scale gives the
    records of the f32 depth map holding float32(value) * float32(scale) — blocking and async —
    and depth_scale <= 0 is rejected."""
    sc = synth.make_scene(16, seed=31)
    uv, desc, n_in = detector_output(sc, seed=32)
    pairs = synth.all_pairs(16).astype(np.int32)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    d_mm = np.where(sc.depth > 0, np.rint(sc.depth * 1000.0), 0).clip(0, 65535).astype(np.uint16)
    d_f = d_mm.astype(np.float32) * np.float32(1e-3)
    ctx = bt.Context(0)
    ctx.reserve(120, 512, 4096, 16, 640, 480)
    rprm, eprm = bt.ransac_params(4096, SEED), bt.edge_params()
    rw = bt.record_words(512)
    args = (pin(sc.mask), pin(uv), pin(desc), pin(n_in), sc.K, pin(sc.perturbed_poses(3)), pin(pairs),
            pin(np.arange(len(pairs), dtype=np.int32)), rprm, eprm)
    want = torch.zeros((len(pairs), rw), dtype=torch.int32).pin_memory()
    ctx.register_raw(pin(d_f), *args, want)
    got = torch.zeros_like(want).pin_memory()
    ctx.register_raw(pin(d_mm), *args, got, depth_scale=1e-3)
    assert np.array_equal(got.numpy(), want.numpy())
    s = torch.cuda.Stream()
    got2 = [torch.zeros_like(want).pin_memory() for _ in range(2)]
    h_dmm = pin(d_mm)                                   # alive until the stream has passed the calls
    for r in got2:
        ctx.register_raw(h_dmm, *args, r, stream=s, blocking=False, depth_scale=1e-3)
    s.synchronize()
    for r in got2:
        assert np.array_equal(r.numpy(), want.numpy())
    assert (bt.decode_records(want, 512)["status"] == 0).all()
    with pytest.raises(bt.BtError, match="EINVAL"):
        ctx.register_raw(pin(d_mm), *args, got, depth_scale=0.0)
    ctx.close()


def test_raw_host_depth_u16_odd_size(bt, torch):
    """The uint16 depth conversion's tail (a pixel count that is not a multiple of 8, odd row
    length): records equal the f32 call on the same values."""
    sc = synth.make_scene(3, n=100, n_max=128, width=161, height=121, distance=0.35, seed=41)
    uv, desc, n_in = detector_output(sc, seed=42)
    pairs = synth.all_pairs(3).astype(np.int32)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    d_mm = np.where(sc.depth > 0, np.rint(sc.depth * 1000.0), 0).clip(0, 65535).astype(np.uint16)
    d_f = d_mm.astype(np.float32) * np.float32(1e-3)
    assert d_mm.size % 8 != 0
    ctx = bt.Context(0)
    ctx.reserve(len(pairs), 128, 1024, 3, 161, 121)
    rprm, eprm = bt.ransac_params(1024, SEED), bt.edge_params()
    args = (pin(sc.mask), pin(uv), pin(desc), pin(n_in), sc.K, pin(sc.perturbed_poses(2)), pin(pairs),
            pin(np.arange(len(pairs), dtype=np.int32)), rprm, eprm)
    want = torch.zeros((len(pairs), bt.record_words(128)), dtype=torch.int32).pin_memory()
    got = torch.zeros_like(want).pin_memory()
    ctx.register_raw(pin(d_f), *args, want)
    ctx.register_raw(pin(d_mm), *args, got, depth_scale=1e-3)
    assert np.array_equal(got.numpy(), want.numpy())
    ctx.close()


@pytest.mark.parametrize("width", [640, 161])
def test_raw_host_mask_bits_equal_bytes(bt, torch, width):
    """A packed-bit mask ([F][H][ceil(W/8)], LSB first; unpacked on the device) gives the records
    of the byte mask — blocking and async, a row length that is and one that is not a multiple of
    8 — and mask + mask_bits together are rejected."""
    H = 480 if width == 640 else 121
    sc = synth.make_scene(3, n=300 if width == 640 else 100, n_max=512 if width == 640 else 128, width=width,
                          height=H, distance=0.6 if width == 640 else 0.35, seed=51)
    n_max = sc.desc.shape[1]
    uv, desc, n_in = detector_output(sc, seed=52)
    pairs = synth.all_pairs(3).astype(np.int32)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    bits = np.packbits(sc.mask != 0, axis=-1, bitorder="little")
    assert bits.shape == (3, H, (width + 7) // 8)
    ctx = bt.Context(0)
    ctx.reserve(len(pairs), n_max, 1024, 3, width, H)
    rprm, eprm = bt.ransac_params(1024, SEED), bt.edge_params()
    tail = (pin(uv), pin(desc), pin(n_in), sc.K, pin(sc.perturbed_poses(4)), pin(pairs),
            pin(np.arange(len(pairs), dtype=np.int32)), rprm, eprm)
    want = torch.zeros((len(pairs), bt.record_words(n_max)), dtype=torch.int32).pin_memory()
    ctx.register_raw(pin(sc.depth), pin((sc.mask != 0).astype(np.uint8)), *tail, want)
    got = torch.zeros_like(want).pin_memory()
    ctx.register_raw(pin(sc.depth), pin(bits), *tail, got, mask_bits=True)
    assert np.array_equal(got.numpy(), want.numpy())
    s = torch.cuda.Stream()
    got2 = [torch.zeros_like(want).pin_memory() for _ in range(2)]
    h_depth, h_bits = pin(sc.depth), pin(bits)          # alive until the stream has passed the calls
    for r in got2:
        ctx.register_raw(h_depth, h_bits, *tail, r, stream=s, blocking=False, mask_bits=True)
    s.synchronize()
    for r in got2:
        assert np.array_equal(r.numpy(), want.numpy())
    ctx.close()


def test_raw_host_large_n_compact_inputs_equal_device_chain(bt, torch):
    """The streaming raw entry at a stress-config keypoint count (n = 2048: the batched
    matching path with its level-2 pass and the top-2 candidate sets) from the compact inputs —
    uint16 depth and a packed-bit mask — equals the device chain bt_estimate_normals ->
    bt_lift_keypoints -> bt_register_pairs on the same (dequantised) maps, bit for bit."""
    sc = synth.make_scene(4, n=2048, n_max=2048, pool_size=7000, seed=81, outlier_frac=0.16)
    uv, desc, n_in = detector_output(sc, seed=82)
    pairs = synth.all_pairs(4).astype(np.int32)
    uid = np.arange(len(pairs), dtype=np.int32) + 3
    poses = sc.perturbed_poses(6)
    d_mm = np.where(sc.depth > 0, np.rint(sc.depth * 1000.0), 0).clip(0, 65535).astype(np.uint16)
    d_f = d_mm.astype(np.float32) * np.float32(1e-3)
    bits = np.packbits(sc.mask != 0, axis=-1, bitorder="little")
    ctx = bt.Context(0)
    ctx.reserve(len(pairs), 2048, 4096, 4, 640, 480)
    rprm, eprm = bt.ransac_params(4096, SEED), bt.edge_params()
    depth = torch.from_numpy(d_f).cuda()
    mask = torch.from_numpy((sc.mask != 0).astype(np.uint8)).cuda()
    normal = torch.empty((4, 480, 640, 3), dtype=torch.float32, device="cuda")
    ctx.estimate_normals(depth, sc.K, normal, jump=0.05)
    maps = bt.FrameBatch(None, None, None, None, depth, normal, mask)
    kp = gpu_lift(bt, torch, ctx, uv, desc, n_in, maps, sc.K)
    dev_rec = torch.zeros((len(pairs), bt.record_words(2048)), dtype=torch.int32, device="cuda")
    ctx.register_pairs(kp, sc.K, torch.from_numpy(poses).cuda(), torch.from_numpy(pairs).cuda(),
                       torch.from_numpy(uid).cuda(), rprm, eprm, dev_rec)
    torch.cuda.synchronize()
    want = dev_rec.cpu().numpy()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    # the host inputs stay alive (and unchanged) until the stream has passed the calls
    h = [pin(x) for x in (d_mm, bits, uv, desc, n_in)]
    hp = [pin(x) for x in (poses, pairs, uid)]
    s = torch.cuda.Stream()
    outs = [torch.zeros((len(pairs), bt.record_words(2048)), dtype=torch.int32).pin_memory() for _ in range(3)]
    for r in outs:
        ctx.register_raw(*h, sc.K, *hp, rprm, eprm, r, stream=s, blocking=False, depth_scale=1e-3, mask_bits=True)
    s.synchronize()
    for r in outs:
        assert np.array_equal(r.numpy(), want)
    assert (bt.decode_records(want, 2048)["status"] == 0).all()
    ctx.close()
