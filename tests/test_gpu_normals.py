"""GPU parity of NEXT-4 input prep (bt_estimate_normals: the normal map from depth, SPEC
estimate_normals S:157-165) against the oracle, through the C ABI: identical validity, unit
normals within 2e-5 (fp32 vs the fp64 oracle) outside grazing pixels whose camera-facing sign
is decided at |n . P| ~ 0."""
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


@pytest.fixture(scope="module")
def ctx(bt):
    c = bt.Context(0)
    c.reserve(4, 512, 1024, 16, 640, 480)
    yield c
    c.close()


def gpu_normals(bt, torch, ctx, depth, K, jump=0.05):
    d = torch.from_numpy(np.ascontiguousarray(depth, np.float32)).cuda()
    out = torch.full(tuple(depth.shape) + (3,), -7.0, dtype=torch.float32, device="cuda")
    ctx.estimate_normals(d, K, out, jump)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def compare(depth, K, g, o):
    vg = np.linalg.norm(g, axis=-1) > 0
    vo = np.linalg.norm(o, axis=-1) > 0
    assert np.array_equal(vg, vo)
    # grazing pixels: the facing sign is decided on n . P ~ 0 (band rule, R22)
    F, H, W = depth.shape if depth.ndim == 3 else (1,) + depth.shape
    u, v = np.meshgrid(np.arange(W), np.arange(H))
    ray = np.stack([(u - K.cx) / K.fx, (v - K.cy) / K.fy, np.ones((H, W))], -1)
    ray /= np.linalg.norm(ray, axis=-1, keepdims=True)
    cosv = np.abs(np.sum(o * ray, -1))
    keep = vo & (cosv > 1e-4)
    if keep.any():
        assert np.abs(g[keep] - o[keep]).max() <= 2e-5
    return vo.sum()


def test_normals_parity_c2_maps(bt, torch, ctx):
    sc = synth.make_scene(16, n=100)
    g = gpu_normals(bt, torch, ctx, sc.depth, sc.K)
    o = oracle.estimate_normals(sc.depth, sc.K)
    assert compare(sc.depth, sc.K, g, o) > 16 * 20000


@pytest.mark.parametrize("W,H", [(157, 119), (64, 16), (3, 3), (1, 5), (130, 33)])
def test_normals_ragged_sizes(bt, torch, ctx, W, H):
    rng = np.random.default_rng(W * H)
    K = synth.Intrinsics(300.0, 310.0, (W - 1) / 2.0, (H - 1) / 2.0, W, H)
    depth = (0.6 + 0.02 * rng.standard_normal((2, H, W))).astype(np.float32)
    depth[rng.uniform(size=depth.shape) < 0.05] = 0.0              # holes
    depth[:, : H // 2, : W // 3] += 0.1                            # a jump edge
    g = gpu_normals(bt, torch, ctx, depth, K)
    o = oracle.estimate_normals(depth, K)
    compare(depth, K, g, o)


def test_normals_edge_cases(bt, torch, ctx):
    K = synth.Intrinsics(600.0, 600.0, 79.5, 59.5, 160, 120)
    z = np.zeros((1, 120, 160), np.float32)
    assert not gpu_normals(bt, torch, ctx, z, K).any()            # every output written (was -7)
    d = np.full((1, 120, 160), 0.8, np.float32)
    g = gpu_normals(bt, torch, ctx, d, K, jump=0.0)                # equal neighbours pass a 0 jump
    assert np.array_equal(g[0, 1:-1, 1:-1], np.broadcast_to(np.float32([0, 0, -1]), (118, 158, 3)))
    with pytest.raises(bt.BtError, match="EINVAL"):
        gpu_normals(bt, torch, ctx, d, K, jump=-1.0)


def test_normals_unaligned_depth_pointer(bt, torch, ctx):
    """A depth pointer that is not 16-B aligned takes the scalar path (no misaligned float4)."""
    K = synth.Intrinsics(600.0, 600.0, 79.5, 59.5, 160, 120)
    sc = synth.make_scene(1, n=50, width=160, height=120, seed=4, distance=0.35)
    flat = torch.zeros(1 + 120 * 160, dtype=torch.float32, device="cuda")
    flat[1:] = torch.from_numpy(sc.depth.reshape(-1)).cuda()
    d = flat[1:].view(1, 120, 160)                                  # 4-byte offset
    out = torch.zeros((1, 120, 160, 3), dtype=torch.float32, device="cuda")
    ctx.estimate_normals(d, K, out)
    torch.cuda.synchronize()
    compare(sc.depth, K, out.cpu().numpy(), oracle.estimate_normals(sc.depth, K))


def test_reserve_rejects_oversized_keypoint_sets(bt):
    c = bt.Context(0)
    with pytest.raises(bt.BtError, match="EUNSUPPORTED"):
        c.reserve(1, 8193, 16)
    c.reserve(1, 8192, 16)                                          # the limit itself is fine
    c.close()
