"""CPU-side checks of the C-ABI boundary: libbt.so loads (no GPU needed to dlopen it) and
exports every function include/bt.h declares; the ctypes structs match the C layout;
the product path refuses to run without its CUDA library (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "bt.h")


@pytest.fixture(scope="module")
def bt():
    from paper_2108_00516_b200 import build
    build.build()
    import paper_2108_00516_b200 as m
    return m


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bt_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(bt):
    names = declared_functions()
    assert len(names) >= 13
    L = ctypes.CDLL(bt.LIB_PATH)
    for n in names:
        getattr(L, n)                                   # raises AttributeError if missing
    assert sorted(bt.SYMBOLS) == names
    nm = subprocess.run(["nm", "-D", "--defined-only", bt.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", nm, re.M), n


def test_record_words(bt):
    # 4 + 24 + ceil(n_max/32) + 64 + 96 (bt.h record layout)
    assert bt.record_words(512) == 204
    assert bt.record_words(4096) == 316
    assert bt.record_words(1) == 189
    assert bt.record_words(0) == 0


def _c_layout():
    code = r"""
#include <stdio.h>
#include <stddef.h>
#include "bt.h"
#define P(T, f) printf(#T "." #f " %zu\n", offsetof(T, f))
int main(void) {
  printf("sizeof.bt_ransac_params %zu\n", sizeof(bt_ransac_params));
  printf("sizeof.bt_keypoints %zu\n", sizeof(bt_keypoints));
  printf("sizeof.bt_maps %zu\n", sizeof(bt_maps));
  printf("sizeof.bt_intrinsics %zu\n", sizeof(bt_intrinsics));
  printf("sizeof.bt_edge_params %zu\n", sizeof(bt_edge_params));
  printf("sizeof.bt_pose %zu\n", sizeof(bt_pose));
  printf("sizeof.bt_graph_params %zu\n", sizeof(bt_graph_params));
  P(bt_graph_params, fixed_node); P(bt_graph_params, rel_tol); P(bt_graph_params, precond);
  P(bt_ransac_params, seed); P(bt_ransac_params, min_sigma_ratio); P(bt_ransac_params, min_inliers);
  P(bt_keypoints, n_kp); P(bt_keypoints, nrm); P(bt_maps, depth); P(bt_maps, mask);
  return 0;
}
"""
    d = "/tmp/bt_abi_layout"
    os.makedirs(d, exist_ok=True)
    open(f"{d}/l.c", "w").write(code)
    subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), f"{d}/l.c", "-o", f"{d}/l"])
    out = subprocess.check_output([f"{d}/l"], text=True)
    return dict(line.split() for line in out.strip().splitlines())


def test_ctypes_structs_match_c_layout(bt):
    c = {k: int(v) for k, v in _c_layout().items()}
    assert ctypes.sizeof(bt.RansacParams) == c["sizeof.bt_ransac_params"]
    assert ctypes.sizeof(bt.Keypoints) == c["sizeof.bt_keypoints"]
    assert ctypes.sizeof(bt.Maps) == c["sizeof.bt_maps"]
    assert ctypes.sizeof(bt.Intrinsics) == c["sizeof.bt_intrinsics"]
    assert ctypes.sizeof(bt.EdgeParams) == c["sizeof.bt_edge_params"]
    assert c["sizeof.bt_pose"] == 48
    assert bt.RansacParams.seed.offset == c["bt_ransac_params.seed"]
    assert bt.RansacParams.min_sigma_ratio.offset == c["bt_ransac_params.min_sigma_ratio"]
    assert bt.RansacParams.min_inliers.offset == c["bt_ransac_params.min_inliers"]
    assert bt.Keypoints.n_kp.offset == c["bt_keypoints.n_kp"]
    assert bt.Keypoints.nrm.offset == c["bt_keypoints.nrm"]
    assert bt.Maps.depth.offset == c["bt_maps.depth"]
    assert bt.Maps.mask.offset == c["bt_maps.mask"]
    assert ctypes.sizeof(bt.GraphParams) == c["sizeof.bt_graph_params"]
    assert bt.GraphParams.fixed_node.offset == c["bt_graph_params.fixed_node"]
    assert bt.GraphParams.rel_tol.offset == c["bt_graph_params.rel_tol"]
    assert bt.GraphParams.precond.offset == c["bt_graph_params.precond"]


def test_no_cpu_fallback(bt):
    """Without an sm_100 device the context refuses to exist: nothing silently runs on CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(bt.BtError):
        bt.Context(0)


def test_library_is_sm100a_only(bt):
    out = subprocess.run(["cuobjdump", "--list-elf", bt.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2108_00516_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", src).lower().replace("oracle/", ""), f
