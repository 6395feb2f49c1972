"""bench.py's JSON-line contract: the keys the driver reads, on both arms.

The reference arm (`--impl reference`, the CPU oracle timed on a bounded sample) runs here on
CPU; the product arm needs the GPU (short run, no e2e / CPU baseline legs)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                         timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]                      # exactly one JSON line
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1"], 600)
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True and d["unit"] == "pairs/s"
    assert "workload" in d["config"] and "model" not in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_product_arm_contract():
    d = _run(["--steps", "5", "--warmup", "3", "--no-e2e", "--no-cpu-baseline"], 900)
    assert BASE_KEYS <= d.keys()
    ref = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"], 600)
    assert d["metric"] == ref["metric"] and d["unit"] == ref["unit"]                 # same metric on both arms
    assert d["config"]["workload"] == ref["config"]["workload"]
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["gpu_launches"] > 0 and d["gpu_launches"] % 5 == 0                    # our kernels, per step
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and r["unit"] in ("GB/s", "TFLOP/s")
    assert r["achieved"] > 0 and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert "traffic" in r
    c = d["clocks"]
    assert c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
    # the HBM-bound stage reports its DRAM traffic against its algorithmic bytes
    dp = d["kernels"].get("k_dense_prep")
    if dp and "traffic_per_step" in dp:
        assert dp["algorithmic_bytes_per_step"] > 0 and dp["traffic_over_algorithmic"] > 0
