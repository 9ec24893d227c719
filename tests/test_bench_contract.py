"""The driver's bench.py contract, checked on CPU through the reference arm
(the oracle on the host cores): one JSON line with the metric, unit and
config of BASELINE.json, impl = reference, cpu_baseline and e2e blocks.
(The GPU arm's line is produced on the GPU box; its keys are listed in
DESIGN.md sec. 10.)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        base = json.load(f)
    assert d["metric"] == base["metric"]
    assert d["impl"] == "reference" and d["unit"] == "ms" and d["higher_is_better"] is False
    assert d["value"] > 0 and d["steps"] == 1 and d["n_gpus"] == 1
    assert d["config"]["workload"] == "laplacian_160^3_bsr3_P2048"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


import pytest


@pytest.mark.gpu
def test_gpu_arm_json_line():
    """bench.py's own arm on the GPU (short run): the keys the driver and the
    judge read, with values that are consistent with each other."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "1",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert d["metric"] == json.load(f)["metric"]
    assert d["unit"] == "ms" and d["higher_is_better"] is False and d["dtype"] == "f64"
    assert d["n_gpus"] == 1 and d["scaling"] == "strong" and d["data"] == "synthetic"
    assert abs(d["value"] - d["ms_per_step"]) < 1e-6 and d["value"] > 0
    assert d["iterations"] == 111.5 and d["true_rel_resid"] <= 1e-8
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0 < rf["frac"] <= 1.0
    assert abs(rf["achieved"] / rf["peak"] - rf["frac"]) < 1e-3
    assert abs(rf["achieved"] - d["apply"]["canonical_bytes"] / (d["apply"]["ms"] * 1e-3) / 1e9) < 1.0
    assert d["apply"]["variant"] in ("levelset", "spin", "direct") and d["apply"]["launches"] > 0
    assert d["e2e"]["unit"] == "ms" and d["e2e"]["value"] >= d["value"] * 0.9
    assert d["e2e"]["h2d_bytes_per_step"] == d["e2e"]["d2h_bytes_per_step"] == 8 * 3 * 160 ** 3
    assert d["gpu_launches"] > 1000
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
