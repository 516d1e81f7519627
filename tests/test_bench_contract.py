"""The bench.py JSON-line contract, checked on the small cfg 0 workload: the reference
(oracle) arm on the CPU, the GPU arm on a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--cfg", "0", "--steps", "3", "--warmup",
                          "3", *args], cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def check_base(d):
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["unit"] == "ms/system"
    assert d["higher_is_better"] is False and d["scaling"] == "weak" and d["vs_baseline"] is None
    assert d["dtype"] == "f64" and (d["steps"], d["warmup"], d["n_gpus"]) == (3, 3, 1)
    assert d["config"]["workload"].startswith("cfg0:")
    assert d["e2e"]["unit"] == d["unit"] and d["e2e"]["value"] > 0


def test_reference_arm_contract():
    d = run_bench("--impl", "reference")
    check_base(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["value"] == d["value"]
    assert (d["e2e"]["h2d_bytes_per_step"], d["e2e"]["d2h_bytes_per_step"]) == (0, 0)


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = run_bench("--no-cpu-baseline")
    check_base(d)
    assert "impl" not in d or d["impl"] != "reference"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["traffic"] is None  # the committed ncu capture is of cfg 3, not this workload
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert len(d["pcg_iterations"]) == 3 and all(i > 0 for i in d["pcg_iterations"])
