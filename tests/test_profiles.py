"""The committed measurement artefacts stay readable by their tools and consistent with what bench.py quotes."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def test_spmv_traffic_matches_its_ncu_capture():
    t = json.load(open(os.path.join(PROF, "spmv_traffic.json")))
    src = t["source"].split(" ")[0]
    assert os.path.exists(os.path.join(ROOT, src)), src
    # DRAM traffic of the dominant kernel: at least its algorithmic bytes, and no wasted re-reads (< 5 % above)
    assert 1.0 <= t["dram_bytes_per_launch"] / t["algorithmic_bytes_per_launch"] < 1.05


def test_launch_list_tools_read_the_committed_csv():
    csv = os.path.join(PROF, "r02_launches_apply_cfg3.csv")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "summary_table.py"), csv], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0, out.stderr[-1000:]
    rows = [ln for ln in out.stdout.splitlines() if ln.startswith("| `k_sell<3, 3")]
    assert len(rows) >= 3, out.stdout[-1000:]
    # the fine-level SELL passes carry at least half of one AMGF apply
    share = sum(float(r.split("|")[4].strip().rstrip(" %")) for r in rows)
    assert share > 50.0, share


def test_bench_line_of_record_is_the_named_workload():
    d = json.load(open(os.path.join(PROF, "r02_bench_cfg3.json")))
    assert d["config"]["workload"].startswith("cfg3:") and d["unit"] == "ms/system" and d["dtype"] == "f64"
    assert abs(d["roofline"]["frac"] - d["roofline"]["achieved"] / d["roofline"]["peak"]) < 1e-9
    assert d["gpu_launches"] > 0 and len(d["pcg_iterations"]) == d["steps"]
