"""Times AMGF apply (and its V-cycle) at cfg 3 with CUDA events, 20 back-to-back applies (each streams > 1 GB,
so the filter factor comes from HBM as in PCG).  Used to compare kernel variants selected by environment
variables (e.g. AMGF_SF_VARIANT); prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = amgf_gen.config(cfg)
cfg_over = json.loads(os.environ["AMGF_TIME_CONFIG"]) if os.environ.get("AMGF_TIME_CONFIG") else None
g = AMGF.from_problem(p, D=p.D_seq[-1], config=cfg_over)
torch.manual_seed(0)
x = torch.randn(p.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
ref = None
res = {"variant": {k: v for k, v in os.environ.items() if k.startswith("AMGF_")}}
for name, fn in (("apply", g.apply), ("vcycle", g.vcycle)):
    for _ in range(3):
        fn(x, out=y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        fn(x, out=y)
    e1.record()
    torch.cuda.synchronize()
    res[name + "_us"] = e0.elapsed_time(e1) / 20 * 1e3
    if name == "apply":
        res["apply_checksum"] = float(y.double().abs().sum())
res["levels"] = g.levels
res["config"] = cfg_over
print(json.dumps(res))
