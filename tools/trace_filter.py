"""Overlap timeline of the A_w solve (filter stream) and the full residual SpMV inside AMGF apply (cfg 3)."""
import os
import sys

os.environ["AMGF_TRACE_FILTER"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

p = amgf_gen.config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
g = AMGF.from_problem(p)
x = torch.randn(p.n, dtype=torch.float64, device="cuda")
for _ in range(4):
    g.apply(x)
torch.cuda.synchronize()
