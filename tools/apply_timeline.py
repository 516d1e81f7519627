"""Per-launch completion timeline of one cfg 3 AMGF apply on both streams (AMGF_LAUNCH_TIMELINE=1, no profiler)."""
import os
import sys

os.environ["AMGF_LAUNCH_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

p = amgf_gen.config(3)
g = AMGF.from_problem(p, D=p.D_seq[-1])
x = torch.randn(p.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    g.apply(x, out=y)
torch.cuda.synchronize()
for k in range(2):
    print(f"--- apply {k}", file=sys.stderr, flush=True)
    g.apply(x, out=y)
    torch.cuda.synchronize()
