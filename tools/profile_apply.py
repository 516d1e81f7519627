"""Profiling driver: cfg 3 setup, warm-up, then ONE AMGF apply and ONE V-cycle inside NVTX ranges
("apply", "vcycle") so that ncu can select exactly those launches (--nvtx --nvtx-include apply/)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = amgf_gen.config(cfg)
g = AMGF.from_problem(p, D=p.D_seq[-1])
x = torch.randn(p.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    g.apply(x, out=y)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("apply")
g.apply(x, out=y)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
torch.cuda.nvtx.range_push("vcycle")
g.vcycle(x, out=y)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok", g.nlev, g.levels)
