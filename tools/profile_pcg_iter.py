"""Profiling driver: cfg 3 setup, warm-up solve, then one PCG solve capped at 2 iterations inside an NVTX
range "pcg" (the launch list of a PCG step), and 3 fine-level SpMVs inside "spmv"."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

p = amgf_gen.config(3)
g = AMGF.from_problem(p, D=p.D_seq[-1])
b = torch.from_numpy(p.b).cuda()
x, rep = g.pcg(b, rtol=p.rtol, max_it=3)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("pcg")
x, rep = g.pcg(b, rtol=p.rtol, max_it=2)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
xr = torch.randn(p.n, dtype=torch.float64, device="cuda")
yr = torch.empty_like(xr)
torch.cuda.nvtx.range_push("spmv")
for _ in range(3):
    g.spmv(xr, 0, out=yr)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok", rep)
