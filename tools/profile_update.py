"""Profiling driver: cfg 3 setup, then one amgf_update_D inside NVTX range "upd" (numeric re-setup)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

p = amgf_gen.config(3)
g = AMGF.from_problem(p, D=p.D_seq[0])
D = torch.from_numpy(p.D_seq[5]).cuda()
g.update_D(D)
torch.cuda.synchronize()
t = time.perf_counter()
torch.cuda.nvtx.range_push("upd")
g.update_D(D)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("update_D wall ms", (time.perf_counter() - t) * 1e3)
