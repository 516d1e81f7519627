"""Quick run of one config on the GPU: setup + one PCG solve per D system (up to 2), prints a summary."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

cfg = int(sys.argv[1])
t = time.time()
p = amgf_gen.config(cfg)
print(f"cfg{cfg} gen {time.time() - t:.1f}s n={p.n} m={p.m}", flush=True)
t = time.time()
g = AMGF.from_problem(p)
torch.cuda.synchronize()
print(f"setup {time.time() - t:.2f}s levels={[L['nodes'] * L['b'] for L in g.levels]} nc={g.nc} bw={g.bw} "
      f"mem={torch.cuda.max_memory_allocated() / 1e9:.2f} GB (torch) ", flush=True)
b = torch.from_numpy(p.b).cuda()
for s in range(min(2, p.D_seq.shape[0])):
    g.update_D(torch.from_numpy(p.D_seq[s]).cuda())
    x, rep = g.pcg(b, rtol=p.rtol)
    print(f"system {s}: {rep}", flush=True)
free, total = torch.cuda.mem_get_info()
print(f"device memory used {(total - free) / 1e9:.1f} GB of {total / 1e9:.1f}")
