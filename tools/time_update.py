"""Times amgf_update_D in the bench's call sequence (after solves), wall and CUDA events, per phase."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

p = amgf_gen.config(3)
stream = torch.cuda.current_stream()
g = AMGF.from_problem(p, D=p.D_seq[0], stream=stream)
D_dev = [torch.from_numpy(p.D_seq[s].copy()).cuda() for s in range(10)]
b = torch.from_numpy(p.b).cuda()
x = torch.empty_like(b)
for k in range(3):
    t = time.perf_counter()
    g.update_D(D_dev[k])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    g.pcg(b, rtol=p.rtol, out=x)
    torch.cuda.synchronize()
    print(f"step {k}: update_D {1e3 * (t1 - t):.1f} ms, pcg {1e3 * (time.perf_counter() - t1):.1f} ms", flush=True)
for k in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record(stream); g.update_D(D_dev[k]); e1.record(stream); e1.synchronize()
    print(f"update_D alone: events {e0.elapsed_time(e1):.1f} ms wall {1e3 * (time.perf_counter() - t):.1f} ms")
