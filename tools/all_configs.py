"""Per-config summary on the GPU: setup, numeric re-setup, PCG iterations and solve ms for
the config's first D system, and back-to-back V-cycle / AMGF-apply times.  One JSON line per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402


def timed(fn, x, y, reps):
    for _ in range(3):
        fn(x, out=y)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn(x, out=y)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


for cfg in [int(c) for c in sys.argv[1:]] or [0, 1, 2, 3]:
    p = amgf_gen.config(cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = AMGF.from_problem(p)
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t) * 1e3
    g.update_D(torch.from_numpy(p.D_seq[0] if p.D_seq.ndim == 2 else p.D).cuda())
    b = torch.from_numpy(p.b).cuda()
    g.pcg(b, rtol=p.rtol)
    _, rep = g.pcg(b, rtol=p.rtol)
    x = torch.randn(p.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    reps = 50 if p.n < 1e6 else 10
    print(json.dumps(dict(cfg=cfg, n=p.n, n_c=g.nc, levels=[L["nodes"] * L["b"] for L in g.levels],
                          setup_ms=setup_ms, update_D_ms=g.setup_times()["total"],
                          pcg_iterations=rep["iterations"], solve_ms=rep["solve_ms"],
                          vcycle_us=timed(g.vcycle, x, y, reps), apply_us=timed(g.apply, x, y, reps))), flush=True)
    g.close()
