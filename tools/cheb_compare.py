"""cfg 3, one system per D_max in {1e2, 1e7, 1e12}: PCG iterations and solve ms for l1-Jacobi vs Chebyshev
smoothing of degree 2 and 3 (variant f4).  One JSON line per (smoother, D_max)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

p = amgf_gen.config(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
b = torch.from_numpy(p.b).cuda()
systems = [0, 5, 9] if p.D_seq.shape[0] >= 10 else [0]
variants = (("l1-jacobi", dict(smoother=0)), ("cheb2", dict(smoother=1, cheb_degree=2)),
            ("cheb3", dict(smoother=1, cheb_degree=3)))
if len(sys.argv) > 2:  # extra: JSON list of [name, config] pairs
    variants = json.loads(sys.argv[2])
for name, cfg in variants:
    g = AMGF.from_problem(p, D=p.D_seq[systems[0]], config=cfg)
    for s in systems:
        g.update_D(torch.from_numpy(p.D_seq[s]).cuda())
        g.pcg(b, rtol=p.rtol)  # warm-up (graph capture)
        _, rep = g.pcg(b, rtol=p.rtol)
        print(json.dumps(dict(smoother=name, system=s, iterations=rep["iterations"], solve_ms=rep["solve_ms"],
                              ms_per_iteration=rep["solve_ms"] / max(rep["iterations"], 1))), flush=True)
    g.close()
