"""SURVEY 8(f) f2 / PAPER.md:351-372 (Fig. amgvsamgf): PCG iterations of AMG-only vs AMGF preconditioning as the
log-barrier diagonal D stiffens, on the GPU path.  D_k = 10^(e * xi_k) with the config's fixed xi_k, e swept.
Prints one JSON line per (config, e)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402


def main(cfgs=(1, 2), exps=(0, 2, 4, 6, 8, 10, 12), max_it=2000):
    for cfg in cfgs:
        p = amgf_gen.config(cfg)
        xi = np.log10(p.D) / max(p.meta["e_max"][0], 1e-300)
        g = AMGF.from_problem(p)
        b = torch.from_numpy(p.b).cuda()
        for e in exps:
            D = 10.0 ** (e * xi)
            g.update_D(D)
            _, ra = g.pcg(b, rtol=p.rtol, max_it=max_it, precond="amgf")
            _, rb = g.pcg(b, rtol=p.rtol, max_it=max_it, precond="amg")
            print(json.dumps(dict(cfg=cfg, n=p.n, D_max=float(D.max()), amgf_iters=ra["iterations"],
                                  amgf_ms=ra["solve_ms"], amg_iters=rb["iterations"], amg_converged=rb["converged"],
                                  amg_ms=rb["solve_ms"])), flush=True)


if __name__ == "__main__":
    main()
