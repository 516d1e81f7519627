"""Interior-point runs (Algorithm 1, paper_2505_18576_b200/ipm.py) on the GPU path: for each config the number
of IP iterations, the AMGF-PCG iterations per Newton step (the paper's k_IP / k_AMGF^avg),
the D range the IP produces, and the time split; one JSON line per config.  Usage: python tools/ip_run.py 0 1 2 3"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import ipm  # noqa: E402

tol_ip = float(os.environ.get("IP_TOL", "1e-6"))
for cfg in [int(a) for a in sys.argv[1:]] or [0, 1, 2]:
    p = amgf_gen.config(cfg)
    P = ipm.IPProblem.from_generated(p)
    solver = ipm.AmgfSolver(p)
    t_solve = [0.0]
    base_solve = solver.solve

    def timed(b, rtol):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = base_solve(b, rtol)
        t_solve[0] += time.perf_counter() - t
        return r
    solver.solve = timed
    t0 = time.perf_counter()
    u, s, lam, z, recs, status = ipm.solve(P, solver, ipm.IPOptions(tol_ip=tol_ip))
    wall = time.perf_counter() - t0
    its = [r.pcg_iterations for r in recs]
    print(json.dumps(dict(cfg=cfg, n=p.n, m=p.m, status=status, tol_ip=tol_ip, ip_iterations=len(recs),
                          pcg_iterations=its, pcg_avg=float(np.mean(its)), pcg_max=int(max(its)),
                          D_min=min(r.D_min for r in recs), D_max=max(r.D_max for r in recs),
                          mu_final=recs[-1].mu, e_opt_final=recs[-1].e_opt, wall_s=wall,
                          gpu_solve_s=t_solve[0], min_gap=float(P.gap(u).min()),
                          contact_force=float(-lam.sum()))), flush=True)
