"""Paper remark upper_bound_estimate (section 4, eq. practical_bound and the Table 1 caption):
k_AMGF <= k_AMG(contact-free) * sqrt(2 (beta + 3) / beta), with beta = kappa(B K) of the contact-free
elasticity operator K preconditioned by one AMG V-cycle, and kappa(M S) <= 2 (beta + 3).

beta and kappa(M S) are estimated from the Ritz values of the PCG runs (the Lanczos matrix built from the
PCG coefficients alpha_k, beta_k, amgf_pcg_history).  The contact-free operator is S with D = 1e-30
(J^T D J below the rounding of K).  One JSON line per (cfg, D_max)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402


def ritz(alpha, beta):
    """Eigenvalues of the CG Lanczos matrix: T_jj = 1/a_j + b_{j-1}/a_{j-1}, T_j,j+1 = sqrt(b_j)/a_j."""
    k = len(alpha)
    T = np.zeros((k, k))
    for j in range(k):
        T[j, j] = 1.0 / alpha[j] + (beta[j - 1] / alpha[j - 1] if j > 0 else 0.0)
        if j + 1 < k:
            T[j, j + 1] = T[j + 1, j] = np.sqrt(beta[j]) / alpha[j]
    return np.linalg.eigvalsh(T)


def run(g, b, rtol, precond):
    _, rep = g.pcg(b, rtol=rtol, precond=precond)
    k = rep["iterations"]
    a, bt = g.history(k)
    ev = ritz(a, bt)
    return k, float(ev[0]), float(ev[-1])


cfgs = [int(c) for c in sys.argv[1:]] or [0, 1, 2]
for cfg in cfgs:
    p = amgf_gen.config(cfg)
    b = torch.from_numpy(p.b).cuda()
    # contact-free reference: AMG-PCG on K (D = 1e-30)
    g0 = AMGF.from_problem(p, D=np.full(p.m, 1e-30))
    k0, lmin0, lmax0 = run(g0, b, p.rtol, "amg")
    beta = lmax0 / lmin0
    bound_k = k0 * np.sqrt(2 * (beta + 3) / beta)
    g0.close()
    g = AMGF.from_problem(p)
    for e in (0, 4, 8, 12):
        rng = np.random.default_rng(cfg)
        xi = rng.random(p.m)
        D = 10.0 ** (e * xi)
        g.update_D(torch.from_numpy(D).cuda())
        k, lmin, lmax = run(g, b, p.rtol, "amgf")
        kappa = lmax / lmin
        print(json.dumps(dict(cfg=cfg, D_max=10.0 ** e, k_amg_contact_free=k0, beta_ritz=beta,
                              k_amgf=k, k_bound=bound_k, k_within_bound=bool(k <= bound_k),
                              kappa_MS_ritz=kappa, kappa_bound=2 * (beta + 3),
                              kappa_within_bound=bool(kappa <= 2 * (beta + 3)),
                              lambda_max_MS_ritz=lmax, lambda_min_MS_ritz=lmin)), flush=True)
    g.close()
