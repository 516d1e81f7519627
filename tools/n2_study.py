"""Controlled iteration study (north star "mesh-independent iteration counts"):
mesh N in {8, 16, 32, 64} (the cfg 0-3 geometries) x interface {matching, offset (node-on-segment)} x
D_max in {1, 1e4, 1e8, 1e12} (D log-uniform in [1, D_max], the same xi per (N, interface)), rtol 1e-8, on the GPU:
AMGF-PCG and AMG-only PCG iterations, kappa(M S) from the PCG Ritz values, the contact-free AMG-PCG count and
beta = kappa(B K) (Ritz), and the paper's practical bound k_AMGF <= k_AMG(contact-free) sqrt(2(beta+3)/beta)
(remark upper_bound_estimate).  Then the cfg 4 decomposition: N = 96 offset with and
without the E = 1e3 inclusion, and the inclusion at N = 32, 48, 64, at rtol 1e-8 and 1e-10.
One JSON line per case.  The oracle confirms the AMGF counts separately (tools/n2_oracle.py)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402

case = amgf_gen.study_case


def ritz(alpha, beta):
    k = len(alpha)
    T = np.zeros((k, k))
    for j in range(k):
        T[j, j] = 1.0 / alpha[j] + (beta[j - 1] / alpha[j - 1] if j > 0 else 0.0)
        if j + 1 < k:
            T[j, j + 1] = T[j + 1, j] = np.sqrt(beta[j]) / alpha[j]
    ev = np.linalg.eigvalsh(T)
    return float(ev[0]), float(ev[-1])


def run(g, b, rtol, precond, max_it=5000):
    _, rep = g.pcg(b, rtol=rtol, precond=precond, max_it=max_it)
    k = rep["iterations"]
    lo, hi = ritz(*g.history(min(k, 2000))) if k > 0 else (1.0, 1.0)
    return k, rep["converged"], lo, hi, rep["solve_ms"]


def study(p, rtols=(1e-8,), amg=True, tag=None):
    b = torch.from_numpy(p.b).cuda()
    out = []
    # contact-free reference: AMG-PCG on K (no constraints: J empty, I_c empty)
    g0 = AMGF(p.nodes, p.K_ptr, p.K_col, p.K_val, np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0),
              np.zeros(0), None, p.B_nns)
    g = AMGF.from_problem(p, D=p.D_seq[0])
    for rtol in rtols:
        k0, _, lo0, hi0, _ = run(g0, b, rtol, "amg")
        beta = hi0 / lo0
        kb = k0 * np.sqrt(2 * (beta + 3) / beta)
        for s, e in enumerate(p.meta["e_max"]):
            g.update_D(p.D_seq[s])
            k, conv, lo, hi, ms = run(g, b, rtol, "amgf")
            rec = dict(case=tag or p.name, N=p.N, n=p.n, matching=bool(p.meta["matching"]),
                       inclusion=bool(p.meta["inclusion"]), rtol=rtol, D_max=10.0 ** e, k_amgf=k, converged=conv,
                       solve_ms=ms, kappa_MS=hi / lo, lambda_max_MS=hi, lambda_min_MS=lo,
                       k_amg_contact_free=k0, beta=beta, k_bound=kb, within_bound=bool(k <= kb),
                       kappa_bound=2 * (beta + 3), levels=[L["nodes"] * L["b"] for L in g.levels])
            if amg:
                ka, ca, _, _, _ = run(g, b, rtol, "amg", max_it=2000)
                rec.update(k_amg=ka, amg_converged=ca)
            print(json.dumps(rec), flush=True)
            out.append(rec)
    g.close()
    g0.close()
    return out


if __name__ == "__main__":
    part = sys.argv[1] if len(sys.argv) > 1 else "grid"
    if part == "grid":
        for N in (8, 16, 32, 64):
            for matching in (True, False):
                study(case(N, matching))
    else:  # the cfg 4 decomposition
        for N, inc in ((32, True), (48, True), (64, True), (96, False), (96, True)):
            study(case(N, False, inclusion=inc), rtols=(1e-8, 1e-10), amg=False)
        p = amgf_gen.config(4)
        study(p, rtols=(1e-8, 1e-10), amg=False, tag="cfg4")
