"""Interior-point outer loop (Algorithm 1), host driver
paper_2505_18576_b200/ipm.py.  CPU tests pin the driver to things other than itself: the analytic KKT points
of 1-dof problems (SPEC.md ipm examples), the 4x4 Newton system of PAPER.md eq:4x4Newton solved densely, and
the equality-constrained QP on the active set the IP run identifies (an independent dense KKT solve).  The GPU
test runs the whole IP loop with the AMGF-PCG path and with the oracle and requires identical trajectories.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import amgf_gen as gen
from paper_2505_18576_b200 import ipm


class DenseSolver:
    """Reference linear solver for the reduced system (dense LU of K + J^T D J)."""

    def __init__(self, P):
        self.P = P

    def set_D(self, D):
        self.A = (self.P.K + self.P.J.T @ sp.diags(D) @ self.P.J).toarray()

    def solve(self, b, rtol):
        return np.linalg.solve(self.A, b), dict(iterations=1, converged=True)


class OracleSolver:
    """The CPU oracle as the IP driver's linear solver (a fresh oracle hierarchy per Newton step)."""

    def __init__(self, oracle_lib, p, **cfg):
        self.lib, self.p, self.cfg = oracle_lib, p, cfg

    def set_D(self, D):
        self.o = self.lib.Oracle.from_problem(self.p, D=D, **self.cfg)

    def solve(self, b, rtol):
        return self.o.pcg(b, rtol=rtol)

    def matvec_K(self, x):
        """K x in the contract's row-chain order (C2), as the GPU's amgf_spmv_K."""
        return self.lib.bsr_spmv(self.p.K_ptr, self.p.K_col, self.p.K_val, x, 3, 3)


def one_dof(g0):
    # min 1/2 u^2 - 2u  s.t.  g0 - u >= 0   (embedded as dof 0 of one 3-dof node; dofs 1, 2 decoupled)
    return ipm.IPProblem([0, 1], [0], np.eye(3).ravel(), [2.0, 0.0, 0.0], [0, 1], [0], [-1.0], [g0], [1.0],
                         np.ones(3))


@pytest.mark.parametrize("g0,ustar,lamstar", [(1.0, 1.0, -1.0), (10.0, 2.0, 0.0)])
def test_one_dof_kkt(g0, ustar, lamstar):
    """SPEC.md ipm examples: active constraint u* = 1 with multiplier 1; inactive u* = 2 with multiplier -> 0
    (lambda = -M_s z here: r_s = -lambda - M_s z)."""
    P = one_dof(g0)
    u, s, lam, z, recs, status = ipm.solve(P, DenseSolver(P))
    assert status == "converged"
    assert abs(u[0] - ustar) < 1e-6 and abs(lam[0] - lamstar) < 1e-6
    assert np.all(s > 0) and np.all(z > 0)
    assert recs[0].alpha_p > 0


def test_reduced_system_matches_4x4_newton():
    """The reduced system gives the u-block of the full Newton system eq:4x4Newton, and the
    recovered s^, lambda^, z^ satisfy all four block rows."""
    p = gen.generate(2, matching=False, e_max=[4.0], seed=3)
    P = ipm.IPProblem.from_generated(p)
    rng = np.random.default_rng(0)
    n, m = P.n, P.m
    u = 1e-3 * rng.standard_normal(n)
    s = 0.1 + rng.random(m)
    z = 0.1 + rng.random(m)
    lam = rng.standard_normal(m)
    mu = 0.05
    r_u, r_s, r_l, r_z = ipm.residuals(P, u, s, lam, z, mu)
    K, J, Ms = P.K.toarray(), P.J.toarray(), np.diag(P.Ms)
    Z = np.zeros
    big = np.block([[K, Z((n, m)), J.T, Z((n, m))],
                    [Z((m, n)), Z((m, m)), -np.eye(m), -Ms],
                    [J, -np.eye(m), Z((m, m)), Z((m, m))],
                    [Z((m, n)), np.diag(z), Z((m, m)), np.diag(s)]])
    sol = np.linalg.solve(big, -np.concatenate([r_u, r_s, r_l, r_z]))
    D = P.Ms * z / s
    b_u, b_s, b_l = -r_u, -(r_s + P.Ms * r_z / s), -r_l
    b = b_u + P.J.T @ (D * b_l + b_s)
    du = np.linalg.solve((P.K + P.J.T @ sp.diags(D) @ P.J).toarray(), b)
    assert np.linalg.norm(du - sol[:n]) <= 1e-8 * np.linalg.norm(sol[:n])
    ds = P.J @ du + r_l
    dl = D * ds - b_s
    dz = -(r_z + z * ds) / s
    rec = np.concatenate([du, ds, dl, dz])
    assert np.linalg.norm(big @ rec + np.concatenate([r_u, r_s, r_l, r_z])) <= 1e-9 * np.linalg.norm(big @ rec)


def test_fraction_to_boundary():
    assert ipm.fraction_to_boundary(np.array([1.0]), np.array([-1.0]), 0.99) == pytest.approx(0.99)
    assert ipm.fraction_to_boundary(np.array([1.0, 2.0]), np.array([1.0, 0.0]), 0.99) == 1.0


@pytest.fixture(scope="module")
def cfg0_run(oracle_lib):
    p = gen.config(0)
    P = ipm.IPProblem.from_generated(p)
    return p, P, ipm.solve(P, OracleSolver(oracle_lib, p), ipm.IPOptions(tol_ip=1e-9))


def test_two_block_ip_converges_to_the_contact_solution(cfg0_run):
    """cfg 0 two-block contact: the IP loop with AMGF-PCG (oracle) solves converges; the KKT conditions are
    re-evaluated independently, and u equals the solution of the equality-constrained QP on the active set
    (dense KKT solve), within the IP tolerance."""
    p, P, (u, s, lam, z, recs, status) = cfg0_run
    assert status == "converged" and 3 <= len(recs) <= 60
    g = P.gap(u)
    assert g.min() > -1e-8                                  # feasible
    assert np.all(s > 0) and np.all(z > 0)
    r_u = P.K @ u - P.f + P.J.T @ lam
    assert np.sqrt(r_u @ (r_u / P.Mu)) < 1e-8
    assert np.abs(z * s).max() < 10 * 1e-9                 # complementarity at mu -> tol/11
    active = -lam > 1e-3 * np.abs(lam).max()
    assert active.sum() > 0.5 * P.m                          # pressed together: most constraints active
    Ja = P.J[np.nonzero(active)[0]]
    na = Ja.shape[0]
    kkt = sp.bmat([[P.K, Ja.T], [Ja, None]]).tocsc()
    ref = sp.linalg.spsolve(kkt, np.concatenate([P.f, -P.g0[active]]))
    # the IP iterate keeps gaps s ~ mu / z on the active set (barrier): u differs from the exact-contact QP by
    # about max(s) / |u| relatively
    assert np.linalg.norm(u - ref[:P.n]) <= 10 * s[active].max() / 0.01 * np.linalg.norm(ref[:P.n])
    assert np.all(ref[P.n:] <= 1e-12 * np.abs(ref[P.n:]).max() + 0)  # contact pressure: multipliers <= 0
    assert na == active.sum()


def test_ip_pcg_counts_recorded(cfg0_run):
    """Every Newton step records its AMGF-PCG iteration count and the D range (the paper's k_AMGF^avg,
    PAPER.md:622); the barrier parameter never increases."""
    _, _, (u, s, lam, z, recs, status) = cfg0_run
    assert all(r.pcg_iterations > 0 for r in recs)
    mus = [r.mu for r in recs]
    assert all(b <= a for a, b in zip(mus, mus[1:]))
    assert all(r.D_min > 0 for r in recs)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [None, 0])
def test_ip_trajectory_gpu_equals_oracle(oracle_lib, cfg):
    """The whole IP loop driven by the GPU's AMGF-PCG (one handle, amgf_update_D per Newton step) follows the
    oracle-driven trajectory bit for bit: same PCG iteration counts, step lengths, barrier parameters, and the
    same final displacement."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required")
    p = gen.generate(3, matching=False, e_max=[4.0], seed=5) if cfg is None else gen.config(cfg)
    kw = dict(coarsest_size=16) if cfg is None else {}
    P = ipm.IPProblem.from_generated(p)
    uo, so, lo, zo, ro, sto = ipm.solve(P, OracleSolver(oracle_lib, p, **kw))
    ug, sg, lg, zg, rg, stg = ipm.solve(P, ipm.AmgfSolver(p, config=kw))
    assert sto == stg == "converged"
    assert [(r.pcg_iterations, r.alpha_p, r.alpha_d, r.mu) for r in rg] == \
           [(r.pcg_iterations, r.alpha_p, r.alpha_d, r.mu) for r in ro]
    assert np.array_equal(ug, uo) and np.array_equal(lg, lo) and np.array_equal(zg, zo)
