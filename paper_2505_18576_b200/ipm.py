"""Interior-point outer loop (Algorithm 1) producing the systems A u^ = b the AMGF-PCG path
solves: SURVEY.md 8(f) row f3, "the step before the hot path".

Problem (section 3, linear elasticity with linearized gap constraints):
    min_u  E(u) = 1/2 u^T K u - f^T u     s.t.  g(u) = g0 + J u >= 0
with slacks s (c(u, s) = g(u) - s = 0, s >= 0), log-barrier subproblems (eq:logbaroptproblem)
and the primal-dual residuals of eq:optConditionsPrimalDual:
    r_u = K u - f + J^T lambda,  r_s = -lambda - M_s z,  r_lambda = g(u) - s,  r_z(mu) = z * s - mu.
Each Newton step eliminates z^ and s^, lambda^ to the reduced SPD system
    A u^ = b,  A = K + J^T D J,  D = diag(M_s z / s),  b = b_u + J^T (D b_lambda + b_s),
with b_u = -r_u, b_s = -(r_s + M_s s^{-1} r_z), b_lambda = -r_lambda, solved by the AMGF-PCG path
(amgf_update_D + amgf_pcg_solve on the GPU).  The search direction is recovered (s^ = J u^ + r_lambda,
lambda^ = D s^ - b_s, z^ = -s^{-1}(r_z + z s^)), steps are limited by the fraction-to-boundary rule and a
filter line search (the method of Waechter-Biegler), and mu decreases once the subproblem error
is below kappa_eps mu (kappa_eps = 10, s_max = 100).  Constants the paper leaves open
(mu0, the mu update, the filter constants, the e_opt scaling) follow SPEC.md's ipm module; R20.

Host orchestration only (numpy vectors of size n and m, one K*u product per iteration); every linear solve is
the GPU's.  The linear solver is passed in (`solver.set_D(D)`, `solver.solve(b, rtol) -> (u, info)`), so the
same driver runs on the GPU path (AmgfSolver) and, in the tests, on the CPU oracle for a bitwise comparison of
whole IP trajectories.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class IPOptions:
    tol_ip: float = 1e-6          # e_opt termination (SPEC.md ipm defaults, section 4 uses 1e-6)
    tol_pcg: float = 1e-10        # PCG relative preconditioned residual
    mu0: float = 1e-1
    kappa_eps: float = 10.0       # tol^(mu) = kappa_eps mu
    s_max: float = 100.0          # optimality-error scaling
    kappa_mu: float = 0.2
    theta_mu: float = 1.5
    max_iter: int = 200
    s_floor: float = 1e-4
    gamma_theta: float = 1e-5     # filter constants (Waechter-Biegler)
    gamma_phi: float = 1e-5
    eta_phi: float = 1e-4
    alpha_min: float = 1e-12
    max_pcg: int = 5000


@dataclasses.dataclass
class IPRecord:
    it: int
    mu: float
    e_opt: float
    e_opt_mu: float
    pcg_iterations: int
    alpha_p: float
    alpha_d: float
    D_min: float
    D_max: float


class IPError(RuntimeError):
    pass


class IPProblem:
    """min 1/2 u^T K u - f^T u  s.t.  g0 + J u >= 0  (K: 3x3 BSR arrays; J: CSR m x n)."""

    def __init__(self, K_ptr, K_col, K_val, f, J_ptr, J_col, J_val, g0, Ms, Mu):
        import scipy.sparse as sp
        self.K_ptr, self.K_col = np.asarray(K_ptr), np.asarray(K_col)
        self.K_val = np.asarray(K_val, dtype=np.float64)
        self.n = 3 * (len(K_ptr) - 1)
        self.m = len(J_ptr) - 1
        self.J = sp.csr_matrix((np.asarray(J_val, dtype=np.float64), np.asarray(J_col), np.asarray(J_ptr)),
                               shape=(self.m, self.n))
        self.f = np.asarray(f, dtype=np.float64)
        self.g0 = np.asarray(g0, dtype=np.float64)
        self.Ms = np.asarray(Ms, dtype=np.float64)
        self.Mu = np.asarray(Mu, dtype=np.float64)
        self._K = None

    @property
    def K(self):
        """K as a scipy CSR matrix (host reference products; the driver uses the solver's K x when it has one)."""
        if self._K is None:
            import scipy.sparse as sp
            self._K = sp.bsr_matrix((self.K_val.reshape(-1, 3, 3), self.K_col, self.K_ptr),
                                    shape=(self.n, self.n)).tocsr()
        return self._K

    @classmethod
    def from_generated(cls, p):
        import amgf_gen
        g0, Ms, Mu = amgf_gen.ip_data(p)
        return cls(p.K_ptr, p.K_col, p.K_val, p.b, p.J_ptr, p.J_col, p.J_val, g0, Ms, Mu)

    def gap(self, u):
        return self.g0 + self.J @ u


def residuals(P: IPProblem, u, s, lam, z, mu, Ku=None):
    """eq:optConditionsPrimalDual; Ku = K u if already computed."""
    r_u = (P.K @ u if Ku is None else Ku) - P.f + P.J.T @ lam
    r_s = -lam - P.Ms * z
    r_l = P.gap(u) - s
    r_z = z * s - mu
    return r_u, r_s, r_l, r_z


def optimality_error(P: IPProblem, res, lam, z, s_max):
    """e_opt with the IPOPT-style scale max(s_max, (|lambda|_1 + |z|_1)/m) / s_max of
    s_max = 100 (SPEC.md ipm design decision; the paper gives s_max but not the formula)."""
    r_u, r_s, r_l, r_z = res
    m = max(P.m, 1)
    scale = max(s_max, (np.abs(lam).sum() + np.abs(z).sum()) / m) / s_max
    e = max(math.sqrt(float(r_u @ (r_u / P.Mu))), math.sqrt(float(r_s @ (r_s / P.Ms))) if P.m else 0.0,
            float(np.abs(r_l).max()) if P.m else 0.0)
    return max(e / scale, float(np.abs(r_z).max()) / scale if P.m else 0.0)


def fraction_to_boundary(v, dv, tau):
    """Largest alpha in (0, 1] with v + alpha dv >= (1 - tau) v (v > 0)."""
    neg = dv < 0
    if not np.any(neg):
        return 1.0
    return float(min(1.0, np.min(-tau * v[neg] / dv[neg])))


def barrier_log(P: IPProblem, s, mu):
    return -mu * float(P.Ms @ np.log(s))


def solve(P: IPProblem, solver, opts: IPOptions | None = None, u0=None, log=None):
    """Algorithm 1.  Returns (u, s, lambda, z, records, status)."""
    o = opts or IPOptions()
    n, m = P.n, P.m
    Kmul = getattr(solver, "matvec_K", None) or (lambda x: P.K @ x)   # K x (the solver's, C2 chains)
    u = np.zeros(n) if u0 is None else np.array(u0, dtype=np.float64)
    mu = o.mu0
    s = np.maximum(P.gap(u), o.s_floor)
    z = mu / s
    lam = -P.Ms * z                       # r_s = 0 at the start
    filt: list[tuple[float, float]] = []
    recs: list[IPRecord] = []
    theta_min = 1e-4 * max(1.0, float(np.abs(P.gap(u) - s).sum()))
    status = "max_iter"
    Ku = Kmul(u)
    for it in range(1, o.max_iter + 1):
        res = residuals(P, u, s, lam, z, 0.0, Ku)
        e_opt = optimality_error(P, res, lam, z, o.s_max)
        if e_opt < o.tol_ip:
            status = "converged"
            break
        res_mu = residuals(P, u, s, lam, z, mu, Ku)
        e_mu = optimality_error(P, res_mu, lam, z, o.s_max)
        while e_mu < o.kappa_eps * mu and mu > o.tol_ip / 11.0:   # inner loop done: decrease mu, reset filter
            mu = max(o.tol_ip / 11.0, min(o.kappa_mu * mu, mu ** o.theta_mu))
            filt = []
            res_mu = residuals(P, u, s, lam, z, mu, Ku)
            e_mu = optimality_error(P, res_mu, lam, z, o.s_max)
        r_u, r_s, r_l, r_z = res_mu
        # ---- reduced Newton system
        D = P.Ms * z / s
        b_u, b_s, b_l = -r_u, -(r_s + P.Ms * r_z / s), -r_l
        b = b_u + P.J.T @ (D * b_l + b_s)
        solver.set_D(D)
        du, info = solver.solve(b, o.tol_pcg)
        if not info.get("converged", True):
            raise IPError(f"PCG did not converge at IP iteration {it}: {info}")
        ds = P.J @ du + r_l
        dl = D * ds - b_s
        dz = -(r_z + z * ds) / s
        # ---- step lengths: fraction to the boundary, then the filter line search on the primal step
        tau = max(0.99, 1.0 - mu)
        a_max = fraction_to_boundary(s, ds, tau)
        a_d = fraction_to_boundary(z, dz, tau)
        theta = float(np.abs(r_l).sum())
        # E along the step is a quadratic: E(u + a du) = E(u) + a (Ku - f).du + a^2/2 du.K du (one K du product)
        Kdu = Kmul(du)
        gE = float((Ku - P.f) @ du)
        cE = 0.5 * float(du @ Kdu)
        phi = barrier_log(P, s, mu)                       # phi relative to E(u)
        grad_phi_d = gE - mu * float((P.Ms / s) @ ds)
        alpha = a_max
        while True:
            st = s + alpha * ds
            theta_t = float(np.abs(P.gap(u + alpha * du) - st).sum())
            phi_t = alpha * gE + alpha * alpha * cE + barrier_log(P, st, mu)
            ok_filter = all(theta_t < tf or phi_t < pf for tf, pf in filt)
            f_type = theta <= theta_min and grad_phi_d < 0   # switching condition: an Armijo (f-type) step
            if f_type:
                accept = phi_t <= phi + o.eta_phi * alpha * grad_phi_d
            else:
                accept = theta_t <= (1 - o.gamma_theta) * theta or phi_t <= phi - o.gamma_phi * theta
            if ok_filter and accept:
                if not f_type:
                    filt.append(((1 - o.gamma_theta) * theta, phi - o.gamma_phi * theta))
                break
            alpha *= 0.5
            if alpha < o.alpha_min:
                raise IPError(f"line search failed at IP iteration {it}")
        # filter entries are relative to E at the accepted point: shift them by the change in E
        dE = alpha * gE + alpha * alpha * cE
        filt = [(tf, pf - dE) for tf, pf in filt]
        Ku = Kmul(u + alpha * du)
        u, s, lam = u + alpha * du, s + alpha * ds, lam + alpha * dl
        z = z + a_d * dz
        recs.append(IPRecord(it, mu, e_opt, e_mu, int(info.get("iterations", 0)), alpha, a_d,
                             float(D.min()) if m else 0.0, float(D.max()) if m else 0.0))
        if log:
            log(recs[-1])
    return u, s, lam, z, recs, status


class AmgfSolver:
    """The GPU path as the IP driver's linear solver: one handle, amgf_update_D per Newton step (numeric
    re-setup of S = K + J^T D J), amgf_pcg_solve with the AMGF preconditioner, and amgf_spmv_K for K x."""

    def __init__(self, p, config=None, precond="amgf"):
        from .amgf import AMGF
        self.p = p
        self.precond = precond
        self.h = AMGF.from_problem(p, config=config)

    def set_D(self, D):
        self.h.update_D(np.ascontiguousarray(D))

    def solve(self, b, rtol):
        x, info = self.h.pcg(np.ascontiguousarray(b), rtol=rtol, max_it=5000, precond=self.precond)
        return x.cpu().numpy(), info

    def matvec_K(self, x):
        return self.h.spmv_K(np.ascontiguousarray(x)).cpu().numpy()
