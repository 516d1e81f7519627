"""Seeded synthetic inputs for the AMGF-PCG solve path (shared by oracle and CUDA path).

This module produces the *inputs* of the method only: the stiffness matrix K,
the gap Jacobian J, the log-barrier diagonal D, the right-hand side b, nodal
coordinates, the rigid-body near-null space and the contact-dof ordering Z.
It holds none of the method's arithmetic (no S = K + J^T D J, no AMG, no
filter, no PCG); both `oracle/` and the CUDA path consume its arrays
byte-identically.

Workload recipe (BASELINE.json configs 0-4):
  * two stacked unit cubes, lower [0,1]^3 and upper [0,1]^2 x [1,2], each
    N^3 trilinear (Q1) hexahedra, h = 1/N, 3D linear elasticity E=1, nu=0.3
    (PAPER.md:303 uses Q1 hexes on a two-block geometry; the BASELINE configs
    fix equal cubes), element stiffness by 2x2x2 Gauss-Legendre.
  * Dirichlet: lower z=0 face clamped, upper z=2 face displaced (0,0,-0.01);
    Dirichlet dofs are kept as identity rows, removed structurally from the
    other rows, the lift -K_FD g_D goes into b.
  * J: one row per upper-body bottom-face node (non-mortar side),
    +1 at its z-dof; matching configs put -1 at the coincident lower top-face
    z-dof, non-matching configs (lateral shift U(-h/2,h/2)) put the 4 bilinear
    node-on-segment weights -w at the lower cell's z-dofs (PAPER.md:52-66,
    SURVEY.md A10). Zero weights are stored.
  * D_k = 10^(e_max * xi_k), xi_k ~ U[0,1) from SplitMix64(seed = cfg index):
    log-uniform in [1, 10^e_max] (BASELINE.json configs).
  * cfg 4: elements of the upper body inside a seeded box of 10% volume get
    E = 1e3.
  * Z: the structurally nonzero columns of J,
    listed in interface-lattice order (face row j, face column i, body) - the
    column order of the embedding P; reading R2.
"""
from __future__ import annotations

import dataclasses
import numpy as np

MASK64 = (1 << 64) - 1


class SplitMix64:
    """SplitMix64 stream; u = (x >> 11) * 2^-53 in [0, 1)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)


@dataclasses.dataclass
class Problem:
    name: str
    N: int
    nodes: int
    n: int
    m: int
    K_ptr: np.ndarray   # int32 [nodes+1]  block-row pointers (3x3 blocks)
    K_col: np.ndarray   # int32 [nnzb]     block columns, ascending per row
    K_val: np.ndarray   # float64 [nnzb, 9] row-major 3x3 blocks
    J_ptr: np.ndarray   # int32 [m+1]
    J_col: np.ndarray   # int32 [nnz(J)]  scalar dof columns, ascending
    J_val: np.ndarray   # float64 [nnz(J)]
    D: np.ndarray       # float64 [m]  (the first system of D_seq)
    D_seq: np.ndarray   # float64 [n_systems, m]
    b: np.ndarray       # float64 [n]
    coords: np.ndarray  # float64 [nodes, 3]
    B_nns: np.ndarray   # float64 [n, 6] row-major rigid-body modes
    Z: np.ndarray       # int32 [n_c] contact dofs in lattice (elimination) order
    rtol: float
    dirichlet: np.ndarray  # bool [nodes]
    meta: dict

    def nbytes(self) -> int:
        return sum(v.nbytes for v in dataclasses.asdict(self).values() if isinstance(v, np.ndarray))


def hex8_stiffness_unit(nu: float) -> np.ndarray:
    """24x24 stiffness of the unit cube Q1 element for E=1 (scales as E*h in 3D)."""
    lam = nu / ((1 + nu) * (1 - 2 * nu))
    mu = 1.0 / (2 * (1 + nu))
    C = np.zeros((6, 6))
    C[:3, :3] = lam
    C[np.arange(3), np.arange(3)] += 2 * mu
    C[3, 3] = C[4, 4] = C[5, 5] = mu
    g = 1.0 / np.sqrt(3.0)
    corners = [(a & 1, (a >> 1) & 1, (a >> 2) & 1) for a in range(8)]
    Ke = np.zeros((24, 24))
    for gz in (-g, g):
        for gy in (-g, g):
            for gx in (-g, g):
                B = np.zeros((6, 24))
                for a, (cx, cy, cz) in enumerate(corners):
                    sx, sy, sz = 2 * cx - 1, 2 * cy - 1, 2 * cz - 1
                    # dN/dxi on [-1,1]^3, then * 2/h with h = 1
                    dx = sx * (1 + sy * gy) * (1 + sz * gz) / 8 * 2
                    dy = sy * (1 + sx * gx) * (1 + sz * gz) / 8 * 2
                    dz = sz * (1 + sx * gx) * (1 + sy * gy) / 8 * 2
                    c = 3 * a
                    B[0, c] = dx
                    B[1, c + 1] = dy
                    B[2, c + 2] = dz
                    B[3, c + 1] = dz
                    B[3, c + 2] = dy
                    B[4, c] = dz
                    B[4, c + 2] = dx
                    B[5, c] = dy
                    B[5, c + 1] = dx
                Ke += B.T @ C @ B * (0.5 ** 3)   # det J = (h/2)^3, weights 1
    return 0.5 * (Ke + Ke.T)


def _assemble_body(N: int, Ke: np.ndarray, E_elem: np.ndarray) -> np.ndarray:
    """Stencil-form assembly: returns Kb[nn, 27, 3, 3] (neighbour d = (dz,dy,dx) lexicographic)."""
    h = 1.0 / N
    n1 = N + 1
    nn = n1 ** 3
    k, j, i = np.meshgrid(np.arange(n1), np.arange(n1), np.arange(n1), indexing="ij")
    i = i.ravel(); j = j.ravel(); k = k.ravel()
    Kb = np.zeros((nn, 27, 3, 3))
    for oz in (-1, 0):
        for oy in (-1, 0):
            for ox in (-1, 0):
                ex, ey, ez = i + ox, j + oy, k + oz
                valid = (ex >= 0) & (ex < N) & (ey >= 0) & (ey < N) & (ez >= 0) & (ez < N)
                idx = np.nonzero(valid)[0]
                scale = E_elem[ez[idx], ey[idx], ex[idx]] * h
                a = (-ox) + 2 * (-oy) + 4 * (-oz)
                ax, ay, az = -ox, -oy, -oz
                for bcor in range(8):
                    bx, by, bz = bcor & 1, (bcor >> 1) & 1, (bcor >> 2) & 1
                    d = (bz - az + 1) * 9 + (by - ay + 1) * 3 + (bx - ax + 1)
                    blk = Ke[3 * a:3 * a + 3, 3 * bcor:3 * bcor + 3]
                    Kb[idx, d] += scale[:, None, None] * blk[None]
    return Kb


CONFIGS = {
    # name: (N, matching, e_max list, inclusion, rtol)
    0: dict(N=8, matching=True, e_max=[8.0], inclusion=False, rtol=1e-8),
    1: dict(N=16, matching=True, e_max=[10.0], inclusion=False, rtol=1e-8),
    2: dict(N=32, matching=False, e_max=[12.0], inclusion=False, rtol=1e-8),
    3: dict(N=64, matching=False, e_max=[2.0 + 10.0 * s / 9.0 for s in range(10)],
            inclusion=False, rtol=1e-8),
    4: dict(N=96, matching=False, e_max=[12.0], inclusion=True, rtol=1e-10),
}


def generate(N: int, matching: bool = True, e_max=(8.0,), seed: int = 0,
             inclusion: bool = False, rtol: float = 1e-8, name: str | None = None,
             nu: float = 0.3) -> Problem:
    n1 = N + 1
    nn = n1 ** 3
    nodes = 2 * nn
    n = 3 * nodes
    m = n1 * n1
    h = 1.0 / N
    rng = SplitMix64(seed)
    u_shift = (rng.uniform(), rng.uniform())
    u_incl = (rng.uniform(), rng.uniform(), rng.uniform())
    xi = np.array([rng.uniform() for _ in range(m)])
    sx, sy = (0.0, 0.0) if matching else ((u_shift[0] - 0.5) * h, (u_shift[1] - 0.5) * h)

    Ke = hex8_stiffness_unit(nu)
    E_low = np.ones((N, N, N))
    E_up = np.ones((N, N, N))
    if inclusion:
        side = 0.1 ** (1.0 / 3.0)
        org = [u * (1.0 - side) for u in u_incl]
        c = (np.arange(N) + 0.5) * h
        inz = (c >= org[2]) & (c <= org[2] + side)
        iny = (c >= org[1]) & (c <= org[1] + side)
        inx = (c >= org[0]) & (c <= org[0] + side)
        mask = inz[:, None, None] & iny[None, :, None] & inx[None, None, :]
        E_up[mask] = 1e3
    Kb = np.concatenate([_assemble_body(N, Ke, E_low), _assemble_body(N, Ke, E_up)])

    # node lattice indices
    k, j, i = np.meshgrid(np.arange(n1), np.arange(n1), np.arange(n1), indexing="ij")
    i = np.tile(i.ravel(), 2); j = np.tile(j.ravel(), 2); k = np.tile(k.ravel(), 2)
    body = np.repeat(np.arange(2), nn)
    coords = np.stack([i * h + body * sx, j * h + body * sy, k * h + body], axis=1).astype(np.float64)
    dirichlet = ((body == 0) & (k == 0)) | ((body == 1) & (k == N))
    gD = np.zeros((nodes, 3))
    gD[(body == 1) & (k == N), 2] = -0.01

    # neighbour ids per stencil slot
    d = np.arange(27)
    dz, dy, dx = d // 9 - 1, (d // 3) % 3 - 1, d % 3 - 1
    ni, nj, nk = i[:, None] + dx, j[:, None] + dy, k[:, None] + dz
    inside = (ni >= 0) & (ni <= N) & (nj >= 0) & (nj <= N) & (nk >= 0) & (nk <= N)
    nbr = body[:, None] * nn + (nk * n1 + nj) * n1 + ni
    nbr = np.where(inside, nbr, -1)

    # lift: b_i = -sum_{j Dirichlet} K_ij g_j on free rows, b_D = g_D
    nbr_dir = inside & dirichlet[np.where(inside, nbr, 0)]
    rows = np.nonzero(nbr_dir.any(axis=1) & ~dirichlet)[0]
    gj = gD[np.where(inside[rows], nbr[rows], 0)] * nbr_dir[rows][:, :, None]   # [r,27,3]
    bvec = np.zeros((nodes, 3))
    bvec[rows] = -np.einsum("sdab,sdb->sa", Kb[rows], gj)
    bvec[dirichlet] = gD[dirichlet]

    # structural pattern: free rows keep in-grid free neighbours (+ self); Dirichlet rows keep self = I3
    is_self = d[None, :] == 13
    keep = inside & ~nbr_dir
    keep = np.where(dirichlet[:, None], is_self & np.ones_like(inside), keep)
    Kb[dirichlet, 13] = np.eye(3)
    counts = keep.sum(axis=1)
    K_ptr = np.zeros(nodes + 1, dtype=np.int64)
    np.cumsum(counts, out=K_ptr[1:])
    K_col = nbr[keep].astype(np.int32)
    K_val = Kb[keep].reshape(-1, 9).copy()

    # gap Jacobian rows: upper-body bottom-face nodes, ordered j then i
    up0 = nn  # upper body offset, k = 0
    rows_cols, rows_vals = [], []
    fj, fi = np.meshgrid(np.arange(n1), np.arange(n1), indexing="ij")
    fj = fj.ravel(); fi = fi.ravel()
    nm_node = up0 + fj * n1 + fi
    low_top = lambda ii, jj: (N * n1 + jj) * n1 + ii
    if matching:
        cols = np.stack([3 * low_top(fi, fj) + 2, 3 * nm_node + 2], axis=1)
        vals = np.stack([-np.ones(m), np.ones(m)], axis=1)
    else:
        x = np.clip(fi * h + sx, 0.0, 1.0)
        y = np.clip(fj * h + sy, 0.0, 1.0)
        cx = np.minimum(np.floor(x / h).astype(np.int64), N - 1)
        cy = np.minimum(np.floor(y / h).astype(np.int64), N - 1)
        xi_ = x / h - cx
        eta = y / h - cy
        w = np.stack([(1 - xi_) * (1 - eta), xi_ * (1 - eta), (1 - xi_) * eta, xi_ * eta], axis=1)
        lc = np.stack([low_top(cx, cy), low_top(cx + 1, cy), low_top(cx, cy + 1), low_top(cx + 1, cy + 1)], axis=1)
        cols = np.concatenate([3 * lc + 2, (3 * nm_node + 2)[:, None]], axis=1)
        vals = np.concatenate([-w, np.ones((m, 1))], axis=1)
    order = np.argsort(cols, axis=1, kind="stable")
    cols = np.take_along_axis(cols, order, axis=1)
    vals = np.take_along_axis(vals, order, axis=1)
    per = cols.shape[1]
    J_ptr = (np.arange(m + 1) * per).astype(np.int32)
    J_col = cols.ravel().astype(np.int32)
    J_val = vals.ravel().astype(np.float64)

    e_list = list(e_max)
    D_seq = np.stack([10.0 ** (e * xi) for e in e_list]).astype(np.float64)

    # rigid-body modes (near-null space), zero on Dirichlet rows
    X = coords[:, 0] - 0.5; Y = coords[:, 1] - 0.5; Zc = coords[:, 2] - 1.0
    B = np.zeros((nodes, 3, 6))
    B[:, 0, 0] = 1; B[:, 1, 1] = 1; B[:, 2, 2] = 1
    B[:, 1, 3] = -Zc; B[:, 2, 3] = Y
    B[:, 0, 4] = Zc; B[:, 2, 4] = -X
    B[:, 0, 5] = -Y; B[:, 1, 5] = X
    B[dirichlet] = 0.0
    B = B.reshape(n, 6)

    # contact dofs in lattice order (face row j, face column i, body lower->upper)
    Zl = np.stack([3 * low_top(fi, fj) + 2, 3 * nm_node + 2], axis=1).ravel().astype(np.int32)

    return Problem(name=name or f"N{N}", N=N, nodes=nodes, n=n, m=m,
                   K_ptr=K_ptr.astype(np.int32), K_col=K_col, K_val=K_val,
                   J_ptr=J_ptr, J_col=J_col, J_val=J_val,
                   D=D_seq[0].copy(), D_seq=D_seq, b=bvec.reshape(n).astype(np.float64),
                   coords=coords, B_nns=np.ascontiguousarray(B), Z=Zl, rtol=rtol,
                   dirichlet=dirichlet,
                   meta=dict(N=N, matching=matching, e_max=e_list, seed=seed,
                             inclusion=inclusion, shift=(sx, sy), nu=nu))


def config(cfg: int) -> Problem:
    c = CONFIGS[cfg]
    return generate(c["N"], matching=c["matching"], e_max=c["e_max"], seed=cfg,
                    inclusion=c["inclusion"], rtol=c["rtol"], name=f"cfg{cfg}")


def with_D(p: Problem, D: np.ndarray) -> Problem:
    q = dataclasses.replace(p)
    q.D = np.ascontiguousarray(D, dtype=np.float64)
    return q


def box_diagonals(p: Problem, e_max: float = 6.0, seed: int = 1000):
    """Bound-constraint diagonals (D_lo, D_up) for the bound-constrained system of Remark boundconstr
    (PAPER.md:271-295): log-barrier Hessians of the box u - u* in [delta_lo, delta_up] on every free dof,
    D = 10^(e_max * xi), xi ~ U[0,1) from SplitMix64(seed), lower diagonal first, dof order; 0 on Dirichlet
    dofs (no bound there).  Inputs only: no method arithmetic."""
    rng = SplitMix64(seed)
    free = np.repeat(~p.dirichlet, 3)
    out = []
    for _ in range(2):
        xi = np.array([rng.uniform() for _ in range(p.n)])
        d = 10.0 ** (e_max * xi)
        d[~free] = 0.0
        out.append(d.astype(np.float64))
    return out[0], out[1]


def ip_data(p: Problem):
    """Interior-point data of the two-block contact problem (section 3; inputs only):
    g0 (m)  gap of each constraint at u = 0: 0, the bodies touch at rest (the top face is pushed down);
    Ms (m)  diagonal lumped boundary mass of the slack space ("diagonal lumped mass-matrix M_s
            associated to s"): the non-mortar face nodes' tributary areas h^2 x (1/2 per boundary axis);
    Mu (n)  lumped volume mass of the displacement space (the M_u^{-1} norm of r_u in e_opt):
            nodal tributary volumes h^3 x (1/2 per boundary axis), per dof."""
    N = p.N
    n1 = N + 1
    h = 1.0 / N
    edge = lambda a: np.where((a == 0) | (a == N), 0.5, 1.0)  # noqa: E731
    fj, fi = np.meshgrid(np.arange(n1), np.arange(n1), indexing="ij")
    Ms = (h * h * edge(fj) * edge(fi)).ravel().astype(np.float64)
    k, j, i = np.meshgrid(np.arange(n1), np.arange(n1), np.arange(n1), indexing="ij")
    vol = (h ** 3 * edge(k) * edge(j) * edge(i)).ravel()
    Mu = np.repeat(np.concatenate([vol, vol]), 3).astype(np.float64)
    return np.zeros(p.m), Ms, Mu


STUDY_E_MAX = [0.0, 4.0, 8.0, 12.0]


def study_case(N: int, matching: bool, inclusion: bool = False) -> Problem:
    """Input of one cell of the iteration study (tools/n2_study.py, profiles/r02_n2_study.md): the cfg geometry
    at N elements per axis and block, matching or offset interface, optional E = 1e3 inclusion, D log-uniform in
    [1, 10^e] for e in STUDY_E_MAX with one xi per (N, interface) from SplitMix64(seed)."""
    seed = 100 + 2 * N + (0 if matching else 1) + (1000 if inclusion else 0)
    return generate(N, matching=matching, e_max=STUDY_E_MAX, seed=seed, inclusion=inclusion,
                    name=f"N{N}{'m' if matching else 'o'}{'i' if inclusion else ''}")
