"""Pins of the CPU oracle against the paper and the mathematics (no GPU).

Each test pins one oracle function to something other than itself: closed
forms, dense numpy/scipy linear algebra on tiny systems, the paper's lemmas
(PAPER.md:421-595), and the hand-derived golden examples of tests/golden/.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spl

import amgf_gen as gen

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "spec_examples.json")))
EPS = np.finfo(np.float64).eps


def tiny(N=2, matching=True, e_max=4.0, seed=7):
    return gen.generate(N, matching=matching, e_max=[e_max], seed=seed)


def K_csr(p):
    return sp.bsr_matrix((p.K_val.reshape(-1, 3, 3), p.K_col, p.K_ptr), shape=(p.n, p.n)).tocsr()


def J_csr(p):
    return sp.csr_matrix((p.J_val, p.J_col, p.J_ptr), shape=(p.m, p.n))


def dense_op(f, n):
    return np.stack([f(e) for e in np.eye(n)], axis=1)


# ---------------------------------------------------------------- dot (C14)
def test_dot_exact_on_integers(oracle_lib):
    rng = np.random.default_rng(0)
    for n in (0, 3, 768, 3 * 256 * 300 + 9):
        u = rng.integers(-1000, 1000, n).astype(float)
        v = rng.integers(-1000, 1000, n).astype(float)
        assert oracle_lib.dot(u, v, 3) == float(int(np.dot(u.astype(np.int64), v.astype(np.int64))))


def test_dot_error_bound(oracle_lib):
    rng = np.random.default_rng(1)
    for b in (3, 6):
        n = b * 100003
        u = rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n))
        v = rng.standard_normal(n)
        exact = math.fsum((u * v).tolist())  # products are exact-ish; bound covers them
        got = oracle_lib.dot(u, v, b)
        bound = (b + 8 + 8 + 256) * EPS * np.sum(np.abs(u * v)) * 1.01
        assert abs(got - exact) <= bound


# ----------------------------------------------------- dense Cholesky / TRSV
def test_cholesky_matches_lapack(oracle_lib):
    rng = np.random.default_rng(2)
    X = rng.standard_normal((40, 40))
    A = X @ X.T + 40 * np.eye(40)
    L = oracle_lib.cholesky(A)
    assert np.allclose(np.triu(L, 1), 0)
    assert np.abs(L - np.linalg.cholesky(A)).max() <= 1e-13 * np.abs(L).max()
    assert np.abs(L @ L.T - A).max() <= 1e-13 * np.abs(A).max()
    v = rng.standard_normal(40)
    x = oracle_lib.chol_solve(L, v)
    assert np.abs(x - np.linalg.solve(A, v)).max() <= 1e-12 * np.abs(x).max()


def test_cholesky_not_spd(oracle_lib):
    A = np.array([[1.0, 2.0], [2.0, 1.0]])
    with pytest.raises(oracle_lib.OracleError) as e:
        oracle_lib.cholesky(A)
    assert e.value.code == -4


# ------------------------------------------------------------ golden (SPEC)
def test_golden_spmv(oracle_lib):
    for ex in GOLD["spmv"]:
        A = np.array(ex["A"], float)
        C = sp.csr_matrix(A)
        C.sort_indices()
        # 1x1 blocks, stored zeros dropped
        y = oracle_lib.bsr_spmv(C.indptr, C.indices, C.data, np.array(ex["x"], float), 1, 1)
        assert np.array_equal(y, np.array(ex["y"], float)), ex["cite"]


def _single_node(oracle_lib, Kblk, J=None, D=None, Z=None):
    Kp = np.array([0, 1], np.int32)
    Kc = np.array([0], np.int32)
    Kv = np.asarray(Kblk, float).reshape(1, 9)
    if J is None or len(J) == 0:
        Jp, Jc, Jv, Dv = np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0), np.zeros(0)
    else:
        Jm = sp.csr_matrix(np.array(J, float))
        Jm.sort_indices()
        Jp, Jc, Jv, Dv = Jm.indptr, Jm.indices, Jm.data, np.array(D, float)
    return oracle_lib.Oracle(1, Kp, Kc, Kv, Jp, Jc, Jv, Dv, Z, np.zeros((3, 6)))


def test_golden_jtdj(oracle_lib):
    for ex in GOLD["jtdj"]:
        J = np.zeros((1, 3)); J[0, :2] = ex["J"][0]
        o = _single_node(oracle_lib, np.eye(3), J, ex["D"])
        S = o.get(2, 0).reshape(3, 3)
        assert np.array_equal(S[:2, :2] - np.eye(2), np.array(ex["S_minus_K"], float)), ex["cite"]


def test_golden_l1(oracle_lib):
    for ex in GOLD["l1"]:
        A = np.array(ex["A"], float)
        blk = np.eye(3); blk[:A.shape[0], :A.shape[0]] = A
        o = _single_node(oracle_lib, blk)
        d = o.get(9, 0)[:A.shape[0]]
        assert np.array_equal(d, np.array(ex["d"], float)), ex["cite"]


def test_golden_contact_dofs(oracle_lib):
    for ex in GOLD["contact_dofs"]:
        o = _single_node(oracle_lib, 4 * np.eye(3), ex["J"], [1.0] * len(ex["J"]))
        assert list(o.get(20)) == ex["Ic"], ex["cite"]


def test_table1_m_and_nc_closed_forms():
    # PAPER.md:619 Table 1 m^max row equals our configs' m; n_c = 2m; PAPER.md:370 scaling
    ms = GOLD["table1_m_max"]["m"]
    for cfg, m in enumerate(ms):
        N = gen.CONFIGS[cfg]["N"]
        assert (N + 1) ** 2 == m
    p0, p1 = gen.config(0), gen.config(1)
    for p in (p0, p1):
        assert p.n == 6 * (p.N + 1) ** 3 and p.m == (p.N + 1) ** 2 and len(p.Z) == 2 * p.m
        assert set(p.Z.tolist()) == set(np.unique(p.J_col).tolist())
    assert 3.4 < len(p1.Z) / len(p0.Z) < 4.5 and 6.5 < p1.n / p0.n < 8.5


# --------------------------------------------------------------- generator
def test_generator_rigid_body_modes_in_kernel_of_K():
    # north_star / SPEC.md:376: rigid-body modes lie in ker K without Dirichlet conditions
    N = 3
    Ke = gen.hex8_stiffness_unit(0.3)
    Kb = gen._assemble_body(N, Ke, np.ones((N, N, N)))
    n1 = N + 1
    k, j, i = np.meshgrid(np.arange(n1), np.arange(n1), np.arange(n1), indexing="ij")
    X, Y, Z = (i.ravel() / N - 0.3), (j.ravel() / N + 0.1), (k.ravel() / N - 0.7)
    rows, cols, vals = [], [], []
    for v in range(n1 ** 3):
        for d in range(27):
            dz, dy, dx = d // 9 - 1, (d // 3) % 3 - 1, d % 3 - 1
            ii, jj, kk = i.ravel()[v] + dx, j.ravel()[v] + dy, k.ravel()[v] + dz
            if 0 <= ii <= N and 0 <= jj <= N and 0 <= kk <= N:
                u = (kk * n1 + jj) * n1 + ii
                for a in range(3):
                    for c in range(3):
                        rows.append(3 * v + a); cols.append(3 * u + c); vals.append(Kb[v, d, a, c])
    K = sp.csr_matrix((vals, (rows, cols)), shape=(3 * n1 ** 3,) * 2)
    B = np.zeros((n1 ** 3, 3, 6))
    B[:, 0, 0] = B[:, 1, 1] = B[:, 2, 2] = 1
    B[:, 1, 3] = -Z; B[:, 2, 3] = Y; B[:, 0, 4] = Z; B[:, 2, 4] = -X; B[:, 0, 5] = -Y; B[:, 1, 5] = X
    B = B.reshape(-1, 6)
    assert np.abs(K @ B).max() <= 1e-13 * abs(K).max()
    assert abs(K - K.T).max() <= 1e-15
    ev = np.linalg.eigvalsh(K.toarray())
    assert np.sum(ev < 1e-10 * ev[-1]) == 6   # exactly the 6 rigid modes


def test_generator_patch_test():
    # linear displacement field => zero residual at interior nodes (consistency of Q1)
    p = tiny(N=4)
    K = K_csr(p)
    u = (p.coords @ np.array([[0.3, -0.1, 0.2], [0.05, 0.4, -0.2], [0.1, 0.2, 0.3]])).reshape(-1)
    r = K @ u
    n1 = p.N + 1
    for v in range(p.nodes):
        i = v % n1; j = (v // n1) % n1; k = (v // n1 ** 2) % n1
        if 0 < i < p.N and 0 < j < p.N and 1 < k < p.N - 1:   # not next to Dirichlet rows
            assert np.abs(r[3 * v:3 * v + 3]).max() < 1e-14


# ------------------------------------------------------------- S, I_c, A_w
@pytest.mark.parametrize("matching", [True, False])
def test_S_equals_dense_K_plus_JtDJ(oracle_lib, matching):
    p = tiny(N=3, matching=matching, e_max=8.0)
    o = oracle_lib.Oracle.from_problem(p)
    S = o.level_matrix(0).tocsr()
    ref = (K_csr(p) + J_csr(p).T @ sp.diags(p.D) @ J_csr(p)).toarray()
    assert np.abs(S.toarray() - ref).max() <= 4 * EPS * np.abs(ref).max()
    # symmetric pattern; only contact-dof entries differ from K
    diff = (S - K_csr(p)).tocoo()
    nz = np.abs(diff.data) > 0
    Zs = set(p.Z.tolist())
    assert all(r in Zs and c in Zs for r, c in zip(diff.row[nz], diff.col[nz]))


@pytest.mark.parametrize("matching", [True, False])
def test_bound_constrained_S(oracle_lib, matching):
    """Remark boundconstr: A~ = K + J~^T D~ J~ with J~ = [J; I; -I], D~ = diag(D, D_lo, D_up),
    built here densely from the explicit stacked J~ (not the oracle's diagonal shortcut).  Off-diagonal
    entries equal the box-free S bit for bit; the diagonal differs by D_lo + D_up; zero bounds give S."""
    p = tiny(N=3, matching=matching, e_max=8.0)
    lo, up = gen.box_diagonals(p, e_max=6.0, seed=11)
    o0 = oracle_lib.Oracle.from_problem(p)
    o = oracle_lib.Oracle.from_problem(p, D_lo=lo, D_up=up)
    S0, S = o0.level_matrix(0).toarray(), o.level_matrix(0).toarray()
    I = sp.identity(p.n, format="csr")
    Jt = sp.vstack([J_csr(p), I, -I]).tocsr()
    Dt = sp.diags(np.concatenate([p.D, lo, up]))
    ref = (K_csr(p) + Jt.T @ Dt @ Jt).toarray()
    assert np.abs(S - ref).max() <= 4 * EPS * np.abs(ref).max()
    off = ~np.eye(p.n, dtype=bool)
    assert np.array_equal(S[off], S0[off])
    d = np.diag(S) - np.diag(S0)
    assert np.allclose(d, lo + up, rtol=1e-15, atol=4 * EPS * np.abs(np.diag(S)).max())
    assert np.array_equal(oracle_lib.Oracle.from_problem(p, D_lo=np.zeros(p.n), D_up=np.zeros(p.n)).get(2), o0.get(2))
    # SPD and the AMGF-PCG solve is the dense solve of A~
    x, info = o.pcg(p.b, rtol=1e-12)
    assert info["converged"]
    xd = np.linalg.solve(ref, p.b)
    assert np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd)
    # a negative bound diagonal is a domain error
    with pytest.raises(oracle_lib.OracleError) as e:
        oracle_lib.Oracle.from_problem(p, D_lo=-lo)
    assert e.value.code == -3


def test_matching_S_block_count(oracle_lib):
    # node-to-node matching: S adds exactly 2 cross blocks per constraint
    p = gen.config(0)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=100000, factor_filter=0)
    assert o.levels[0]["nnzb"] == len(p.K_col) + 2 * p.m == 27824


def test_Aw_is_principal_submatrix_and_factor(oracle_lib):
    p = tiny(N=3, matching=False, e_max=6.0)
    o = oracle_lib.Oracle.from_problem(p)
    S = o.level_matrix(0).toarray()
    Aw = o.get(21)
    assert np.array_equal(Aw, S[np.ix_(p.Z, p.Z)])
    Lw = o.get(22)
    pi = o.get(25)
    assert sorted(pi.tolist()) == list(range(len(p.Z)))
    Awp = Aw[np.ix_(pi, pi)]
    assert np.abs(Lw @ Lw.T - Awp).max() <= 1e-13 * np.abs(Aw).max()
    # filter solves A_w exactly: residual in span(Z) is corrected exactly (north_star)
    w = np.random.default_rng(3).standard_normal(len(p.Z))
    y = o.filter_solve(Aw @ w)
    assert np.abs(y - w).max() <= 1e-6 * np.abs(w).max()
    assert np.abs(Aw @ y - Aw @ w).max() <= 1e-12 * np.abs(Aw @ w).max()


@pytest.mark.parametrize("levels", [0, 1, 3])
def test_nd_order_structure(oracle_lib, levels):
    """Reading R16: the nested-dissection order is a permutation; a separator of width bw decouples its two
    sides (no A_w entry across it), so the dense factor of A_w[pi,pi] has no fill outside the profile:
    leaf rows within bw of the diagonal inside their leaf, separator rows from their subtree start."""
    p = gen.config(1)
    o = oracle_lib.Oracle.from_problem(p, nd_levels=levels)
    bw = int(o.get(26)[0])
    pi = o.get(25)
    assert sorted(pi.tolist()) == list(range(o.nc))
    S = o.level_matrix(0).toarray()
    Aw = S[np.ix_(p.Z, p.Z)]
    ii, jj = np.nonzero(Aw)
    assert np.abs(ii - jj).max() == bw
    L = o.get(22)
    # block structure from pi: maximal runs of consecutive Z positions
    starts = [0] + [i for i in range(1, o.nc) if pi[i] != pi[i - 1] + 1]
    nblocks = len(starts)
    assert nblocks % 2 == 1 and nblocks <= 2 ** (levels + 1) - 1 and (levels == 0) == (nblocks == 1)
    env = np.zeros(o.nc, int)
    # reconstruct subtrees recursively from the postorder (leaf, leaf, sep) pattern: a block of length bw
    # preceded by two subtrees is a separator
    stack = []
    bounds = starts + [o.nc]
    for b in range(nblocks):
        b0, b1 = bounds[b], bounds[b + 1]
        is_sep = levels > 0 and (b1 - b0) == bw and len(stack) >= 2
        if is_sep:
            r = stack.pop(); l = stack.pop()
            env[b0:b1] = l[0]
            stack.append((l[0], b1))
        else:
            env[b0:b1] = np.maximum(np.arange(b0, b1) - bw, b0)
            stack.append((b0, b1))
    for i in range(o.nc):
        assert not L[i, :env[i]].any()


def test_Z_validation(oracle_lib):
    p = tiny(N=2)
    bad = p.Z.copy(); bad[0] = 0
    with pytest.raises(oracle_lib.OracleError):
        oracle_lib.Oracle.from_problem(p, Z=bad)
    o = oracle_lib.Oracle.from_problem(p, Z=None)
    assert np.array_equal(o.get(20), np.sort(p.Z))
    with pytest.raises(oracle_lib.OracleError):          # must contain every column of J
        oracle_lib.Oracle.from_problem(p, Z=p.Z[1:])
    extra = np.concatenate([p.Z, [0]]).astype(np.int32)  # supersets are allowed
    assert oracle_lib.Oracle.from_problem(p, Z=extra).nc == len(p.Z) + 1


def test_domain_errors(oracle_lib):
    p = tiny(N=2)
    D = p.D.copy(); D[0] = 0.0
    with pytest.raises(oracle_lib.OracleError) as e:
        oracle_lib.Oracle.from_problem(p, D=D)
    assert e.value.code == -3
    D[0] = np.nan
    with pytest.raises(oracle_lib.OracleError) as e:
        oracle_lib.Oracle.from_problem(p, D=D)
    assert e.value.code == -2


# ---------------------------------------------------------- aggregation
def _graph(o, level):
    A = o.level_matrix(level).tocsr()
    b = o.levels[level]["b"]
    comp = o.get(15, level)
    ptr, col = o.get(0, level), o.get(1, level)
    nb = o.levels[level]["nodes"]
    adj = [set(int(c) for c in col[ptr[v]:ptr[v + 1]] if c != v and comp[c] == comp[v]) for v in range(nb)]
    return adj


@pytest.mark.parametrize("N,matching", [(3, True), (4, False)])
def test_aggregation_is_greedy_mis2(oracle_lib, N, matching):
    p = tiny(N=N, matching=matching)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=16)
    for level in range(o.nlev - 1):
        adj = _graph(o, level)
        nb = len(adj)
        root = o.get(14, level).astype(bool)
        agg = o.get(10, level)
        seed = o.cfg["agg_seed"]
        pr = [(oracle_lib.priority(v, seed), -v) for v in range(nb)]
        d2 = []
        for v in range(nb):
            s1 = adj[v]
            s2 = set().union(*[adj[u] for u in s1]) if s1 else set()
            d2.append((s1 | s2) - {v})
        iso = [len(adj[v]) == 0 for v in range(nb)]
        for v in range(nb):
            if iso[v]:
                assert agg[v] == -1 and not root[v]
                continue
            higher_roots = [u for u in d2[v] if root[u] and pr[u] > pr[v]]
            # lexicographically-first MIS of G^2: v is a root iff no higher-priority root within distance 2
            assert root[v] == (len(higher_roots) == 0)
            if root[v]:
                assert not any(root[u] for u in d2[v])
            assert agg[v] >= 0
        # aggregate ids are ranks of the roots; aggregates are connected and single-component
        roots = np.nonzero(root)[0]
        assert np.array_equal(agg[roots], np.arange(len(roots)))
        comp = o.get(15, level)
        for a in range(len(roots)):
            mem = set(np.nonzero(agg == a)[0].tolist())
            assert len({int(comp[v]) for v in mem}) == 1
            seen, todo = {int(roots[a])}, [int(roots[a])]
            while todo:
                v = todo.pop()
                for u in adj[v]:
                    if u in mem and u not in seen:
                        seen.add(u); todo.append(u)
            assert seen == mem


def test_level0_components_are_bodies(oracle_lib):
    p = tiny(N=3, matching=False)
    o = oracle_lib.Oracle.from_problem(p)
    comp = o.get(15, 0)
    body = np.repeat([0, 1], p.nodes // 2)
    free = ~p.dirichlet
    assert len(set(comp[free & (body == 0)])) == 1 and len(set(comp[free & (body == 1)])) == 1
    assert set(comp[free & (body == 0)]) != set(comp[free & (body == 1)])


# ------------------------------------------------------------- hierarchy
@pytest.mark.parametrize("matching", [True, False])
def test_hierarchy_galerkin_and_prolongator(oracle_lib, matching):
    p = tiny(N=4, matching=matching, e_max=6.0)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=16)
    assert o.nlev >= 2
    for l in range(o.nlev - 1):
        A = o.level_matrix(l).toarray()
        P = o.level_matrix(l, "P").toarray()
        R = o.level_matrix(l, "R").toarray()
        b = o.levels[l]["b"]
        # R = P^T exactly
        assert np.array_equal(R, P.T)
        # tentative prolongator: orthonormal columns per aggregate, reproduces near-null space
        agg = o.get(10, l)
        Pt_val = o.get(13, l).reshape(-1, b, 6)
        nb = o.levels[l]["nodes"]
        Pt = np.zeros((nb * b, 6 * o.levels[l]["n_agg"]))
        q = 0
        for v in range(nb):
            if agg[v] >= 0:
                Pt[v * b:(v + 1) * b, 6 * agg[v]:6 * agg[v] + 6] = Pt_val[q]; q += 1
        assert np.abs(Pt.T @ Pt - np.eye(Pt.shape[1])).max() <= 1e-12
        Bf = o.get(11, l)
        Bc = o.get(11, l + 1)
        mask = (agg >= 0).repeat(b)
        assert np.abs((Pt @ Bc)[mask] - Bf[mask]).max() <= 1e-12 * max(1, np.abs(Bf).max())
        # smoothed prolongator P = (I - omega D^{-1} A) Pt (reading R6)
        lam, om = o.get(12, l)
        assert abs(om - 4.0 / (3.0 * lam)) <= 4 * EPS * om
        dpt = np.diag(A)
        Pref = Pt - om * (A @ Pt) / dpt[:, None]
        assert np.abs(P - Pref).max() <= 1e-13 * np.abs(Pref).max()
        # lambda_hat is a power-iteration estimate of lambda_max(D^{-1}A)
        Dm = np.diag(1 / np.sqrt(dpt))
        lmax = np.linalg.eigvalsh(Dm @ A @ Dm)[-1]
        assert 0.6 * lmax <= lam <= 1.05 * lmax
        # Galerkin coarse operator, exactly symmetric, SPD
        Ac = o.level_matrix(l + 1).toarray()
        G = P.T @ A @ P
        assert np.abs(Ac - G).max() <= 1e-12 * np.abs(G).max()
        assert np.array_equal(Ac, Ac.T)
        assert np.linalg.eigvalsh(Ac)[0] > 0
        # l1 diagonal
        assert np.abs(o.get(9, l) - np.abs(A).sum(axis=1)).max() <= 64 * EPS * np.abs(A).sum(axis=1).max()


def test_power_iteration_converges(oracle_lib):
    p = tiny(N=3)
    o = oracle_lib.Oracle.from_problem(p, power_iters=300, coarsest_size=16)
    A = o.level_matrix(0).toarray()
    Dm = np.diag(1 / np.sqrt(np.diag(A)))
    lmax = np.linalg.eigvalsh(Dm @ A @ Dm)[-1]
    assert abs(o.get(12, 0)[0] - lmax) <= 2e-3 * lmax


def test_spmv_and_restriction_match_scipy(oracle_lib):
    p = tiny(N=4, matching=False)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=16)
    x = np.random.default_rng(4).standard_normal(p.n)
    A = o.level_matrix(0)
    y = o.spmv(x)
    assert np.abs(y - A @ x).max() <= 64 * EPS * (abs(A) @ np.abs(x)).max()


# ------------------------------------------------------------ V-cycle (B)
def _dense_vcycle(o):
    """B from the operator-product form of the V-cycle: E = (I-D^{-1}A)(I-P B_c R A)(I-D^{-1}A)."""
    Bc = np.linalg.inv(o.get(23))
    for l in range(o.nlev - 2, -1, -1):
        A = o.level_matrix(l).toarray()
        P = o.level_matrix(l, "P").toarray()
        Dinv = np.diag(1 / o.get(9, l))
        I = np.eye(A.shape[0])
        E = (I - Dinv @ A) @ (I - P @ Bc @ P.T @ A) @ (I - Dinv @ A)
        Bc = (I - E) @ np.linalg.inv(A)
    return Bc


@pytest.mark.parametrize("N,matching,e_max", [(2, True, 4.0), (3, False, 3.0)])
def test_vcycle_operator(oracle_lib, N, matching, e_max):
    """l1-Jacobi smoother (smoother=0, contract C4)."""
    p = tiny(N=N, matching=matching, e_max=e_max)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=16, smoother=0)
    assert o.nlev >= 2
    B = dense_op(o.vcycle, p.n)
    Bref = _dense_vcycle(o)
    assert np.abs(B - Bref).max() <= 1e-9 * np.abs(Bref).max()
    # symmetric, positive definite, convergent with omega <= 1
    assert np.abs(B - B.T).max() <= 1e-11 * np.abs(B).max()
    assert np.linalg.eigvalsh(0.5 * (B + B.T))[0] > 0
    A = o.level_matrix(0).toarray()
    Lc = np.linalg.cholesky(A)
    ev = np.linalg.eigvalsh(Lc.T @ B @ Lc)
    assert ev[-1] <= 1 + 1e-9 and ev[0] > 0


def test_single_level_vcycle_is_exact(oracle_lib):
    p = tiny(N=2)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=10 ** 6)
    assert o.nlev == 1
    A = o.level_matrix(0).toarray()
    r = np.random.default_rng(5).standard_normal(p.n)
    assert np.abs(A @ o.vcycle(r) - r).max() <= 1e-10 * np.abs(r).max()
    # B exact => M = A^{-1} for any I_c
    assert np.abs(A @ o.apply(r) - r).max() <= 1e-9 * np.abs(r).max()


# ------------------------------------------------------------- AMGF (M)
def _P_embed(p, n):
    P = np.zeros((n, len(p.Z)))
    P[p.Z, np.arange(len(p.Z))] = 1.0
    return P


@pytest.mark.parametrize("N,matching,e_max", [(2, True, 4.0), (3, False, 4.0)])
def test_amgf_operator_identity_and_splitting(oracle_lib, N, matching, e_max):
    # Def. AMGF eq:M_itmat and eq:M_splitting, at D <= 1e4 (reading R13)
    p = tiny(N=N, matching=matching, e_max=e_max)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=16)
    n = p.n
    A = o.level_matrix(0).toarray()
    M = dense_op(o.apply, n)
    B = dense_op(o.vcycle, n)
    P = _P_embed(p, n)
    Aw = P.T @ A @ P
    I = np.eye(n)
    Pi = I - P @ np.linalg.solve(Aw, P.T @ A)
    lhs = I - M @ A
    rhs = (I - B @ A) @ Pi @ (I - B @ A)
    # rounding of the inner solves grows with cond(A) ~ 1e6 at D <= 1e4 (reading R13): measured 5e-8 (10 power
    # steps) and 1.5e-7 (6, R19) against max|I - MA| = 0.7 / 1.7; a dropped term or wrong sign is O(1)
    assert np.abs(lhs - rhs).max() <= 1e-6 * max(1.0, np.abs(lhs).max())
    # splitting form
    Binv = np.linalg.inv(B)
    nc = P.shape[1]
    Z0 = np.zeros((n, nc))
    L1 = np.block([[Binv, Z0], [P.T @ A, np.eye(nc)]])
    Mid = np.block([[np.linalg.inv(2 * Binv - A), Z0], [Z0.T, Aw]])
    U1 = np.block([[Binv, A @ P], [Z0.T, np.eye(nc)]])
    Mbar = L1 @ Mid @ U1
    IP = np.hstack([I, P])
    Msplit = IP @ np.linalg.solve(Mbar, IP.T)
    assert np.abs(M - Msplit).max() <= 1e-6 * np.abs(M).max()
    # filter projector: Pi P = 0 (exact correction in span(Z)), Pi^2 = Pi
    assert np.abs(Pi @ P).max() <= 1e-9
    assert np.abs(Pi @ Pi - Pi).max() <= 1e-8


@pytest.mark.parametrize("N,matching", [(2, True), (3, False)])
def test_amgf_Jt_basis(oracle_lib, N, matching):
    """Variant f4, P = J^T (the generality remark; reading R21): A_w = J S J^T entry by entry
    (dense product), the apply equals I - M A = (I - B A)(I - P A_w^{-1} P^T A)(I - B A) with P = J^T densely,
    errors in range(J^T) are corrected exactly by the filter projector, and the Lemma main bound holds."""
    p = tiny(N=N, matching=matching, e_max=4.0)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=16, filter_basis=1)
    n = p.n
    assert o.nf == p.m
    A = o.level_matrix(0).toarray()
    P = J_csr(p).T.toarray()
    Aw_ref = P.T @ A @ P
    Aw = o.get(21)
    assert np.abs(Aw - Aw_ref).max() <= 8 * EPS * np.abs(Aw_ref).max()
    # the factor is of A_w[pi, pi]
    pi = o.get(25)
    Lw = o.get(22)
    assert np.abs(Lw @ Lw.T - Aw[np.ix_(pi, pi)]).max() <= 1e-12 * np.abs(Aw).max()
    M = dense_op(o.apply, n)
    B = dense_op(o.vcycle, n)
    I = np.eye(n)
    Pi = I - P @ np.linalg.solve(Aw_ref, P.T @ A)
    lhs = I - M @ A
    rhs = (I - B @ A) @ Pi @ (I - B @ A)
    assert np.abs(lhs - rhs).max() <= 1e-6 * max(1.0, np.abs(lhs).max())
    assert np.abs(Pi @ P).max() <= 1e-9 * max(1.0, np.abs(P).max())
    # the identity embedding's filter space contains range(J^T): a different (smaller) correction
    assert np.abs(M - dense_op(oracle_lib.Oracle.from_problem(p, coarsest_size=16).apply, n)).max() > 1e-6
    Lc = np.linalg.cholesky(A)
    evM = np.sort(np.linalg.eigvals(Lc.T @ M @ Lc).real)
    om = np.linalg.eigvals(Lc.T @ B @ Lc).real.max()
    V = sla.null_space(P.T @ A)
    beta = sla.eigh(V.T @ np.linalg.inv(0.5 * (B + B.T)) @ V, V.T @ A @ V, eigvals_only=True)[-1]
    assert evM[0] > 0 and evM[-1] <= 1 + 1e-8
    assert evM[-1] / evM[0] <= 2 * (beta + 2 + om) / (2 - om) * (1 + 1e-6)


@pytest.mark.parametrize("e_max", [0.0, 4.0, 8.0, 12.0])
def test_amgf_spectral_bounds(oracle_lib, e_max):
    # Lemma "Lower bound" => lambda_max(MA) <= 1 (reading R12),
    # Lemma main: kappa(MA) <= 2(beta+2+omega)/(2-omega)
    p = tiny(N=3, matching=False, e_max=e_max)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=16)
    n = p.n
    A = o.level_matrix(0).toarray()
    M = dense_op(o.apply, n)
    B = dense_op(o.vcycle, n)
    Lc = np.linalg.cholesky(A)
    evM = np.linalg.eigvals(Lc.T @ M @ Lc).real
    evM.sort()
    tol = 1e-8 if e_max <= 8 else 2e-4    # [E2]: fp64 limit at D = 1e12
    assert evM[-1] <= 1 + tol
    assert evM[0] > 0
    om = np.linalg.eigvals(Lc.T @ B @ Lc).real.max()
    assert om <= 1 + tol
    P = _P_embed(p, n)
    V = sla.null_space(P.T @ A)               # A-orthogonal complement of range(P)
    Binv = np.linalg.inv(0.5 * (B + B.T))
    beta = sla.eigh(V.T @ Binv @ V, V.T @ A @ V, eigvals_only=True)[-1]
    kappa = evM[-1] / evM[0]
    assert kappa <= 2 * (beta + 2 + om) / (2 - om) * (1 + 1e-6)


def test_amgf_degenerate_Ic(oracle_lib):
    # I_c empty => M = 2B - BAB; I_c = all => M = A^{-1}
    p = tiny(N=2)
    Kp, Kc, Kv = p.K_ptr, p.K_col, p.K_val
    empty = oracle_lib.Oracle(p.nodes, Kp, Kc, Kv, np.zeros(1, np.int32), np.zeros(0, np.int32),
                              np.zeros(0), np.zeros(0), None, p.B_nns, coarsest_size=16)
    n = p.n
    A = empty.level_matrix(0).toarray()
    M = dense_op(empty.apply, n)
    B = dense_op(empty.vcycle, n)
    assert np.abs(M - (2 * B - B @ A @ B)).max() <= 1e-10 * np.abs(M).max()
    J = sp.identity(n, format="csr")
    full = oracle_lib.Oracle(p.nodes, Kp, Kc, Kv, J.indptr, J.indices, J.data, np.full(n, 1e-3), None,
                             p.B_nns, coarsest_size=16)
    A = full.level_matrix(0).toarray()
    assert full.nc == n
    r = np.random.default_rng(6).standard_normal(n)
    assert np.abs(A @ full.apply(r) - r).max() <= 1e-10 * np.abs(r).max()
    x, rep = full.pcg(r, rtol=1e-8)
    assert rep["iterations"] == 1 and rep["converged"]


# ------------------------------------------------------------------- PCG
@pytest.mark.parametrize("matching,e_max", [(True, 8.0), (False, 4.0)])
def test_pcg_against_direct_and_monotone(oracle_lib, matching, e_max):
    p = tiny(N=4, matching=matching, e_max=e_max)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=16)
    A = o.level_matrix(0).tocsc()
    xs = spl.spsolve(A, p.b)
    x, rep = o.pcg(p.b, rtol=1e-10)
    assert rep["converged"] and rep["relres"] < 1e-10
    An = lambda e: math.sqrt(e @ (A @ e))
    assert An(x - xs) <= 1e-7 * An(xs)
    errs = []
    for k in range(1, rep["iterations"] + 1):
        xk, _ = o.pcg(p.b, rtol=0.0, maxit=k)
        errs.append(An(xk - xs))
    assert all(e2 <= e1 * (1 + 1e-9) + 1e-14 for e1, e2 in zip(errs, errs[1:]))
    # zero rhs => zero iterations
    x0, r0 = o.pcg(np.zeros(p.n))
    assert r0["iterations"] == 0 and not x0.any()


def test_amgf_robust_vs_amg(oracle_lib):
    # Fig. amgvsamgf: B-only PCG degrades with cond(D), AMGF does not
    p = gen.config(0)
    o_lo = oracle_lib.Oracle.from_problem(p, D=np.ones(p.m))
    o_hi = oracle_lib.Oracle.from_problem(p)
    it = lambda o, pc: o.pcg(p.b, rtol=1e-8, maxit=400, precond=pc)[1]["iterations"]
    amgf_lo, amgf_hi = it(o_lo, "amgf"), it(o_hi, "amgf")
    amg_hi = it(o_hi, "amg")
    assert amg_hi >= 4 * amgf_hi
    assert amgf_hi <= 2 * amgf_lo


# ------------------------------------------------ Chebyshev smoother (variant f4, reading R18)
@pytest.mark.parametrize("k,ratio", [(1, 30.0), (2, 30.0), (3, 30.0), (4, 10.0)])
def test_cheb_coefficients_closed_form(oracle_lib, k, ratio):
    """The oracle's three-term coefficients reproduce the scaled Chebyshev polynomial: running the update
    recurrence on a scalar 'matrix' lambda gives the error factor T_k((theta - lambda)/delta) / T_k(sigma)."""
    from numpy.polynomial import chebyshev as C
    c0, ab = oracle_lib.cheb_coefs(k, ratio)
    theta, delta = (1 + 1 / ratio) / 2, (1 - 1 / ratio) / 2
    Tk = C.Chebyshev.basis(k)
    for lam in np.linspace(0.0, 1.0, 23):
        e = 1.0  # error of x for b = 0 (x* = 0): x = e, the update uses r = -lam * x
        d = c0 * (-lam * e)
        e = e + d
        for a, b in ab:
            d = a * d + b * (-lam * e)
            e = e + d
        assert abs(e - Tk((theta - lam) / delta) / Tk(theta / delta)) <= 1e-12


def _dense_vcycle_cheb(o, k, ratio):
    """B from the operator-product form with Chebyshev smoothers S = T_k((theta I - D^{-1}A)/delta)/T_k(sigma)
    (matrix three-term recurrence T_{j+1} = 2 X T_j - T_{j-1})."""
    theta, delta = (1 + 1 / ratio) / 2, (1 - 1 / ratio) / 2
    from numpy.polynomial import chebyshev as C
    tks = C.Chebyshev.basis(k)(theta / delta)
    Bc = np.linalg.inv(o.get(23))
    for l in range(o.nlev - 2, -1, -1):
        A = o.level_matrix(l).toarray()
        P = o.level_matrix(l, "P").toarray()
        I = np.eye(A.shape[0])
        X = (theta * I - np.diag(1 / o.get(9, l)) @ A) / delta
        T0, T1 = I, X
        for _ in range(k - 1):
            T0, T1 = T1, 2 * X @ T1 - T0
        S = (T1 if k >= 1 else T0) / tks
        E = S @ (I - P @ Bc @ P.T @ A) @ S
        Bc = (I - E) @ np.linalg.inv(A)
    return Bc


@pytest.mark.parametrize("N,matching,k", [(2, True, 2), (3, False, 3), (3, False, 1)])
def test_cheb_vcycle_operator(oracle_lib, N, matching, k):
    p = tiny(N=N, matching=matching, e_max=3.0)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=16, smoother=1, cheb_degree=k, cheb_ratio=30.0)
    assert o.nlev >= 2
    B = dense_op(o.vcycle, p.n)
    Bref = _dense_vcycle_cheb(o, k, 30.0)
    assert np.abs(B - Bref).max() <= 1e-9 * np.abs(Bref).max()
    assert np.abs(B - B.T).max() <= 1e-11 * np.abs(B).max()  # symmetric smoother => symmetric V-cycle
    A = o.level_matrix(0).toarray()
    Lc = np.linalg.cholesky(A)
    ev = np.linalg.eigvalsh(Lc.T @ B @ Lc)
    assert ev[-1] <= 1 + 1e-9 and ev[0] > 0  # convergent on [0, 1]: |T_k((theta-l)/delta)| <= T_k(sigma)


def test_cheb_config_errors(oracle_lib):
    p = tiny(N=2)
    for bad in (dict(smoother=1, cheb_degree=0), dict(smoother=1, cheb_ratio=1.0), dict(smoother=3)):
        with pytest.raises(Exception):
            oracle_lib.Oracle.from_problem(p, **bad)


# ------------------------------------------------------------- nodal-block l1 smoother (variant f4, C24/C25)
def _block_diag_B(o, l):
    """Dense block-diagonal B of level l rebuilt from the oracle's stored factors (L L^T per node)."""
    Lv = o.levels[l]
    b, nodes = Lv["b"], Lv["nodes"]
    f = o.get(16, l)
    B = np.zeros((nodes * b, nodes * b))
    for i in range(nodes):
        Lf = np.zeros((b, b))
        Lf[np.tril_indices(b)] = f[i, :b * (b + 1) // 2]
        assert np.array_equal(f[i, b * (b + 1) // 2:], 1.0 / np.diag(Lf))
        B[i * b:(i + 1) * b, i * b:(i + 1) * b] = Lf @ Lf.T
    return B


@pytest.mark.parametrize("N,matching", [(2, True), (3, False)])
def test_block_l1_smoother(oracle_lib, N, matching):
    """Nodal-block l1 smoother (smoother 2, reading R22): per node B_i = A_ii + diag(off-block l1 row sums),
    checked against A densely; lambda_max(B^{-1} A) <= 1 (block l1 => convergent with weight 1);
    the V-cycle equals the dense composition of x = B^{-1} b, the coarse correction and x + B^{-1}(b - A x), and
    is symmetric, positive definite and convergent."""
    p = tiny(N=N, matching=matching, e_max=3.0)
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=16, smoother=2)
    assert o.nlev >= 2
    for l in range(o.nlev - 1):
        A = o.level_matrix(l).toarray()
        b = o.levels[l]["b"]
        B = _block_diag_B(o, l)
        ref = np.zeros_like(A)
        offl1 = np.abs(A).sum(1)
        for i in range(A.shape[0] // b):
            sl = slice(i * b, (i + 1) * b)
            ref[sl, sl] = A[sl, sl]
            offl1[sl] -= np.abs(A[sl, sl]).sum(1)
        ref += np.diag(offl1)
        assert np.abs(B - ref).max() <= 1e-12 * np.abs(ref).max()
        ev = np.linalg.eigvals(np.linalg.solve(B, A)).real
        assert ev.max() <= 1 + 1e-10 and ev.min() > 0
    # V-cycle operator (E = (I - B^-1 A)(I - P Bc R A)(I - B^-1 A) level by level)
    Bc = np.linalg.inv(o.level_matrix(o.nlev - 1).toarray())
    for l in range(o.nlev - 2, -1, -1):
        A = o.level_matrix(l).toarray()
        P = o.level_matrix(l, "P").toarray()
        Sm = np.eye(A.shape[0]) - np.linalg.solve(_block_diag_B(o, l), A)
        E = Sm @ (np.eye(A.shape[0]) - P @ Bc @ P.T @ A) @ Sm
        Bc = (np.eye(A.shape[0]) - E) @ np.linalg.inv(A)
    V = dense_op(o.vcycle, p.n)
    assert np.abs(V - Bc).max() <= 1e-9 * np.abs(Bc).max()
    assert np.abs(V - V.T).max() <= 1e-11 * np.abs(V).max()
    A = o.level_matrix(0).toarray()
    Lc = np.linalg.cholesky(A)
    ev = np.linalg.eigvalsh(Lc.T @ V @ Lc)
    assert ev[-1] <= 1 + 1e-9 and ev[0] > 0
