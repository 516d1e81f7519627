"""CPU oracle for the AMGF-PCG path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product path
(paper_2505_18576_b200) never imports, links or executes anything here, and
this package never imports the product path.  See oracle/amgf_oracle.c for the
paper citations of each function and DESIGN.md "Contract" for the arithmetic.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "amgf_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]


def _host_has_fma() -> bool:
    try:
        return any(ln.startswith("flags") and " fma " in ln + " " for ln in open("/proc/cpuinfo"))
    except OSError:
        return False


# -mfma lets gcc emit fma() as one vfmadd instruction instead of a libm call.  fma() is one correctly
# rounded operation either way (IEEE 754 fusedMultiplyAdd), so the results are bit-identical (pinned by
# tests/test_oracle_pins.py::test_fma_build_bit_identical); -ffp-contract=off still forbids any FMA that
# is not written.  The oracle's dense Cholesky (a dependent FMA chain) runs about 1.6x faster.
if _host_has_fma():
    CFLAGS = CFLAGS + ["-mfma"]


def cheb_coefs(k: int, ratio: float):
    """Chebyshev smoother coefficients (c0, [(a_s, b_s) for s = 1..k-1]) of the oracle (reading R18)."""
    out = np.zeros(2 * k)
    lib().orc_cheb_coefs(k, ratio, _p(out))
    return out[0], [(out[2 * s - 1], out[2 * s]) for s in range(1, k)]


def build(force: bool = False, out: str = _LIB, flags=None) -> str:
    flags = CFLAGS if flags is None else flags
    stamp = out + ".flags"
    same = os.path.exists(stamp) and open(stamp).read() == " ".join(flags)
    if force or not same or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *flags, "-o", out, _SRC, "-lm"])
        with open(stamp, "w") as f:
            f.write(" ".join(flags))
    return out


class OrcConfig(ctypes.Structure):
    _fields_ = [("pre_sweeps", ctypes.c_int), ("post_sweeps", ctypes.c_int),
                ("coarsest_size", ctypes.c_int), ("max_levels", ctypes.c_int),
                ("power_iters", ctypes.c_int), ("factor_filter", ctypes.c_int),
                ("agg_seed", ctypes.c_uint64), ("nd_levels", ctypes.c_int), ("smoother", ctypes.c_int),
                ("cheb_degree", ctypes.c_int), ("filter_basis", ctypes.c_int), ("cheb_ratio", ctypes.c_double)]


DEFAULTS = dict(pre_sweeps=1, post_sweeps=1, coarsest_size=64, max_levels=25,
                power_iters=6, factor_filter=1, agg_seed=0x5EED, nd_levels=3, smoother=1, cheb_degree=2,
                cheb_ratio=20.0, filter_basis=0)

_lib = None


def lib():
    global _lib
    if _lib is None:
        if os.environ.get("AMGF_ORACLE_NOFMA") == "1":   # libm fma() calls (pin of the -mfma build)
            path = build(out=os.path.join(_HERE, "liboracle_nofma.so"), flags=[f for f in CFLAGS if f != "-mfma"])
        else:
            path = build()
        L = ctypes.CDLL(path)
        P = ctypes.c_void_p
        L.orc_create.restype = P
        L.orc_create.argtypes = [ctypes.c_int, P, P, P, ctypes.c_int, P, P, P, P, P, ctypes.c_int, P,
                                 ctypes.POINTER(OrcConfig), ctypes.POINTER(ctypes.c_int)]
        L.orc_create_box.restype = P
        L.orc_create_box.argtypes = [ctypes.c_int, P, P, P, ctypes.c_int, P, P, P, P, P, P, P, ctypes.c_int, P,
                                     ctypes.POINTER(OrcConfig), ctypes.POINTER(ctypes.c_int)]
        L.orc_free.argtypes = [P]
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_dot.restype = ctypes.c_double
        L.orc_dot.argtypes = [ctypes.c_long, ctypes.c_int, P, P]
        L.orc_cholesky_dense.argtypes = [ctypes.c_int, P, P]
        L.orc_trsv_dense.argtypes = [ctypes.c_int, P, P, P]
        L.orc_nd_order.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
        L.orc_priority.restype = ctypes.c_uint64
        L.orc_priority.argtypes = [ctypes.c_int, ctypes.c_uint64]
        L.orc_vcycle.argtypes = [P, P, P]
        L.orc_cheb_coefs.argtypes = [ctypes.c_int, ctypes.c_double, P]
        L.orc_apply.argtypes = [P, P, P]
        L.orc_spmv.argtypes = [P, ctypes.c_int, P, P]
        L.orc_filter_solve.argtypes = [P, P, P]
        L.orc_pcg.argtypes = [P, P, P, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                              ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), P]
        L.orc_info.argtypes = [P, P]
        L.orc_bsr_spmv.argtypes = [ctypes.c_int] * 4 + [P] * 5
        L.orc_get.argtypes = [P, ctypes.c_int, ctypes.c_int, P]
        L.orc_times.argtypes = [P, P]
        L.orc_nf.argtypes = [P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


def dot(u, v, b=3) -> float:
    u = _c(u, np.float64); v = _c(v, np.float64)
    return lib().orc_dot(u.size, b, _p(u), _p(v))


def cholesky(A):
    A = _c(A, np.float64); n = A.shape[0]
    L = np.zeros_like(A)
    st = lib().orc_cholesky_dense(n, _p(A), _p(L))
    if st:
        raise OracleError(st, lib().orc_last_error().decode())
    return L


def chol_solve(L, v):
    L = _c(L, np.float64); v = _c(v, np.float64)
    x = np.zeros_like(v)
    lib().orc_trsv_dense(L.shape[0], _p(L), _p(v), _p(x))
    return x


def bsr_spmv(ptr, col, val, x, br, bc):
    ptr = _c(ptr, np.int32); col = _c(col, np.int32); val = _c(val, np.float64); x = _c(x, np.float64)
    nbr = len(ptr) - 1
    y = np.zeros(nbr * br)
    lib().orc_bsr_spmv(nbr, len(x) // bc, br, bc, _p(ptr), _p(col), _p(val), _p(x), _p(y))
    return y


def nd_order(nc: int, bw: int, levels: int):
    out = np.zeros(max(nc, 1), np.int32)
    lib().orc_nd_order(nc, bw, levels, _p(out))
    return out[:nc]


def priority(v: int, seed: int) -> int:
    return lib().orc_priority(v, seed)


class Oracle:
    """Oracle AMGF hierarchy for one system S = K + J^T D J."""

    def __init__(self, nodes, K_ptr, K_col, K_val, J_ptr, J_col, J_val, D, Z, B_nns, D_lo=None, D_up=None, **cfg):
        """D_lo / D_up (n, >= 0, optional): bound-constraint diagonals of A~ = K + J~^T D~ J~."""
        c = dict(DEFAULTS); c.update(cfg)
        self.cfg = c
        self._keep = [_c(K_ptr, np.int32), _c(K_col, np.int32), _c(K_val, np.float64),
                      _c(J_ptr, np.int32), _c(J_col, np.int32), _c(J_val, np.float64),
                      _c(D, np.float64), None if Z is None else _c(Z, np.int32),
                      _c(B_nns, np.float64)]
        k = self._keep
        m = len(k[3]) - 1
        conf = OrcConfig(**c)
        st = ctypes.c_int(0)
        box = [None if v is None else _c(v, np.float64) for v in (D_lo, D_up)]
        self._keep += box
        self.h = lib().orc_create_box(nodes, _p(k[0]), _p(k[1]), _p(k[2]), m, _p(k[3]), _p(k[4]), _p(k[5]),
                                      _p(k[6]), _p(box[0]), _p(box[1]), _p(k[7]), 0 if Z is None else len(k[7]),
                                      _p(k[8]), ctypes.byref(conf), ctypes.byref(st))
        if not self.h:
            raise OracleError(st.value, lib().orc_last_error().decode())
        self.n = 3 * nodes
        self._k = None
        info = np.zeros(3 + 5 * 32, dtype=np.int64)
        lib().orc_info(self.h, _p(info))
        self.nlev, self.nc, self.nco = int(info[0]), int(info[1]), int(info[2])
        self.nf = int(lib().orc_nf(self.h))   # filter-space dimension (n_c, or m for filter_basis = 1)
        self.levels = [dict(nodes=int(info[3 + 5 * l]), b=int(info[4 + 5 * l]), nnzb=int(info[5 + 5 * l]),
                            nnzb_P=int(info[6 + 5 * l]), n_agg=int(info[7 + 5 * l])) for l in range(self.nlev)]

    @classmethod
    def from_problem(cls, p, D=None, Z="lattice", D_lo=None, D_up=None, **cfg):
        Zv = p.Z if isinstance(Z, str) and Z == "lattice" else Z
        return cls(p.nodes, p.K_ptr, p.K_col, p.K_val, p.J_ptr, p.J_col, p.J_val,
                   p.D if D is None else D, Zv, p.B_nns, D_lo=D_lo, D_up=D_up, **cfg)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_free(self.h)
            self.h = None

    # --- getters ---
    def get(self, which, level=0):
        L = self.levels[level]
        b, nodes = L["b"], L["nodes"]
        shapes = {0: (nodes + 1, np.int32), 1: (L["nnzb"], np.int32), 2: ((L["nnzb"], b * b), np.float64),
                  3: (nodes + 1, np.int32), 4: (L["nnzb_P"], np.int32), 5: ((L["nnzb_P"], b * 6), np.float64),
                  6: (L["n_agg"] + 1, np.int32), 7: (L["nnzb_P"], np.int32), 8: ((L["nnzb_P"], 6 * b), np.float64),
                  9: (nodes * b, np.float64), 10: (nodes, np.int32), 11: ((nodes * b, 6), np.float64),
                  12: (2, np.float64), 13: ((nodes, b * 6), np.float64), 14: (nodes, np.int32), 15: (nodes, np.int32),
                  16: ((nodes, b * (b + 1) // 2 + b), np.float64),
                  20: (self.nc, np.int32), 21: ((self.nf, self.nf), np.float64), 22: ((self.nf, self.nf), np.float64),
                  23: ((self.nco, self.nco), np.float64), 24: ((self.nco, self.nco), np.float64),
                  25: (self.nf, np.int32), 26: (1, np.int32)}
        shape, dt = shapes[which]
        out = np.zeros(shape, dtype=dt)
        if which == 13:
            # Pt has one block per aggregated node
            nz = int((self.get(10, level) >= 0).sum())
            out = np.zeros((nz, b * 6), dtype=dt)
        if lib().orc_get(self.h, which, level, _p(out)) != 0:
            raise OracleError(-1, f"get {which} failed")
        return out

    def level_matrix(self, level=0, kind="A"):
        """scipy BSR of a level operator (A, P or R)."""
        import scipy.sparse as sp
        L = self.levels[level]
        b = L["b"]
        if kind == "A":
            ptr, col, val = self.get(0, level), self.get(1, level), self.get(2, level).reshape(-1, b, b)
            return sp.bsr_matrix((val, col, ptr), shape=(L["nodes"] * b, L["nodes"] * b))
        nc = L["n_agg"]
        if kind == "P":
            ptr, col, val = self.get(3, level), self.get(4, level), self.get(5, level).reshape(-1, b, 6)
            return sp.bsr_matrix((val, col, ptr), shape=(L["nodes"] * b, nc * 6))
        ptr, col, val = self.get(6, level), self.get(7, level), self.get(8, level).reshape(-1, 6, b)
        return sp.bsr_matrix((val, col, ptr), shape=(nc * 6, L["nodes"] * b))

    def times(self):
        """Wall seconds of the setup phases (instrumentation): S, A_w assembly, A_w Cholesky, hierarchy."""
        t = np.zeros(4)
        lib().orc_times(self.h, _p(t))
        return dict(zip(("S", "A_w_assembly", "A_w_cholesky", "hierarchy"), t.tolist()))

    def export(self, path):
        """Write this oracle hierarchy in the amgf_export exchange format (include/amgf.h: manifest + raw
        little-endian arrays), so the CUDA path can apply exactly this preconditioner (amgf_import).  The
        writer is independent of the CUDA path's reader: it only lays out the oracle's own arrays."""
        os.makedirs(path, exist_ok=True)
        c = self.cfg
        lines = ["amgf_hierarchy 1", f"nodes {self.levels[0]['nodes']}", f"nlev {self.nlev}", f"nc {self.nc}",
                 f"bw {int(self.get(26)[0])}", f"nco {self.nco}"]
        for k in ("pre_sweeps", "post_sweeps", "smoother", "cheb_degree", "nd_levels", "coarsest_size",
                  "max_levels", "power_iters"):
            lines.append(f"{k} {int(c[k])}")
        lines.append(f"cheb_ratio {float(c['cheb_ratio'])!r}")
        lines.append(f"agg_seed {int(c['agg_seed'])}")
        for l, L in enumerate(self.levels):
            co = l == self.nlev - 1
            lines.append(f"level {l} {L['nodes']} {L['b']} {L['nnzb']} {0 if co else L['nnzb_P']} "
                         f"{0 if co else L['n_agg']}")
        with open(os.path.join(path, "amgf_hierarchy.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")

        def w(name, a, dt):
            np.ascontiguousarray(a, dtype=dt).astype(np.dtype(dt).newbyteorder("<")).tofile(os.path.join(path, name))

        for l in range(self.nlev):
            for which, stem, dt in ((0, "A_ptr.i32", np.int32), (1, "A_col.i32", np.int32), (2, "A_val.f64", np.float64),
                                    (9, "l1.f64", np.float64)):
                w(f"L{l}_{stem}", self.get(which, l), dt)
            if l < self.nlev - 1:
                for which, stem, dt in ((3, "P_ptr.i32", np.int32), (4, "P_col.i32", np.int32),
                                        (5, "P_val.f64", np.float64), (6, "R_ptr.i32", np.int32),
                                        (7, "R_col.i32", np.int32), (8, "R_val.f64", np.float64)):
                    w(f"L{l}_{stem}", self.get(which, l), dt)
        w("Z.i32", self.get(20), np.int32)
        w("pi.i32", self.get(25), np.int32)
        w("Lw.f64", self.get(22) if self.nc else np.zeros(0), np.float64)
        w("Lc.f64", self.get(24), np.float64)

    # --- operators ---
    def spmv(self, x, level=0):
        x = _c(x, np.float64); y = np.zeros_like(x)
        lib().orc_spmv(self.h, level, _p(x), _p(y))
        return y

    def vcycle(self, b):
        b = _c(b, np.float64); x = np.zeros_like(b)
        lib().orc_vcycle(self.h, _p(b), _p(x))
        return x

    def apply(self, r):
        r = _c(r, np.float64); z = np.zeros_like(r)
        lib().orc_apply(self.h, _p(r), _p(z))
        return z

    def filter_solve(self, v):
        v = _c(v, np.float64); y = np.zeros_like(v)
        lib().orc_filter_solve(self.h, _p(v), _p(y))
        return y

    def pcg(self, b, rtol=1e-8, maxit=5000, precond="amgf"):
        b = _c(b, np.float64); x = np.zeros_like(b)
        it = ctypes.c_int(0); rr = ctypes.c_double(0)
        hist = np.zeros(maxit + 1)
        st = lib().orc_pcg(self.h, _p(b), _p(x), rtol, maxit, 0 if precond == "amgf" else 1,
                           ctypes.byref(it), ctypes.byref(rr), _p(hist))
        if st < 0:
            raise OracleError(st, lib().orc_last_error().decode())
        return x, dict(iterations=it.value, relres=rr.value, converged=(st == 0), history=hist[:it.value + 1])
