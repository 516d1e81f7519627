"""ctypes binding of libamgf.so (names follow include/amgf.h).  Marshalling only: every step of the
setup and of the solve runs in the library's CUDA kernels.  torch provides device memory and streams.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libamgf.so")
_lib = None

STATUS = {0: "AMGF_OK", 1: "AMGF_NOT_CONVERGED", -1: "AMGF_ERR_ARG", -2: "AMGF_ERR_NONFINITE",
          -3: "AMGF_ERR_DOMAIN", -4: "AMGF_ERR_NOT_SPD", -5: "AMGF_ERR_RANK", -6: "AMGF_ERR_BREAKDOWN",
          -7: "AMGF_ERR_CUDA", -8: "AMGF_ERR_OOM", -9: "AMGF_ERR_LIMIT", -10: "AMGF_ERR_FORMAT"}

SYMBOLS = ["amgf_default_config", "amgf_setup", "amgf_update_D", "amgf_update_D_box", "amgf_apply", "amgf_vcycle", "amgf_spmv",
           "amgf_spmv_K", "amgf_pcg_solve", "amgf_pcg_solve_host", "amgf_level_info", "amgf_level_get", "amgf_launch_count",
           "amgf_pcg_history", "amgf_setup_times", "amgf_export", "amgf_import", "amgf_debug_guard_check",
           "amgf_last_error",
           "amgf_destroy"]
MAX_LEVELS = 32


def lib_path() -> str:
    return _LIB_PATH


class Config(ctypes.Structure):
    _fields_ = [("pre_sweeps", ctypes.c_int32), ("post_sweeps", ctypes.c_int32),
                ("coarsest_size", ctypes.c_int32), ("max_levels", ctypes.c_int32),
                ("power_iters", ctypes.c_int32), ("nd_levels", ctypes.c_int32),
                ("smoother", ctypes.c_int32), ("cheb_degree", ctypes.c_int32),
                ("agg_seed", ctypes.c_uint64), ("cheb_ratio", ctypes.c_double),
                ("filter_basis", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class Report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("rel_pres_norm", ctypes.c_double), ("solve_ms", ctypes.c_double), ("setup_ms", ctypes.c_double),
                ("n_levels", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("level_dofs", ctypes.c_int64 * MAX_LEVELS), ("level_nnzb", ctypes.c_int64 * MAX_LEVELS)]

    def as_dict(self):
        nl = self.n_levels
        return dict(iterations=self.iterations, converged=bool(self.converged), relres=self.rel_pres_norm,
                    solve_ms=self.solve_ms, setup_ms=self.setup_ms, n_levels=nl,
                    level_dofs=list(self.level_dofs[:nl]), level_nnzb=list(self.level_nnzb[:nl]))


class AmgfError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


def load_library():
    """Load the in-tree libamgf.so.  Raises if it is missing: there is no fallback path."""
    global _lib
    if _lib is not None:
        return _lib
    # AMGF_LIB: an alternative in-tree build of the same library (A/B timing experiments only)
    path = os.path.join(os.path.dirname(_LIB_PATH), os.environ["AMGF_LIB"]) if os.environ.get("AMGF_LIB") else _LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"libamgf.so not built ({path}); run __graft_entry__.build()")
    L = ctypes.CDLL(path)
    P, I, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_double
    L.amgf_default_config.argtypes = [ctypes.POINTER(Config)]
    L.amgf_setup.argtypes = [I, P, P, P, I, P, P, P, P, P, I, P, ctypes.POINTER(Config), P, ctypes.POINTER(P)]
    L.amgf_setup.restype = I
    L.amgf_update_D.argtypes = [P, P, P]
    L.amgf_update_D.restype = I
    L.amgf_update_D_box.argtypes = [P, P, P, P, P]
    L.amgf_update_D_box.restype = I
    for f in ("amgf_apply", "amgf_vcycle"):
        getattr(L, f).argtypes = [P, P, P, P]
        getattr(L, f).restype = I
    L.amgf_spmv.argtypes = [P, I, P, P, P]
    L.amgf_spmv.restype = I
    L.amgf_spmv_K.argtypes = [P, P, P, P]
    L.amgf_spmv_K.restype = I
    L.amgf_pcg_solve.argtypes = [P, P, P, D, I, I, ctypes.POINTER(Report), P]
    L.amgf_pcg_solve.restype = I
    L.amgf_pcg_solve_host.argtypes = [P, P, P, D, I, I, ctypes.POINTER(Report), P]
    L.amgf_pcg_solve_host.restype = I
    L.amgf_level_info.argtypes = [P, P]
    L.amgf_level_info.restype = I
    L.amgf_level_get.argtypes = [P, I, I, P]
    L.amgf_level_get.restype = I
    L.amgf_setup_times.argtypes = [P, P]
    L.amgf_setup_times.restype = I
    L.amgf_pcg_history.argtypes = [P, I, P, P]
    L.amgf_pcg_history.restype = I
    L.amgf_export.argtypes = [P, ctypes.c_char_p]
    L.amgf_export.restype = I
    L.amgf_import.argtypes = [ctypes.c_char_p, P, ctypes.POINTER(P)]
    L.amgf_import.restype = I
    L.amgf_debug_guard_check.argtypes = [P]
    L.amgf_debug_guard_check.restype = ctypes.c_int64
    L.amgf_launch_count.argtypes = [P]
    L.amgf_launch_count.restype = ctypes.c_int64
    L.amgf_last_error.restype = ctypes.c_char_p
    L.amgf_destroy.argtypes = [P]
    _lib = L
    return L


def _check(st, allow=(0,)):
    if st not in allow:
        raise AmgfError(st, load_library().amgf_last_error().decode())
    return st


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class AMGF:
    """AMGF preconditioner + PCG for S = K + J^T D J on one GPU (C-ABI handle wrapper)."""

    def __init__(self, nodes, K_ptr, K_col, K_val, J_ptr, J_col, J_val, D, Z, B_nns, config=None, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("AMGF needs a CUDA device (no CPU fallback)")
        L = load_library()
        self.torch = torch
        dev = torch.device("cuda")

        def t(a, dt):
            if isinstance(a, np.ndarray):
                return torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)
            return a.to(dev, dt).contiguous()

        self._in = dict(K_ptr=t(K_ptr, torch.int32), K_col=t(K_col, torch.int32), K_val=t(K_val, torch.float64),
                        J_ptr=t(J_ptr, torch.int32), J_col=t(J_col, torch.int32), J_val=t(J_val, torch.float64),
                        D=t(D, torch.float64), Z=None if Z is None else t(Z, torch.int32),
                        B=t(B_nns, torch.float64))
        self.nodes = int(nodes)
        self.n = 3 * self.nodes
        self.m = self._in["J_ptr"].numel() - 1
        cfg = Config()
        L.amgf_default_config(ctypes.byref(cfg))
        for k, v in (config or {}).items():
            setattr(cfg, k, v)
        self.config = cfg
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        h = ctypes.c_void_p()
        i = self._in
        st = L.amgf_setup(self.nodes, _ptr(i["K_ptr"]), _ptr(i["K_col"]), _ptr(i["K_val"]), self.m,
                          _ptr(i["J_ptr"]), _ptr(i["J_col"]), _ptr(i["J_val"]), _ptr(i["D"]), _ptr(i["Z"]),
                          0 if i["Z"] is None else i["Z"].numel(), _ptr(i["B"]), ctypes.byref(cfg),
                          ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h))
        _check(st)
        self.h = h
        self._load_info()

    def _load_info(self):
        L = load_library()
        info = np.zeros(4 + 6 * 32 + 5, dtype=np.int64)
        _check(L.amgf_level_info(self.h, info.ctypes.data_as(ctypes.c_void_p)))
        self.nlev, self.nc, self.nco, self.bw = (int(v) for v in info[:4])
        self.levels = [dict(nodes=int(info[4 + 6 * l]), b=int(info[5 + 6 * l]), nnzb=int(info[6 + 6 * l]),
                            nnzb_P=int(info[7 + 6 * l]), n_agg=int(info[8 + 6 * l]), slots=int(info[9 + 6 * l]))
                       for l in range(self.nlev)]
        self.loff_size, self.nd_nblocks = int(info[4 + 6 * 32]), int(info[5 + 6 * 32])
        self.tail_level, self.tail_ncta = int(info[6 + 6 * 32]), int(info[7 + 6 * 32])
        self.nf = int(info[8 + 6 * 32])

    @classmethod
    def import_dir(cls, path, stream=None):
        """Handle on a hierarchy written in the amgf_export format (by amgf_export or by the oracle)."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("AMGF needs a CUDA device (no CPU fallback)")
        L = load_library()
        self = cls.__new__(cls)
        self.torch = torch
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self._in = {}
        h = ctypes.c_void_p()
        _check(L.amgf_import(os.fsencode(path), ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h)))
        self.h = h
        self.config = None
        self._load_info()
        self.nodes = self.levels[0]["nodes"]
        self.n = 3 * self.nodes
        self.m = 0
        self.imported = True
        return self

    def export(self, path):
        """Write this handle's hierarchy and factors to the existing directory `path` (amgf_export)."""
        _check(load_library().amgf_export(self.h, os.fsencode(path)))

    @classmethod
    def from_problem(cls, p, D=None, Z="lattice", config=None, stream=None):
        Zv = p.Z if isinstance(Z, str) and Z == "lattice" else Z
        return cls(p.nodes, p.K_ptr, p.K_col, p.K_val, p.J_ptr, p.J_col, p.J_val,
                   p.D if D is None else D, Zv, p.B_nns, config=config, stream=stream)

    def close(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.amgf_destroy(h)
        self.h = None

    def __del__(self):
        self.close()

    @property
    def _s(self):
        return ctypes.c_void_p(self.stream.cuda_stream)

    def _vec(self, x=None, n=None):
        T = self.torch
        if x is None:
            return T.empty(n if n is not None else self.n, dtype=T.float64, device="cuda")
        if isinstance(x, np.ndarray):
            x = T.from_numpy(np.ascontiguousarray(x))
        if n is not None and x.numel() != n:
            raise ValueError(f"vector of {x.numel()} entries, expected {n}")
        return x if (x.is_cuda and x.dtype == T.float64 and x.is_contiguous()) else x.to("cuda", T.float64).contiguous()

    def update_D(self, D):
        D = self._vec(D, None if getattr(self, "imported", False) else self.m)  # imported: the library rejects
        self._in["D_upd"] = D
        _check(load_library().amgf_update_D(self.h, _ptr(D), self._s))

    def update_D_box(self, D, D_lo=None, D_up=None):
        """Numeric re-setup of A~ = K + J^T D J + diag(D_lo) + diag(D_up) (bound constraints)."""
        D = self._vec(D, self.m)
        lo = None if D_lo is None else self._vec(D_lo, self.n)
        up = None if D_up is None else self._vec(D_up, self.n)
        self._in["D_upd"], self._in["D_lo"], self._in["D_up"] = D, lo, up
        _check(load_library().amgf_update_D_box(self.h, _ptr(D), _ptr(lo), _ptr(up), self._s))

    def apply(self, r, out=None):
        r = self._vec(r, self.n)
        z = out if out is not None else self._vec(n=self.n)
        _check(load_library().amgf_apply(self.h, _ptr(r), _ptr(z), self._s))
        return z

    def vcycle(self, b, out=None):
        b = self._vec(b, self.n)
        x = out if out is not None else self._vec(n=self.n)
        _check(load_library().amgf_vcycle(self.h, _ptr(b), _ptr(x), self._s))
        return x

    def spmv(self, x, level=0, out=None):
        x = self._vec(x, self.levels[level]["nodes"] * self.levels[level]["b"])
        y = out if out is not None else self._vec(n=x.numel())
        _check(load_library().amgf_spmv(self.h, level, _ptr(x), _ptr(y), self._s))
        return y

    def spmv_K(self, x, out=None):
        """y = K x (the stiffness matrix of the setup; interior-point residuals)."""
        x = self._vec(x, self.n)
        y = out if out is not None else self._vec(n=self.n)
        _check(load_library().amgf_spmv_K(self.h, _ptr(x), _ptr(y), self._s))
        return y

    def pcg(self, b, rtol=1e-8, max_it=5000, precond="amgf", out=None):
        b = self._vec(b, self.n)
        x = out if out is not None else self._vec(n=self.n)
        rep = Report()
        st = load_library().amgf_pcg_solve(self.h, _ptr(b), _ptr(x), rtol, max_it, 0 if precond == "amgf" else 1,
                                           ctypes.byref(rep), self._s)
        _check(st, allow=(0, 1))
        return x, rep.as_dict()

    def pcg_host(self, b_host, x_host, rtol=1e-8, max_it=5000, precond="amgf"):
        """b_host, x_host: CPU float64 tensors (pinned for async copies)."""
        if b_host.numel() != self.n or x_host.numel() != self.n or b_host.is_cuda or x_host.is_cuda:
            raise ValueError("pcg_host needs host (CPU) float64 tensors of n entries")
        rep = Report()
        st = load_library().amgf_pcg_solve_host(self.h, ctypes.c_void_p(b_host.data_ptr()),
                                                ctypes.c_void_p(x_host.data_ptr()), rtol, max_it,
                                                0 if precond == "amgf" else 1, ctypes.byref(rep), self._s)
        _check(st, allow=(0, 1))
        return rep.as_dict()

    def setup_times(self):
        """Phase times (ms) of the last update_D: total, S, hierarchy, coarsest, A_w factor (side stream)."""
        ms = np.zeros(5)
        _check(load_library().amgf_setup_times(self.h, ms.ctypes.data_as(ctypes.c_void_p)))
        return dict(zip(("total", "S", "hierarchy", "coarsest", "A_w_factor_side"), ms.tolist()))

    def history(self, n):
        """alpha_k, beta_k (k = 1..n) of the last PCG solve (numpy arrays)."""
        a = np.zeros(n)
        bt = np.zeros(n)
        _check(load_library().amgf_pcg_history(self.h, n, a.ctypes.data_as(ctypes.c_void_p),
                                                bt.ctypes.data_as(ctypes.c_void_p)))
        return a, bt

    def guard_violations(self) -> int:
        """Overwritten guard zones of this handle (AMGF_GUARD=1 debug allocations; -2 if not enabled)."""
        return int(load_library().amgf_debug_guard_check(self.h))

    @property
    def launches(self) -> int:
        return int(load_library().amgf_launch_count(self.h))

    @staticmethod
    def _band_stride(bw):
        R = (bw + 31) // 32 + 1
        return 32 * R if R <= 8 else (bw + 2) & ~1

    def get(self, which, level=0):
        Lv = self.levels[level]
        b, nodes = Lv["b"], Lv["nodes"]
        R = (self.bw + 31) // 32 + 1
        W = 32 * R if R <= 8 else (self.bw + 2) & ~1
        shapes = {0: (nodes + 1, np.int32), 1: (Lv["nnzb"], np.int32), 2: ((Lv["nnzb"], b * b), np.float64),
                  3: (nodes + 1, np.int32), 4: (Lv["nnzb_P"], np.int32), 5: ((Lv["nnzb_P"], b * 6), np.float64),
                  6: (Lv["n_agg"] + 1, np.int32), 7: (Lv["nnzb_P"], np.int32),
                  8: ((Lv["nnzb_P"], 6 * b), np.float64), 9: (nodes * b, np.float64), 10: (nodes, np.int32),
                  11: ((nodes * b, 6), np.float64), 12: (2, np.float64), 14: (nodes, np.int32),
                  15: (nodes, np.int32), 20: (self.nc, np.int32), 22: ((self.nf, W), np.float64),
                  23: (self.loff_size, np.float64), 25: (self.nf, np.int32),
                  24: ((self.nco, self._band_stride(self.nco - 1)), np.float64)}
        if which == 27:
            dt = np.dtype([("p0", np.int32), ("len", np.int32), ("kind", np.int32), ("t0", np.int32),
                           ("off", np.int64), ("level", np.int32), ("rs", np.int32)])
            out = np.zeros(self.nd_nblocks, dtype=dt)
            _check(load_library().amgf_level_get(self.h, which, level, out.ctypes.data_as(ctypes.c_void_p)))
            return out
        shape, dt = shapes[which]
        out = np.zeros(shape, dtype=dt)
        _check(load_library().amgf_level_get(self.h, which, level, out.ctypes.data_as(ctypes.c_void_p)))
        return out
