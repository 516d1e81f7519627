"""Per-warp timeline of the level-1 SELL SpMV (k_sell_r1) in one V-cycle at cfg 3 (A/B build libamgf_tr.so,
-DAMGF_R1_TRACE): start / end (globaltimer), SM and the warp's longest row; prints the kernel span, warp
duration vs row length, and how many warps are still running over the kernel's lifetime."""
import ctypes
import os
import sys

os.environ.setdefault("AMGF_LIB", "libamgf_tr.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import amgf_gen  # noqa: E402
from paper_2505_18576_b200 import AMGF  # noqa: E402
from paper_2505_18576_b200.amgf import load_library  # noqa: E402

p = amgf_gen.config(3)
g = AMGF.from_problem(p, D=p.D_seq[5])
b = torch.from_numpy(np.random.default_rng(0).standard_normal(p.n)).cuda()
for _ in range(3):
    g.vcycle(b)
torch.cuda.synchronize()
L = load_library()
buf = (ctypes.c_ulonglong * (8192 * 4))()
L.amgf_debug_r1_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert L.amgf_debug_r1_trace(ctypes.addressof(buf), 8192 * 4) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4)
nrows = int(t[0, 3] >> 32)
nw = (nrows + 31) // 32
t = t[:nw]
t0, t1, sm, ml = t[:, 0].astype(np.int64), t[:, 1].astype(np.int64), t[:, 2], (t[:, 3] & 0xffffffff).astype(np.int64)
base = t0.min()
s, e = (t0 - base) / 1e3, (t1 - base) / 1e3
print(f"nrows {nrows} warps {nw}: kernel span {e.max():.1f} us; warp start max {s.max():.1f} us")
print(f"warp duration us: mean {np.mean(e - s):.1f} p50 {np.median(e - s):.1f} p90 {np.percentile(e - s, 90):.1f} max {np.max(e - s):.1f}")
print(f"warp end us: p10 {np.percentile(e, 10):.1f} p50 {np.median(e):.1f} p90 {np.percentile(e, 90):.1f} max {e.max():.1f}")
for L_ in (20, 30, 40, 50, 60):
    m = (ml >= L_ - 5) & (ml < L_ + 5)
    if m.any():
        print(f"  longest row {L_ - 5}-{L_ + 4} slots: {m.sum()} warps, duration mean {np.mean((e - s)[m]):.1f} us")
for q in np.linspace(0, e.max(), 11):
    print(f"  t={q:5.1f} us: running warps {int(((s <= q) & (e > q)).sum())}")
per_sm = np.bincount(sm.astype(np.int64), weights=e, minlength=148)
cnt = np.bincount(sm.astype(np.int64), minlength=148)
last = np.zeros(148)
for i in range(nw):
    last[int(sm[i])] = max(last[int(sm[i])], e[i])
print(f"per-SM last warp end: min {last[cnt > 0].min():.1f} p50 {np.median(last[cnt > 0]):.1f} max {last.max():.1f} us; warps per SM {cnt.min()}-{cnt.max()}")
