"""Full-size parity against cached oracle results (tests/golden/oracle/, written by tools/oracle_golden.py,
which runs the unchanged plain oracle with its dense A_w factor and imports nothing but oracle/ and
amgf_gen/).

For every cached system -- cfg 3's ten interior-point-like systems (D up to 1e12; the bench workload, in
the bench's launch configuration: one handle, amgf_update_D per system, the device PCG loop) and cfg 4
(5.48M dofs, rtol 1e-10, inclusion E = 1e3) -- the CUDA path must reproduce, bit for bit (DESIGN.md
section 3; digests have np.array_equal semantics, amgf_gen/digest.py):
  * every hierarchy array (operators, l1 diagonals, aggregates, roots, prolongators, restrictions,
    near-null spaces, lambda/omega) and Z, pi;
  * the dense Cholesky factor of A_w[pi, pi] (rebuilt from the GPU's nested-dissection storage) and of the
    coarsest operator;
  * S x, B x (V-cycle) and M x (AMGF apply) of a seeded probe x;
  * the PCG iteration count, the final relative preconditioned residual and the solution
    (PAPER.md:368 criterion; Def. AMGF).
"""
import glob
import json
import os

import numpy as np
import pytest

import amgf_gen as gen
from amgf_gen.digest import digest, hierarchy_items, probe_vector

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
FILES = sorted(glob.glob(os.path.join(HERE, "golden", "oracle", "cfg*_s*.json")),
               key=lambda f: (int(os.path.basename(f)[3]), int(os.path.basename(f).split("_s")[1][:-5])))


def _load(f):
    return json.load(open(f))


@pytest.fixture(scope="module")
def handles():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2505_18576_b200 as m
    m.load_library()
    cache = {}
    yield m, cache
    for p, g in cache.values():
        g.close()


def gpu_dense_factor(g):
    nc, bw = g.nc, g.bw
    band = g.get(22)
    L = np.zeros((nc, nc))
    for t in range(bw + 1):
        i = np.arange(t, nc)
        L[i, i - t] = band[i, bw - t]
    if g.loff_size:
        off = g.get(23)
        for b in g.get(27):
            if b["kind"] == 1:
                p0, ln, t0, o, rs = int(b["p0"]), int(b["len"]), int(b["t0"]), int(b["off"]), int(b["rs"])
                L[p0:p0 + ln, t0:p0] = off[o:o + rs * ln].reshape(ln, rs)[:, :p0 - t0]
    return L


def gpu_dense_coarsest(g):
    n = g.nco
    band = g.get(24)
    L = np.zeros((n, n))
    for t in range(n):
        i = np.arange(t, n)
        L[i, i - t] = band[i, n - 1 - t]
    return L


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f)[:-5] for f in FILES])
def test_cached_oracle_parity(handles, path):
    m, cache = handles
    import torch
    rec = _load(path)
    cfg, s = rec["cfg"], rec["system"]
    if cfg not in cache:
        for k in list(cache):          # one full-size handle resident at a time
            cache.pop(k)[1].close()
        torch.cuda.empty_cache()
        p = gen.config(cfg)
        cache[cfg] = (p, m.AMGF.from_problem(p, D=p.D_seq[s]))
    p, g = cache[cfg]
    assert digest(p.D_seq[s]) == rec["D_digest"]
    g.update_D(p.D_seq[s])             # the bench's per-system step: numeric re-setup for this D
    assert (g.nlev, g.nc, g.nco, g.bw) == (rec["nlev"], rec["nc"], rec["nco"], rec["bw"])
    bad = [key for key, w, l in hierarchy_items(g.nlev) if digest(g.get(w, l)) != rec["arrays"][key]]
    assert not bad, f"hierarchy arrays differ from the oracle: {bad}"
    assert digest(g.get(25)) == rec["arrays"]["pi"]
    if g.nc:
        assert digest(gpu_dense_factor(g)) == rec["arrays"]["L_w"], "A_w factor"
    assert digest(gpu_dense_coarsest(g)) == rec["arrays"]["coarsest_L"], "coarsest factor"
    x = probe_vector(p.n, rec["probe_seed"])
    assert digest(g.spmv(x).cpu().numpy()) == rec["probe"]["spmv"], "S x"
    assert digest(g.vcycle(x).cpu().numpy()) == rec["probe"]["vcycle"], "B x"
    z = g.apply(x).cpu().numpy()
    if digest(z) != rec["probe"]["apply"]:
        smp = {int(i): float.fromhex(v) for i, v in rec["probe"]["apply_samples"].items()}
        diff = max(abs(z[i] - v) / max(abs(v), 1e-300) for i, v in smp.items())
        pytest.fail(f"M x differs from the oracle (max sampled relative difference {diff:.3e})")
    b = torch.from_numpy(p.b).cuda()
    xg, rg = g.pcg(b, rtol=rec["pcg"]["rtol"], max_it=5000)
    assert rg["iterations"] == rec["pcg"]["iterations"], (rg["iterations"], rec["pcg"]["iterations"])
    assert float(rg["relres"]).hex() == rec["pcg"]["relres"]
    assert rg["converged"] == rec["pcg"]["converged"]
    assert digest(xg.cpu().numpy()) == rec["pcg"]["x"], "solution"
