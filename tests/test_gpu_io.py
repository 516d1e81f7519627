"""amgf_export / amgf_import on the GPU.

North star: "single preconditioner applies on an identical exported hierarchy".  The oracle writes its own
hierarchy (oracle.Oracle.export, dense factors included); the CUDA path imports it and must apply exactly
that preconditioner: M r, B r, A_l x and whole PCG solves bitwise equal to the oracle's.
The imported hierarchy is built with settings the GPU's own setup is NOT run with here (other power-step
count, l1-Jacobi, other Chebyshev degree), so only the imported data can produce the oracle's bits.
"""
import os

import numpy as np
import pytest

import amgf_gen as gen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def amgf_mod():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2505_18576_b200 as m
    m.load_library()
    return m


def tiny(N=3, matching=False, e_max=8.0, seed=7):
    return gen.generate(N, matching=matching, e_max=[e_max], seed=seed)


def check_import(oracle_lib, amgf_mod, p, tmp_path, rtol=1e-10, **cfg):
    o = oracle_lib.Oracle.from_problem(p, **cfg)
    d = str(tmp_path / "h")
    o.export(d)
    g = amgf_mod.AMGF.import_dir(d)
    assert (g.nlev, g.nc, g.nco) == (o.nlev, o.nc, o.nco)
    rng = np.random.default_rng(123)
    r = rng.standard_normal(p.n)
    for l in range(o.nlev):
        x = rng.standard_normal(o.levels[l]["nodes"] * o.levels[l]["b"])
        assert np.array_equal(g.spmv(x, l).cpu().numpy(), o.spmv(x, l)), ("spmv", l)
    assert np.array_equal(g.vcycle(r).cpu().numpy(), o.vcycle(r)), "vcycle"
    assert np.array_equal(g.apply(r).cpu().numpy(), o.apply(r)), "apply"
    xo, ro = o.pcg(p.b, rtol=rtol)
    xg, rg = g.pcg(p.b, rtol=rtol)
    assert rg["iterations"] == ro["iterations"] and rg["relres"] == ro["relres"]
    assert np.array_equal(xg.cpu().numpy(), xo)
    assert rg["n_levels"] == o.nlev
    assert rg["level_dofs"] == [L["nodes"] * L["b"] for L in o.levels]
    assert rg["level_nnzb"] == [L["nnzb"] for L in o.levels]
    return o, g


@pytest.mark.parametrize("cfg", [
    dict(coarsest_size=16),
    dict(coarsest_size=16, power_iters=10),
    dict(coarsest_size=16, smoother=0),
    dict(coarsest_size=16, cheb_degree=3, cheb_ratio=30.0, nd_levels=1),
    dict(coarsest_size=10 ** 6),                     # one level: the coarsest factor is the whole solve
])
def test_import_oracle_hierarchy_tiny(oracle_lib, amgf_mod, tmp_path, cfg):
    check_import(oracle_lib, amgf_mod, tiny(), tmp_path, **cfg)


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_import_oracle_hierarchy_configs(oracle_lib, amgf_mod, tmp_path, cfg):
    p = gen.config(cfg)
    check_import(oracle_lib, amgf_mod, p, tmp_path, rtol=p.rtol, power_iters=10)


def test_export_matches_oracle(oracle_lib, amgf_mod, tmp_path):
    """The GPU's own hierarchy, exported, holds the oracle's arrays (same values; +-0 of exact zeros aside)."""
    p = gen.config(1)
    o = oracle_lib.Oracle.from_problem(p)
    g = amgf_mod.AMGF.from_problem(p)
    do, dg = tmp_path / "o", tmp_path / "g"
    o.export(str(do))
    os.makedirs(dg)
    g.export(str(dg))
    assert sorted(os.listdir(do)) == sorted(os.listdir(dg))
    assert open(do / "amgf_hierarchy.txt").read().split("\n")[:6] == open(dg / "amgf_hierarchy.txt").read().split("\n")[:6]
    for f in os.listdir(do):
        if f.endswith(".txt"):
            continue
        dt = np.int32 if f.endswith(".i32") else np.float64
        assert np.array_equal(np.fromfile(do / f, dt), np.fromfile(dg / f, dt)), f
    # and the GPU's export re-imports to the same preconditioner
    h = amgf_mod.AMGF.import_dir(str(dg))
    r = np.random.default_rng(5).standard_normal(p.n)
    assert np.array_equal(h.apply(r).cpu().numpy(), g.apply(r).cpu().numpy())


def test_import_errors(oracle_lib, amgf_mod, tmp_path):
    p = tiny()
    o = oracle_lib.Oracle.from_problem(p, coarsest_size=16)
    d = tmp_path / "h"
    o.export(str(d))
    g = amgf_mod.AMGF.import_dir(str(d))
    with pytest.raises(amgf_mod.AmgfError) as e:       # no K, J, D on an imported handle
        g.update_D(np.ones(p.m))
    assert e.value.code == -1
    # a factor entry outside the nested-dissection structure
    nc = o.nc
    Lw = np.fromfile(d / "Lw.f64", np.float64).reshape(nc, nc)
    bad = Lw.copy()
    bad[nc - 1, 0] = 1e-3
    bad.tofile(d / "Lw.f64")
    with pytest.raises(amgf_mod.AmgfError) as e:
        amgf_mod.AMGF.import_dir(str(d))
    assert e.value.code == -10
    Lw.tofile(d / "Lw.f64")
    # truncated operator file
    a = np.fromfile(d / "L0_A_val.f64", np.float64)
    a[:-1].tofile(d / "L0_A_val.f64")
    with pytest.raises(amgf_mod.AmgfError) as e:
        amgf_mod.AMGF.import_dir(str(d))
    assert e.value.code == -10
    a.tofile(d / "L0_A_val.f64")
    # wrong elimination order
    pi = np.fromfile(d / "pi.i32", np.int32)
    pi[[0, 1]] = pi[[1, 0]]
    pi.tofile(d / "pi.i32")
    with pytest.raises(amgf_mod.AmgfError) as e:
        amgf_mod.AMGF.import_dir(str(d))
    assert e.value.code == -10
    with pytest.raises(amgf_mod.AmgfError) as e:
        amgf_mod.AMGF.import_dir(str(tmp_path / "missing"))
    assert e.value.code == -10
