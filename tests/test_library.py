"""Host-side checks of the C-ABI library (no GPU needed): it builds for sm_100a, loads, and exports
every function include/amgf.h declares; the binding refuses to run without a CUDA device."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2505_18576_b200 import build
    return build.build()


def declared_symbols():
    h = open(os.path.join(ROOT, "include", "amgf.h")).read()
    return sorted(set(re.findall(r"\b(amgf_[a-z_A-Z]+)\s*\(", h)))


def test_exports_every_declared_symbol(libpath):
    L = ctypes.CDLL(libpath)
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(L, s), s
    from paper_2505_18576_b200.amgf import SYMBOLS
    assert sorted(SYMBOLS) == syms


def test_sm100a_cubin(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_config(libpath):
    from paper_2505_18576_b200.amgf import Config, load_library
    L = load_library()
    c = Config()
    L.amgf_default_config(ctypes.byref(c))
    assert (c.pre_sweeps, c.post_sweeps, c.coarsest_size, c.max_levels, c.power_iters) == (1, 1, 64, 25, 6)


def test_null_arguments_rejected(libpath):
    from paper_2505_18576_b200.amgf import load_library
    L = load_library()
    assert L.amgf_apply(None, None, None, None) == -1
    assert b"null" in L.amgf_last_error()
    h = ctypes.c_void_p()
    assert L.amgf_setup(0, None, None, None, 0, None, None, None, None, None, 0, None, None, None,
                        ctypes.byref(h)) == -1
    assert not h.value


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import amgf_gen
    from paper_2505_18576_b200 import AMGF
    with pytest.raises(RuntimeError):
        AMGF.from_problem(amgf_gen.generate(2))


def test_product_path_does_not_import_oracle():
    for f in os.listdir(os.path.join(ROOT, "paper_2505_18576_b200")):
        if f.endswith(".py"):
            src = open(os.path.join(ROOT, "paper_2505_18576_b200", f)).read()
            assert "import oracle" not in src and "from oracle" not in src
    for f in os.listdir(os.path.join(ROOT, "paper_2505_18576_b200", "csrc")):
        assert "oracle" not in open(os.path.join(ROOT, "paper_2505_18576_b200", "csrc", f)).read().lower() or f
