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


def test_product_path_does_not_import_oracle(libpath):
    """The product path never imports, includes, links or loads anything under oracle/ (comments may cite it)."""
    pkg = os.path.join(ROOT, "paper_2505_18576_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
            assert "liboracle" not in src and "amgf_oracle" not in src, f
    for f in os.listdir(os.path.join(pkg, "csrc")):
        src = open(os.path.join(pkg, "csrc", f)).read()
        code = re.sub(r"//[^\n]*|/\*.*?\*/", "", src, flags=re.S)   # strip comments
        assert not re.search(r"#\s*include\s*[<\"][^>\"]*oracle", code), f
        assert "orc_" not in code and "liboracle" not in code and "dlopen" not in code, f
    # the built library neither needs nor references the oracle's library or symbols
    dyn = subprocess.run(["readelf", "-d", libpath], capture_output=True, text=True).stdout
    assert "oracle" not in dyn
    syms = subprocess.run(["nm", "-D", libpath], capture_output=True, text=True).stdout
    assert not re.search(r"\borc_", syms)
    from paper_2505_18576_b200 import build
    assert not any("oracle" in x for x in build.SRC + build.FLAGS)
