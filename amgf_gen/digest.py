"""Array digests for the cached-oracle parity fixtures (tests/golden/oracle/).

No method arithmetic: a SHA-256 over the bytes of an array, used by the oracle-only golden script
(tools/oracle_golden.py) to record results too large to commit, and by the GPU parity tests to check
the CUDA path's arrays against them.  Floating-point arrays are hashed after adding +0.0, which maps
-0.0 to +0.0 and leaves every other value (and NaN payloads aside, every bit) unchanged: the digest then
has the same equality semantics as np.array_equal, the comparison the in-memory parity tests use
(reading R3: the banded factor may hold +0 where the dense factor holds -0 and vice versa).
"""
from __future__ import annotations

import hashlib

import numpy as np


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    if a.dtype.kind == "f":
        a = np.ascontiguousarray(a.astype(np.float64) + 0.0)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode() + b"|" + str(a.shape).encode() + b"|")
    h.update(memoryview(a).cast("B"))
    return h.hexdigest()


def sample_hex(x, count: int = 16) -> dict:
    """count entries of a vector at fixed, evenly spread indices, as exact float.hex strings."""
    x = np.asarray(x, dtype=np.float64).ravel()
    if x.size == 0:
        return {}
    idx = np.unique(np.linspace(0, x.size - 1, count).astype(np.int64))
    return {int(i): float(x[i]).hex() for i in idx}


def probe_vector(n: int, seed: int) -> np.ndarray:
    """The seeded probe right-hand side both sides apply the operators to."""
    return np.random.default_rng(seed).standard_normal(n)


# Hierarchy arrays compared between the oracle and the CUDA path, by the `which` codes both sides'
# getters share (oracle.Oracle.get / AMGF.get; include/amgf.h amgf_level_get).
LEVEL_ITEMS = {0: "A.ptr", 1: "A.col", 2: "A.val", 9: "l1", 15: "comp"}
TRANSFER_ITEMS = {10: "agg", 14: "root", 12: "lambda_omega", 3: "P.ptr", 4: "P.col", 5: "P.val",
                  6: "R.ptr", 7: "R.col", 8: "R.val"}


def hierarchy_items(nlev: int):
    """[(key, which, level)] for every compared array of an nlev-level hierarchy."""
    out = [("Z", 20, 0)]
    for l in range(nlev):
        out += [(f"L{l}/{nm}", w, l) for w, nm in LEVEL_ITEMS.items()]
        if l < nlev - 1:
            out += [(f"L{l}/{nm}", w, l) for w, nm in TRANSFER_ITEMS.items()]
            out.append((f"L{l + 1}/near_null", 11, l + 1))
    return out
