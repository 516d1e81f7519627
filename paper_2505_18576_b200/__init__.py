"""B200-native AMGF-PCG (arxiv 2505.18576, "AMG with Filtering").

The compute path is libamgf.so (hand-written sm_100a CUDA, C-ABI in include/amgf.h); this package
is only the argument-marshalling binding.  It never falls back to a CPU implementation: if the
library or a CUDA device is missing, it raises.
"""
from .amgf import AMGF, AmgfError, Config, lib_path, load_library  # noqa: F401
