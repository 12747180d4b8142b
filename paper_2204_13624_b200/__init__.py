"""B200-native ComBo Lippmann-Schwinger hot path (arXiv:2204.13624).

The product is the C-ABI shared library ``libcombo_cuda.so`` (include/combo_cuda.h)
built from ``csrc/`` for sm_100a. This package is a thin ctypes mirror of the
reference's C++ solver / material API (same names and semantics as
/root/reference/proj/include/combo/*.hpp) used by the tests and bench.py.
There is no CPU fallback: every call goes through the CUDA library and raises
if it is missing or no GPU is present.
"""
from .combo import (  # noqa: F401
    ComboError,
    Context,
    CellMaterials,
    SolverConfig,
    LaminateOptions,
    neo_hookean,
    neo_hookean_enu,
    linear,
    iso_mandel,
    lib_path,
    load_library,
    GREEN,
    SCHEME,
    slab_row,
    chunk_range,
)
