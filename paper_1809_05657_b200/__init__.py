"""B200-native HDArray def/use exchange runtime (arXiv:1809.05657).

The product is libhdarray.so (C-ABI in include/hdarray.h, CUDA for sm_100a);
this package is its thin ctypes binding.  See DESIGN.md.
"""
from .hdarray import *  # noqa: F401,F403
from .hdarray import HDArray, HDAError, lib, plan_cells, trapezoid  # noqa: F401
