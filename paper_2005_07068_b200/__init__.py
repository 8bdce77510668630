"""B200-native swarm scorer for arXiv 2005.07068 (26-DOF hand pose, PSO + ray-cast model).

The product is the C-ABI library ``libhp.so`` (include/hp.h, CUDA for sm_100a) and this
thin binding.  See DESIGN.md.
"""
from .hp import (Context, CostParams, FitResult, HandDims, HPError, Intrinsics,  # noqa: F401
                 NDOF, NPRIM, bounds, default_cost, default_dims, default_intrinsics,
                 exported_symbols, intrinsics_from, lib, LIB_PATH)
