"""B200-native product-to-sum element-matrix fill (arXiv:1703.09619, 3-D Legendre).

Hot path: libp2s_b200.so (sm_100a kernels behind the C-ABI of
include/p2s_b200.h).  This package holds the ctypes binding, the
reference-shaped host API and the benchmark configurations.
"""
from .capi import (ALPHA_EXPSIN, ALPHA_JACOBIAN, ALPHA_SINE, DD, DP, PD, PP, Context,
                   InvalidArgument, P2SError, UnsupportedShape, build, lib, shape_supported)
from .configs import CONFIGS, FillConfig, algorithmic_counts

__all__ = [
    "PP", "DD", "DP", "PD", "ALPHA_SINE", "ALPHA_JACOBIAN", "ALPHA_EXPSIN", "Context", "P2SError",
    "InvalidArgument", "UnsupportedShape", "build", "lib", "shape_supported", "CONFIGS",
    "FillConfig", "algorithmic_counts",
]
