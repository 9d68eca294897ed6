"""B200-native sketched GMRES / sketched Rayleigh-Ritz (arXiv 2111.00113).

Hot path: k-truncated Arnoldi basis + sparse-sign sketch + small sketched solves, all in
hand-written sm_100a CUDA kernels behind the C-ABI of include/sks.h (libsks.so).  This
package is the thin Python binding (marshalling only).  No CPU fallback.
"""
from .api import (  # noqa: F401
    Context, StencilOperator, CsrOperator, SgmresResult, SksError, partition, get_unique_id, LoopbackGroup,
)
from ._lib import load, LIBPATH, EXPORTS  # noqa: F401

__all__ = ["Context", "LoopbackGroup", "StencilOperator", "CsrOperator", "SgmresResult", "SksError", "partition",
           "get_unique_id", "load", "LIBPATH", "EXPORTS"]
