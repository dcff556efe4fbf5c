"""B200-native DiLoCoX outer-synchronisation path (arxiv 2506.21263).

pseudo-gradient -> warm-started low-rank + q-bit quantisation -> all-gather of the
compressed factors over NVLink -> fused reconstruct / error-feedback / Nesterov, with the
one-step-delay overlap. Device work goes through the C-ABI in include/dlx_b200.h
(libdlx_b200.so, sm_100a); there is no CPU fallback.
"""
from . import layouts  # noqa: F401
from ._lib import (CudaError, Error, FormatError, IoError, NcclError, NumericError,  # noqa: F401
                   ShapeError, ValidationError, lib)

__all__ = ["layouts", "lib", "Error", "ValidationError", "ShapeError", "FormatError",
           "NumericError", "IoError", "CudaError", "NcclError"]
