"""B200-native (sm_100a) 2D selective scan of 2DMamba (arXiv 2412.00678).

The hot path -- tiled 2D selective scan forward and backward -- runs in
hand-written CUDA (lib/libscan2d_cuda.so, C ABI in include/scan2d_cuda.h).
Importing this package fails loudly when that library has not been built.
"""
from . import _native  # noqa: F401  (raises ImportError when the CUDA library is missing)
from .api import (GradBundle, SavedForward, Scan2dBandOp, Scan2dFunction, Scan2dOp,  # noqa: F401
                  TiledForwardResult, scan2d, tiled_scan_2d_backward, tiled_scan_2d_forward, train_host)

__all__ = [
    "GradBundle",
    "SavedForward",
    "Scan2dBandOp",
    "Scan2dFunction",
    "Scan2dOp",
    "TiledForwardResult",
    "scan2d",
    "tiled_scan_2d_backward",
    "tiled_scan_2d_forward",
    "train_host",
]
