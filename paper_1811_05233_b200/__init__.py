"""B200-native 2D-Torus all-reduce (Mikami et al., arXiv 1811.05233, Sec. 2.2).

The product path is libtorus.so (include/torus.h): hand-written sm_100a kernels that
move gradients over NVLink 5 / NVSwitch through CUDA IPC.  This package is the thin
Python binding over that C-ABI.
"""
from .torus import TorusComm, VirtualTorus, partition, pick_grid, pick_grid_model, predict_time  # noqa: F401
from ._lib import TorusError, LIB_PATH  # noqa: F401

__all__ = ["TorusComm", "VirtualTorus", "pick_grid", "pick_grid_model", "predict_time", "partition",
           "TorusError", "LIB_PATH"]
