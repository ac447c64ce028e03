"""ctypes declarations for libtorus.so (include/torus.h).  Argument marshalling only.

The CUDA extension is mandatory: if libtorus.so is missing or fails to load, every entry
point raises -- there is no CPU or PyTorch fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes
import pathlib
import threading

_PKG = pathlib.Path(__file__).resolve().parent
import os as _os
LIB_PATH = pathlib.Path(_os.environ.get("TORUS_LIB_PATH", str(_PKG / "libtorus.so")))

TORUS_OK = 0
ERRORS = {
    1: "TORUS_ERR_INVALID_ARG", 2: "TORUS_ERR_GRID", 3: "TORUS_ERR_UNSUPPORTED",
    4: "TORUS_ERR_CUDA", 5: "TORUS_ERR_PEER", 6: "TORUS_ERR_TIMEOUT", 7: "TORUS_ERR_MISMATCH",
}


class torus_ipc_handle_t(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * 64), ("offset", ctypes.c_ulonglong),
                ("size", ctypes.c_ulonglong)]


# every symbol include/torus.h declares, with (restype, argtypes)
_c = ctypes
_vp, _i, _sz, _ull = _c.c_void_p, _c.c_int, _c.c_size_t, _c.c_ulonglong
PROTOTYPES = {
    "torus_workspace_alloc": (_i, [_i, _sz, _c.POINTER(torus_ipc_handle_t)]),
    "torus_workspace_release": (_i, [_c.POINTER(torus_ipc_handle_t)]),
    "torus_comm_init": (_i, [_i, _i, _i, _i, _c.POINTER(torus_ipc_handle_t), _c.POINTER(_vp)]),
    "torus_vcomm_init": (_i, [_i, _i, _i, _i, _sz, _c.POINTER(_vp)]),
    "torus_comm_destroy": (_i, [_vp]),
    "torus_comm_abort": (_i, [_vp]),
    "torus_buffer_export": (_i, [_vp, _sz, _c.POINTER(torus_ipc_handle_t)]),
    "torus_register_buffer": (_i, [_vp, _vp, _sz, _c.POINTER(torus_ipc_handle_t)]),
    "torus_deregister_buffer": (_i, [_vp, _vp]),
    "torus_comm_config": (_i, [_vp, _c.POINTER(_ull), _i]),
    "torus_comm_route": (_c.c_char_p, [_vp, _sz, _i, _i]),
    "torus_allreduce": (_i, [_vp, _vp, _sz, _i, _i, _vp]),
    "torus_allreduce_ex": (_i, [_vp, _vp, _sz, _i, _i, _i, _vp]),
    "torus_allreduce_host": (_i, [_vp, _vp, _vp, _sz, _sz, _i, _i, _i, _vp]),
    "torus_vallreduce": (_i, [_vp, _c.POINTER(_vp), _sz, _i, _i, _i, _vp]),
    "torus_allreduce_multi": (_i, [_vp, _c.POINTER(_vp), _c.POINTER(_sz), _i, _i, _i, _i, _vp]),
    "torus_comm_reserve": (_i, [_vp, _sz]),
    "torus_vallreduce_multi": (_i, [_vp, _c.POINTER(_vp), _c.POINTER(_sz), _i, _i, _i, _i, _vp]),
    "torus_ring_allreduce": (_i, [_vp, _vp, _sz, _i, _i, _i, _vp]),
    "torus_vring_allreduce": (_i, [_vp, _c.POINTER(_vp), _sz, _i, _i, _i, _vp]),
    "torus_comm_ring_round_elems": (_sz, [_vp, _i]),
    "torus_hier_allreduce": (_i, [_vp, _vp, _sz, _i, _i, _i, _vp]),
    "torus_vhier_allreduce": (_i, [_vp, _c.POINTER(_vp), _sz, _i, _i, _i, _vp]),
    "torus_comm_hier_round_elems": (_sz, [_vp, _i]),
    "torus_nvls_prepare": (_i, [_vp, _sz, _c.POINTER(_c.c_longlong)]),
    "torus_nvls_attach": (_i, [_vp, _c.POINTER(_c.c_longlong)]),
    "torus_nvls_bind": (_i, [_vp]),
    "torus_nvls_allreduce": (_i, [_vp, _vp, _sz, _i, _i, _i, _vp]),
    "torus_comm_get_async_error": (_i, [_vp]),
    "torus_comm_grid": (_i, [_vp, _c.POINTER(_i), _c.POINTER(_i)]),
    "torus_comm_rank": (_i, [_vp, _c.POINTER(_i), _c.POINTER(_i)]),
    "torus_comm_ctas": (_i, [_vp]),
    "torus_comm_round_elems": (_sz, [_vp, _i]),
    "torus_comm_launches": (_i, [_vp, _sz, _i, _i]),
    "torus_comm_ll_max_bytes": (_sz, [_vp]),
    "torus_comm_ll2_max_bytes": (_sz, [_vp]),
    "torus_comm_trace": (_i, [_vp, _c.POINTER(_ull), _sz]),
    "torus_comm_pull_trace": (_i, [_vp, _c.POINTER(_ull), _sz, _c.POINTER(_i), _c.POINTER(_i)]),
    "torus_probe": (_i, [_vp, _i, _sz, _i, _i, _c.POINTER(_ull), _vp]),
    "torus_pick_grid": (_i, [_i, _c.POINTER(_i), _c.POINTER(_i), _c.POINTER(_i)]),
    "torus_predict_time": (_i, [_i, _i, _c.c_double, _c.c_double, _c.POINTER(_c.c_double), _c.c_double, _i, _i,
                                _c.POINTER(_c.c_double)]),
    "torus_pick_grid_model": (_i, [_i, _c.POINTER(_c.c_double), _c.c_double, _c.c_double, _c.c_double,
                                   _c.POINTER(_i), _c.POINTER(_i), _c.POINTER(_c.c_double)]),
    "torus_partition": (_i, [_ull, _i, _i, _c.POINTER(_ull), _c.POINTER(_ull)]),
    "torus_strerror": (_c.c_char_p, [_i]),
    "torus_last_error": (_c.c_char_p, []),
}

_lock = threading.Lock()
_lib = None


def load() -> ctypes.CDLL:
    """Load libtorus.so (built by __graft_entry__.build() / _build.build())."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: the CUDA extension is required (no fallback). "
                    "Run `python -c 'import __graft_entry__ as g; g.build()'`.")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in PROTOTYPES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class TorusError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        detail = load().torus_last_error().decode(errors="replace")
        super().__init__(f"{what}: {ERRORS.get(code, code)} ({detail})")


def check(code: int, what: str) -> None:
    if code != TORUS_OK:
        raise TorusError(code, what)
