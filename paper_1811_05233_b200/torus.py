"""Python binding of the 2D-Torus all-reduce.  Argument marshalling only:
every step of the collective runs in libtorus.so's sm_100a kernels.  PyTorch supplies
device memory, streams and the process group used once to exchange IPC handles.

    comm = TorusComm.init(X=2, Y=4)          # one process per GPU, after init_process_group
    comm.all_reduce(grad, op="mean")         # in place, async on the current stream
    comm.all_reduce(grad32, op="mean", wire=torch.float16)   # PAPER.md:121 FP16 comm
"""
from __future__ import annotations

import ctypes
from typing import Sequence

import torch

from . import _lib
from ._lib import check, torus_ipc_handle_t

DTYPES = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2, torch.int32: 3}
OPS = {"sum": 0, "mean": 1}


def _dtype_code(dt) -> int:
    try:
        return DTYPES[dt]
    except KeyError:
        raise TypeError(f"unsupported dtype {dt}; supported: f32, f16, bf16, i32") from None


def _stream_ptr(stream) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def pick_grid(world: int, p2p: Sequence[Sequence[int]] | None = None) -> tuple[int, int]:
    """Topology layer (torus_pick_grid): choose (X, Y) for `world` GPUs."""
    L = _lib.load()
    X, Y = ctypes.c_int(), ctypes.c_int()
    arr = None
    if p2p is not None:
        flat = [int(v) for row in p2p for v in row]
        arr = (ctypes.c_int * len(flat))(*flat)
    check(L.torus_pick_grid(world, arr, ctypes.byref(X), ctypes.byref(Y)), "torus_pick_grid")
    return X.value, Y.value


def _bw_array(bw):
    if bw is None:
        return None
    flat = [float(v) for row in bw for v in row]
    return (ctypes.c_double * len(flat))(*flat)


def predict_time(X: int, Y: int, nbytes: float, alpha_us: float, bw=None, beta_gbs: float = 560.0,
                 algo: str = "torus", schedule: str = "oneshot") -> float:
    """alpha-beta prediction in microseconds (torus_predict_time)."""
    out = ctypes.c_double()
    check(_lib.load().torus_predict_time(X, Y, nbytes, alpha_us, _bw_array(bw), beta_gbs,
                                         {"torus": 0, "ring": 1, "hier": 2}[algo],
                                         {"ring": 0, "oneshot": 1}[schedule], ctypes.byref(out)),
          "torus_predict_time")
    return out.value


def pick_grid_model(world: int, nbytes: float, alpha_us: float, bw=None,
                    beta_gbs: float = 560.0) -> tuple[int, int, float]:
    """Grid with the smallest predicted time (torus_pick_grid_model): (X, Y, predicted us)."""
    X, Y, p = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
    check(_lib.load().torus_pick_grid_model(world, _bw_array(bw), alpha_us, beta_gbs, nbytes,
                                            ctypes.byref(X), ctypes.byref(Y), ctypes.byref(p)),
          "torus_pick_grid_model")
    return X.value, Y.value, p.value


def partition(n: int, parts: int, q: int) -> tuple[list[int], list[int]]:
    """Host partition logic of the library, exported for tests."""
    L = _lib.load()
    off = (ctypes.c_ulonglong * parts)()
    ln = (ctypes.c_ulonglong * parts)()
    check(L.torus_partition(n, parts, q, off, ln), "torus_partition")
    return list(off), list(ln)


def exchange_blobs(blob: bytes, world: int, group=None) -> list[bytes]:
    """All-gather one opaque blob per rank (the exported IPC handle), in rank order."""
    if world == 1:
        return [blob]
    import torch.distributed as dist
    out: list = [None] * world
    dist.all_gather_object(out, blob, group=group)
    return out


def handles_array(blobs: Sequence[bytes]):
    """Marshal gathered blobs into the C array torus_comm_init takes."""
    n = ctypes.sizeof(torus_ipc_handle_t)
    arr = (torus_ipc_handle_t * len(blobs))()
    for r, blob in enumerate(blobs):
        if len(blob) != n:
            raise ValueError(f"rank {r}: IPC handle blob of {len(blob)} bytes, expected {n}")
        ctypes.memmove(ctypes.byref(arr[r]), blob, n)
    return arr


def config_disagreement(cfg, world: int, group=None) -> list:
    """All-gather every rank's configuration fingerprint; ranks that differ from rank 0."""
    if world == 1:
        return []
    import torch.distributed as dist
    cfgs: list = [None] * world
    dist.all_gather_object(cfgs, tuple(cfg), group=group)
    return [r for r, c in enumerate(cfgs) if c != cfgs[0]]


def agree_status(rc: int, msg: str, world: int, group=None) -> list:
    """Every rank learns every rank's init status; returns [(rank, (rc, msg))] failures."""
    if world == 1:
        status = [(rc, msg)]
    else:
        import torch.distributed as dist
        status = [None] * world
        dist.all_gather_object(status, (rc, msg), group=group)
    return [(r, s) for r, s in enumerate(status) if s[0] != 0]


class _CommBase:
    _comm: ctypes.c_void_p

    def grid(self) -> tuple[int, int]:
        X, Y = ctypes.c_int(), ctypes.c_int()
        check(_lib.load().torus_comm_grid(self._comm, ctypes.byref(X), ctypes.byref(Y)), "grid")
        return X.value, Y.value

    def ctas(self) -> int:
        return _lib.load().torus_comm_ctas(self._comm)

    def round_elems(self, wire: torch.dtype) -> int:
        return _lib.load().torus_comm_round_elems(self._comm, _dtype_code(wire))

    def hier_round_elems(self, wire: torch.dtype) -> int:
        return _lib.load().torus_comm_hier_round_elems(self._comm, _dtype_code(wire))

    def ring_round_elems(self, wire: torch.dtype) -> int:
        return _lib.load().torus_comm_ring_round_elems(self._comm, _dtype_code(wire))

    def launches(self, count: int, dtype: torch.dtype, wire: torch.dtype | None = None) -> int:
        return _lib.load().torus_comm_launches(self._comm, count, _dtype_code(dtype),
                                               _dtype_code(wire or dtype))

    def route(self, count: int, dtype: torch.dtype, wire: torch.dtype | None = None) -> str:
        """Kernel a call with these arguments runs (torus_comm_route)."""
        return _lib.load().torus_comm_route(self._comm, count, _dtype_code(dtype),
                                            _dtype_code(wire or dtype)).decode()

    def config(self) -> tuple[int, ...]:
        """Configuration fingerprint that must agree across ranks (torus_comm_config)."""
        words = (ctypes.c_ulonglong * 32)()
        n = _lib.load().torus_comm_config(self._comm, words, 32)
        if n < 0:
            check(-n, "torus_comm_config")
        return tuple(int(w) for w in words[:n])

    def ll_max_bytes(self) -> int:
        """Small-message threshold in wire bytes (torus_comm_ll_max_bytes; 0 = off)."""
        return int(_lib.load().torus_comm_ll_max_bytes(self._comm))

    def ll2_max_bytes(self) -> int:
        """Two-shot (mid-size) threshold in wire bytes (torus_comm_ll2_max_bytes; 0 = off)."""
        return int(_lib.load().torus_comm_ll2_max_bytes(self._comm))

    def probe(self, mode: int, nbytes: int = 0, iters: int = 0, ctas: int = 0,
              stream: torch.cuda.Stream | None = None) -> int:
        """Calibration probe (torus_probe); returns ns for mode 2, else 0 (time it yourself)."""
        ns = ctypes.c_ulonglong(0)
        check(_lib.load().torus_probe(self._comm, mode, nbytes, iters, ctas,
                                      ctypes.byref(ns) if mode in (2, 6, 7, 8, 9) else None,
                                      _stream_ptr(stream)), "torus_probe")
        return ns.value

    def trace(self):
        """Device trace of the last launch (TORUS_TRACE=1): numpy [ctas, 64, 8] of ns."""
        import numpy as np
        out = np.zeros((self.ctas(), 64, 8), dtype=np.uint64)
        check(_lib.load().torus_comm_trace(
            self._comm, out.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), out.nbytes),
            "torus_comm_trace")
        return out

    def pull_trace(self, max_ctas: int = 1024):
        """Device trace of the last pull-kernel launch (TORUS_TRACE=1): (numpy [ctas, 64, 8]
        of ns, ctas per rank, CTA split [S0, R, VR, VA, H, SIG])."""
        import numpy as np
        out = np.zeros((max_ctas, 64, 8), dtype=np.uint64)
        g = ctypes.c_int()
        kinds = (ctypes.c_int * 6)()
        check(_lib.load().torus_comm_pull_trace(
            self._comm, out.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), out.nbytes,
            ctypes.byref(g), kinds), "torus_comm_pull_trace")
        return out, g.value, list(kinds)

    def async_error(self) -> int:
        return _lib.load().torus_comm_get_async_error(self._comm)

    def destroy(self) -> None:
        if getattr(self, "_comm", None):
            c, self._comm = self._comm, None
            check(_lib.load().torus_comm_destroy(c), "torus_comm_destroy")

    def __del__(self):  # best effort; destroy() is collective, call it explicitly
        pass


class TorusComm(_CommBase):
    """One rank of the 2D-Torus communicator (one process per GPU)."""

    def __init__(self, comm: ctypes.c_void_p, rank: int, world: int, device: int):
        self._comm = comm
        self.rank, self.world, self.device = rank, world, device

    @classmethod
    def init(cls, group=None, X: int = 0, Y: int = 0, ws_bytes: int = 0,
             device: int | None = None, ctas: int = 0) -> "TorusComm":
        """Collective: every rank of `group` allocates and exports its slab, the 64-byte
        IPC handles are all-gathered in rank order, every rank opens its peers' slabs,
        and all ranks agree on success (no half-built communicator survives)."""
        import torch.distributed as dist
        L = _lib.load()
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        dev = torch.cuda.current_device() if device is None else device
        torch.cuda.set_device(dev)
        h = torus_ipc_handle_t()
        check(L.torus_workspace_alloc(dev, ws_bytes, ctypes.byref(h)), "torus_workspace_alloc")
        arr = handles_array(exchange_blobs(bytes(h), world, group))
        comm = ctypes.c_void_p()
        import os
        old = os.environ.get("TORUS_CTAS")
        if ctas:  # CTA budget (concurrent comms must fit on the SMs together)
            os.environ["TORUS_CTAS"] = str(ctas)
        try:
            rc = L.torus_comm_init(rank, world, X, Y, arr, ctypes.byref(comm))
        finally:
            if ctas:
                if old is None:
                    del os.environ["TORUS_CTAS"]
                else:
                    os.environ["TORUS_CTAS"] = old
        msg = "" if rc == 0 else L.torus_last_error().decode(errors="replace")
        bad = agree_status(rc, msg, world, group)
        if bad:
            if rc == 0:
                L.torus_comm_abort(comm)  # peers failed: no collective barrier possible
            else:
                L.torus_workspace_release(ctypes.byref(h))
            raise RuntimeError(f"torus_comm_init failed on ranks {bad}")
        self = cls(comm, rank, world, dev)
        # every knob that decides which bytes and flags a call touches must agree across
        # ranks: all-gather the library's configuration fingerprint
        diff = config_disagreement(self.config(), world, group)
        if diff:
            L.torus_comm_abort(comm)
            self._comm = None
            raise _lib.TorusError(7, f"torus_comm_init: configuration differs on ranks {diff} "
                                     "(TORUS_* environment or CTA budget)")
        return self

    def all_reduce(self, t: torch.Tensor, op: str = "mean", wire: torch.dtype | None = None,
                   stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """In-place all-reduce of a contiguous CUDA tensor (sum or mean over all ranks)."""
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("torus all_reduce needs a contiguous CUDA tensor")
        check(_lib.load().torus_allreduce_ex(
            self._comm, ctypes.c_void_p(t.data_ptr()), t.numel(), _dtype_code(t.dtype),
            _dtype_code(wire or t.dtype), OPS[op], _stream_ptr(stream)), "torus_allreduce_ex")
        return t


    def all_reduce_host(self, host: torch.Tensor, dev: torch.Tensor, op: str = "mean",
                        wire: torch.dtype | None = None, piece: int = 0,
                        stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """All-reduce of a (pinned) CPU tensor through the device buffer `dev` (same dtype,
        >= as many elements): H2D, all-reduce and D2H pipelined over pieces of `piece`
        elements (torus_allreduce_host).  Asynchronous on `stream`; `host` holds the result
        once the stream reaches it."""
        if host.is_cuda or not host.is_contiguous() or not dev.is_cuda or not dev.is_contiguous():
            raise ValueError("all_reduce_host needs a contiguous CPU tensor and a contiguous CUDA tensor")
        if host.dtype != dev.dtype or dev.numel() < host.numel():
            raise ValueError("dev must have host's dtype and at least as many elements")
        check(_lib.load().torus_allreduce_host(
            self._comm, ctypes.c_void_p(host.data_ptr()), ctypes.c_void_p(dev.data_ptr()), host.numel(),
            piece, _dtype_code(host.dtype), _dtype_code(wire or host.dtype), OPS[op], _stream_ptr(stream)),
            "torus_allreduce_host")
        return host

    def register(self, t: torch.Tensor, group=None) -> torch.Tensor:
        """Collective: register `t` (a contiguous CUDA tensor every rank will pass to
        all_reduce) for zero-copy -- peers then read its inputs straight over NVLink
        (torus_buffer_export / all-gather / torus_register_buffer)."""
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("register needs a contiguous CUDA tensor")
        L = _lib.load()
        h = torus_ipc_handle_t()
        nbytes = t.numel() * t.element_size()
        check(L.torus_buffer_export(ctypes.c_void_p(t.data_ptr()), nbytes, ctypes.byref(h)),
              "torus_buffer_export")
        arr = handles_array(exchange_blobs(bytes(h), self.world, group))
        check(L.torus_register_buffer(self._comm, ctypes.c_void_p(t.data_ptr()), nbytes, arr),
              "torus_register_buffer")
        return t

    def deregister(self, t: torch.Tensor) -> None:
        check(_lib.load().torus_deregister_buffer(self._comm, ctypes.c_void_p(t.data_ptr())),
              "torus_deregister_buffer")

    def reserve(self, staging_bytes: int) -> None:
        check(_lib.load().torus_comm_reserve(self._comm, staging_bytes), "torus_comm_reserve")

    def all_reduce_multi(self, tensors: Sequence[torch.Tensor], op: str = "mean",
                         wire: torch.dtype | None = None,
                         stream: torch.cuda.Stream | None = None) -> Sequence[torch.Tensor]:
        """Bucketed all-reduce of a list of same-dtype contiguous CUDA tensors (NEXT-1):
        equal to all-reducing their concatenation, cast/scale fused."""
        if not tensors:
            return tensors
        dt = tensors[0].dtype
        for t in tensors:
            if not t.is_cuda or not t.is_contiguous() or t.dtype != dt:
                raise ValueError("all_reduce_multi needs contiguous CUDA tensors of one dtype")
        n = len(tensors)
        ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() for t in tensors])
        counts = (ctypes.c_size_t * n)(*[t.numel() for t in tensors])
        check(_lib.load().torus_allreduce_multi(
            self._comm, ptrs, counts, n, _dtype_code(dt), _dtype_code(wire or dt), OPS[op],
            _stream_ptr(stream)), "torus_allreduce_multi")
        return tensors

    def ring_all_reduce(self, t: torch.Tensor, op: str = "mean", wire: torch.dtype | None = None,
                        stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """The flat-ring BASELINE (torus_ring_allreduce), same semantics, HOP rounding."""
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("ring all_reduce needs a contiguous CUDA tensor")
        check(_lib.load().torus_ring_allreduce(
            self._comm, ctypes.c_void_p(t.data_ptr()), t.numel(), _dtype_code(t.dtype),
            _dtype_code(wire or t.dtype), OPS[op], _stream_ptr(stream)), "torus_ring_allreduce")
        return t


    def nvls_init(self, nbytes: int, group=None) -> None:
        """Collective NVLS setup (NEXT-4): multicast object over all ranks + staging."""
        import torch.distributed as dist
        L = _lib.load()
        blob = (ctypes.c_longlong * 2)()
        check(L.torus_nvls_prepare(self._comm, nbytes, blob), "torus_nvls_prepare")
        blobs: list = [None] * self.world
        dist.all_gather_object(blobs, (int(blob[0]), int(blob[1])), group=group)
        b0 = (ctypes.c_longlong * 2)(*blobs[0])
        rc = L.torus_nvls_attach(self._comm, b0)
        st: list = [None] * self.world
        dist.all_gather_object(st, rc, group=group)  # every device added before any bind
        check(rc, "torus_nvls_attach")
        if any(st):
            raise RuntimeError(f"torus_nvls_attach failed on some rank: {st}")
        rc = L.torus_nvls_bind(self._comm)
        dist.all_gather_object(st, rc, group=group)
        check(rc, "torus_nvls_bind")
        if any(st):
            raise RuntimeError(f"torus_nvls_bind failed on some rank: {st}")

    def nvls_all_reduce(self, t: torch.Tensor, op: str = "mean", wire: torch.dtype | None = None,
                        stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """In-switch-reduction all-reduce (NEXT-4); tolerance-level parity (switch order)."""
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("nvls all_reduce needs a contiguous CUDA tensor")
        check(_lib.load().torus_nvls_allreduce(
            self._comm, ctypes.c_void_p(t.data_ptr()), t.numel(), _dtype_code(t.dtype),
            _dtype_code(wire or t.dtype), OPS[op], _stream_ptr(stream)), "torus_nvls_allreduce")
        return t

    def hier_all_reduce(self, t: torch.Tensor, op: str = "mean", wire: torch.dtype | None = None,
                        stream: torch.cuda.Stream | None = None) -> torch.Tensor:
        """The hierarchical BASELINE [6] (torus_hier_allreduce), HOP rounding."""
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("hier all_reduce needs a contiguous CUDA tensor")
        check(_lib.load().torus_hier_allreduce(
            self._comm, ctypes.c_void_p(t.data_ptr()), t.numel(), _dtype_code(t.dtype),
            _dtype_code(wire or t.dtype), OPS[op], _stream_ptr(stream)), "torus_hier_allreduce")
        return t


class VirtualTorus(_CommBase):
    """A whole X-by-Y grid emulated on one GPU (one cooperative launch per round); runs
    the product kernel with every virtual rank's peer pointers aimed at local slabs."""

    def __init__(self, X: int, Y: int, device: int = 0, ctas: int = 0, ws_bytes: int = 0):
        L = _lib.load()
        torch.cuda.set_device(device)
        self._comm = ctypes.c_void_p()
        check(L.torus_vcomm_init(device, X, Y, ctas, ws_bytes, ctypes.byref(self._comm)),
              "torus_vcomm_init")
        self.X, self.Y, self.N, self.device = X, Y, X * Y, device

    def all_reduce(self, tensors: Sequence[torch.Tensor], op: str = "mean",
                   wire: torch.dtype | None = None,
                   stream: torch.cuda.Stream | None = None) -> Sequence[torch.Tensor]:
        if len(tensors) != self.N:
            raise ValueError(f"need {self.N} tensors, one per virtual rank")
        t0 = tensors[0]
        for t in tensors:
            if not t.is_cuda or not t.is_contiguous() or t.dtype != t0.dtype or t.numel() != t0.numel():
                raise ValueError("virtual ranks need equal contiguous CUDA tensors")
        ptrs = (ctypes.c_void_p * self.N)(*[t.data_ptr() for t in tensors])
        check(_lib.load().torus_vallreduce(
            self._comm, ptrs, t0.numel(), _dtype_code(t0.dtype), _dtype_code(wire or t0.dtype),
            OPS[op], _stream_ptr(stream)), "torus_vallreduce")
        return tensors

    def all_reduce_multi(self, buckets: Sequence[Sequence[torch.Tensor]], op: str = "mean",
                         wire: torch.dtype | None = None,
                         stream: torch.cuda.Stream | None = None):
        """Fused bucket call over the virtual ranks (torus_vallreduce_multi): buckets[r] is
        rank r's list of tensors (same shapes on every rank)."""
        if len(buckets) != self.N:
            raise ValueError(f"need {self.N} tensor lists, one per virtual rank")
        nt = len(buckets[0])
        dt = buckets[0][0].dtype
        ptrs = (ctypes.c_void_p * (self.N * nt))(*[t.data_ptr() for b in buckets for t in b])
        counts = (ctypes.c_size_t * nt)(*[t.numel() for t in buckets[0]])
        check(_lib.load().torus_vallreduce_multi(self._comm, ptrs, counts, nt, _dtype_code(dt),
                                                 _dtype_code(wire or dt), OPS[op], _stream_ptr(stream)),
              "torus_vallreduce_multi")
        return buckets

    def ring_all_reduce(self, tensors: Sequence[torch.Tensor], op: str = "mean",
                        wire: torch.dtype | None = None,
                        stream: torch.cuda.Stream | None = None) -> Sequence[torch.Tensor]:
        """Flat-ring baseline over the virtual ranks (torus_vring_allreduce)."""
        t0 = tensors[0]
        ptrs = (ctypes.c_void_p * self.N)(*[t.data_ptr() for t in tensors])
        check(_lib.load().torus_vring_allreduce(
            self._comm, ptrs, t0.numel(), _dtype_code(t0.dtype), _dtype_code(wire or t0.dtype),
            OPS[op], _stream_ptr(stream)), "torus_vring_allreduce")
        return tensors

    def hier_all_reduce(self, tensors: Sequence[torch.Tensor], op: str = "mean",
                        wire: torch.dtype | None = None,
                        stream: torch.cuda.Stream | None = None) -> Sequence[torch.Tensor]:
        """Hierarchical baseline over the virtual ranks (torus_vhier_allreduce)."""
        t0 = tensors[0]
        ptrs = (ctypes.c_void_p * self.N)(*[t.data_ptr() for t in tensors])
        check(_lib.load().torus_vhier_allreduce(
            self._comm, ptrs, t0.numel(), _dtype_code(t0.dtype), _dtype_code(wire or t0.dtype),
            OPS[op], _stream_ptr(stream)), "torus_vhier_allreduce")
        return tensors
