"""CPU oracle for the 2D-Torus all-reduce -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1811_05233_b200`` never imports it, and the C source under this directory shares
no code with ``paper_1811_05233_b200/csrc`` (see torus_oracle.h).

This module is argument marshalling only (ctypes over ``liboracle.so``); every step of
the method is computed in ``torus_oracle.c`` (Sec. 2.2).

Array conventions: f32 -> numpy float32, f16 -> numpy float16, bf16 -> numpy uint16
(raw bfloat16 bit patterns; numpy has no bfloat16), i32 -> numpy int32.
"""
from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess
import threading

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
_SRC = _HERE / "torus_oracle.c"
_SO = _HERE / "liboracle.so"
_lock = threading.Lock()
_lib = None

CODES = {"f32": 0, "f16": 1, "bf16": 2, "i32": 3}
NP_STORAGE = {"f32": np.float32, "f16": np.float16, "bf16": np.uint16, "i32": np.int32}
OPS = {"sum": 0, "mean": 1}
POLICIES = {"phase": 0, "hop": 1}
PHASES = ("h_rs", "v_rs", "v_ag", "h_ag")


class _Counters(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_longlong * 4), ("sent", ctypes.c_longlong * 4),
                ("recv", ctypes.c_longlong * 4)]


def build(force: bool = False) -> pathlib.Path:
    """Compile liboracle.so with gcc (plain C11, no fast-math, no FP contraction)."""
    if force or not _SO.exists() or _SO.stat().st_mtime < max(
            _SRC.stat().st_mtime, (_HERE / "torus_oracle.h").stat().st_mtime):
        tmp = _SO.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-Wall", "-Wextra", "-fPIC", "-shared", str(_SRC), "-o", str(tmp)])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(str(_SO))
            vpp = ctypes.POINTER(ctypes.c_void_p)
            ll, i = ctypes.c_longlong, ctypes.c_int
            L.orc_qpart.argtypes = [ll, i, i, ctypes.POINTER(ll), ctypes.POINTER(ll)]
            L.orc_torus_allreduce.argtypes = [i, i, ll, i, i, i, i, i, ll, vpp, vpp,
                                              ctypes.POINTER(_Counters)]
            L.orc_torus_element.argtypes = [i, i, ll, i, i, i, i, i, ll, ll, vpp, ctypes.c_void_p]
            L.orc_ring_allreduce.argtypes = [i, ll, i, i, i, i, i, ll, vpp, vpp,
                                             ctypes.POINTER(_Counters)]
            L.orc_hier_allreduce.argtypes = [i, i, ll, i, i, i, i, i, vpp, vpp,
                                             ctypes.POINTER(_Counters)]
            L.orc_brute_sum_f64.argtypes = [i, ll, i, i, vpp, ctypes.POINTER(ctypes.c_double)]
            L.orc_f32_to_f16.argtypes = [ctypes.c_float]
            L.orc_f32_to_f16.restype = ctypes.c_uint16
            L.orc_f16_to_f32.argtypes = [ctypes.c_uint16]
            L.orc_f16_to_f32.restype = ctypes.c_float
            L.orc_f32_to_bf16.argtypes = [ctypes.c_float]
            L.orc_f32_to_bf16.restype = ctypes.c_uint16
            L.orc_bf16_to_f32.argtypes = [ctypes.c_uint16]
            L.orc_bf16_to_f32.restype = ctypes.c_float
            _lib = L
    return _lib


def _ptrs(arrays):
    arr = (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])
    return ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p))


def _check_inputs(inputs, dtype):
    st = NP_STORAGE[dtype]
    out = []
    for a in inputs:
        a = np.ascontiguousarray(a)
        if a.dtype != st:
            raise TypeError(f"oracle: {dtype} inputs must be stored as {np.dtype(st)}, got {a.dtype}")
        out.append(a)
    if len({a.size for a in out}) > 1:
        raise ValueError("oracle: all ranks must pass equal-length buffers (SPEC.md:181)")
    return out


def _counters_dict(ctr, n):
    return [{"steps": dict(zip(PHASES, ctr[r].steps)), "sent": dict(zip(PHASES, ctr[r].sent)),
             "recv": dict(zip(PHASES, ctr[r].recv))} for r in range(n)]


def _rc(rc, what):
    if rc != 0:
        raise RuntimeError(f"oracle {what} failed with code {rc}")


def qpart(n: int, parts: int, q: int = 1):
    off = (ctypes.c_longlong * parts)()
    ln = (ctypes.c_longlong * parts)()
    _rc(lib().orc_qpart(n, parts, q, off, ln), "qpart")
    return list(off), list(ln)


def torus_allreduce(inputs, X, Y, dtype, wire=None, op="sum", policy="phase", q=1,
                    round_elems=0, counters=False):
    """Simulate the X-by-Y 2D-Torus all-reduce of ``inputs`` (one array per rank)."""
    wire = wire or dtype
    ins = _check_inputs(inputs, dtype)
    if len(ins) != X * Y:
        raise ValueError("oracle: need X*Y input buffers")
    outs = [np.empty_like(a) for a in ins]
    ctr = (_Counters * (X * Y))()
    _rc(lib().orc_torus_allreduce(X, Y, ins[0].size, CODES[dtype], CODES[wire], OPS[op],
                                  POLICIES[policy], q, round_elems, _ptrs(ins), _ptrs(outs), ctr),
        "torus_allreduce")
    return (outs, _counters_dict(ctr, X * Y)) if counters else outs


def torus_element(inputs_at, X, Y, D, i, dtype, wire=None, op="sum", policy="phase", q=1,
                  round_elems=0):
    """Closed-form output element ``i`` given the N ranks' full input arrays."""
    wire = wire or dtype
    ins = _check_inputs(inputs_at, dtype)
    out = np.zeros(1, dtype=NP_STORAGE[dtype])
    _rc(lib().orc_torus_element(X, Y, D, CODES[dtype], CODES[wire], OPS[op], POLICIES[policy],
                                q, round_elems, i, _ptrs(ins), out.ctypes.data), "torus_element")
    return out[0]


def torus_elements(inputs, X, Y, idx, dtype, wire=None, op="sum", policy="phase", q=1,
                   round_elems=0):
    """Closed-form outputs at the indices ``idx`` (full-size sampled parity)."""
    D = inputs[0].size
    return np.array([torus_element(inputs, X, Y, D, int(i), dtype, wire, op, policy, q,
                                   round_elems) for i in idx], dtype=NP_STORAGE[dtype])


def ring_allreduce(inputs, dtype, wire=None, op="sum", policy="phase", q=1, round_elems=0,
                   counters=False):
    wire = wire or dtype
    ins = _check_inputs(inputs, dtype)
    outs = [np.empty_like(a) for a in ins]
    ctr = (_Counters * len(ins))()
    _rc(lib().orc_ring_allreduce(len(ins), ins[0].size, CODES[dtype], CODES[wire], OPS[op],
                                 POLICIES[policy], q, round_elems, _ptrs(ins), _ptrs(outs), ctr),
        "ring_allreduce")
    return (outs, _counters_dict(ctr, len(ins))) if counters else outs


def hier_allreduce(inputs, X, Y, dtype, wire=None, op="sum", policy="phase", q=1,
                   counters=False):
    wire = wire or dtype
    ins = _check_inputs(inputs, dtype)
    outs = [np.empty_like(a) for a in ins]
    ctr = (_Counters * len(ins))()
    _rc(lib().orc_hier_allreduce(X, Y, ins[0].size, CODES[dtype], CODES[wire], OPS[op],
                                 POLICIES[policy], q, _ptrs(ins), _ptrs(outs), ctr),
        "hier_allreduce")
    return (outs, _counters_dict(ctr, len(ins))) if counters else outs


def brute_sum_f64(inputs, dtype, op="sum"):
    ins = _check_inputs(inputs, dtype)
    out = np.empty(ins[0].size, dtype=np.float64)
    _rc(lib().orc_brute_sum_f64(len(ins), ins[0].size, CODES[dtype], OPS[op], _ptrs(ins),
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))),
        "brute_sum_f64")
    return out


def _conv(name, x, out_dtype):
    x = np.ascontiguousarray(x)
    y = np.empty(x.size, dtype=out_dtype)
    getattr(lib(), name)(ctypes.c_void_p(x.ctypes.data), ctypes.c_void_p(y.ctypes.data),
                         ctypes.c_longlong(x.size))
    return y


def f32_to_f16_array(x):
    """float32 array -> binary16 bit patterns (uint16), software RNE."""
    return _conv("orc_f32_to_f16_array", np.asarray(x, dtype=np.float32), np.uint16)


def f16_to_f32_array(bits):
    return _conv("orc_f16_to_f32_array", np.asarray(bits, dtype=np.uint16), np.float32)


def f32_to_bf16_array(x):
    return _conv("orc_f32_to_bf16_array", np.asarray(x, dtype=np.float32), np.uint16)


def bf16_to_f32_array(bits):
    return _conv("orc_bf16_to_f32_array", np.asarray(bits, dtype=np.uint16), np.float32)


def f32_to_f16_bits(x: float) -> int:
    return lib().orc_f32_to_f16(x)


def f16_bits_to_f32(h: int) -> float:
    return lib().orc_f16_to_f32(h)


def f32_to_bf16_bits(x: float) -> int:
    return lib().orc_f32_to_bf16(x)


def bf16_bits_to_f32(h: int) -> float:
    return lib().orc_bf16_to_f32(h)
