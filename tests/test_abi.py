"""CPU-side checks of the C-ABI library (no GPU needed): libtorus.so loads, exports every
symbol include/torus.h declares, and its host logic (partition, topology, validation,
error strings) behaves as specified.  The host partition is compared with the oracle's
independent implementation, bit for bit."""
import ctypes
import os
import re

import pytest

import oracle
from paper_1811_05233_b200 import _lib, partition, pick_grid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "torus.h")).read()
    return sorted(set(re.findall(r"TORUS_API\s+[\w\s\*]+?\b(torus_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    names = _declared_symbols()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), f"libtorus.so does not export {n}"
        assert n in _lib.PROTOTYPES, f"binding lacks a prototype for {n}"
    assert set(_lib.PROTOTYPES) == set(names)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("n", [0, 1, 7, 1000, 25_557_032, 2 ** 40 + 3])
@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8, 64])
@pytest.mark.parametrize("q", [1, 4, 8])
def test_partition_matches_oracle(n, parts, q):
    assert partition(n, parts, q) == oracle.qpart(n, parts, q)


def test_northstar_partition_values():
    """the 25,557,032-element fp16 buffer on 2x4 with the 16-byte quantum."""
    off, ln = partition(25_557_032, 2, 8)
    assert ln == [12_778_520, 12_778_512]
    assert partition(ln[0], 4, 8)[1] == [3_194_632] * 3 + [3_194_624]
    assert partition(ln[1], 4, 8)[1] == [3_194_632] * 2 + [3_194_624] * 2


def test_pick_grid():
    assert pick_grid(8, [[1] * 8] * 8) == (8, 1)           # one NVSwitch domain
    two = [[1 if i // 4 == j // 4 else 0 for j in range(8)] for i in range(8)]
    assert pick_grid(8, two) == (4, 2)                      # rows = P2P domains
    assert pick_grid(1, [[1]]) == (1, 1)
    # an isolated GPU: every grid crosses the slow path once; the model keeps one row
    assert pick_grid(3, [[1, 0, 0], [0, 1, 1], [0, 1, 1]]) == (3, 1)


def test_null_and_bad_arguments_rejected_without_gpu():
    L = _lib.load()
    assert L.torus_allreduce(None, None, 10, 1, 0, None) == 1
    assert L.torus_allreduce_ex(None, None, 10, 0, 1, 0, None) == 1
    assert L.torus_comm_grid(None, None, None) == 1
    assert L.torus_comm_destroy(None) == 0
    assert L.torus_comm_round_elems(None, 1) == 0
    assert L.torus_comm_launches(None, 10, 1, 1) == -1
    assert L.torus_comm_ll_max_bytes(None) == 0
    assert L.torus_comm_ll2_max_bytes(None) == 0
    assert L.torus_comm_ctas(None) == -1
    h = (_lib.torus_ipc_handle_t * 2)()
    c = ctypes.c_void_p()
    assert L.torus_comm_init(0, 2, 3, 1, h, ctypes.byref(c)) == 2   # 3*1 != 2
    assert L.torus_comm_init(2, 2, 2, 1, h, ctypes.byref(c)) == 2   # rank out of range
    assert L.torus_comm_init(0, 100, 10, 10, h, ctypes.byref(c)) == 2
    assert L.torus_workspace_alloc(0, 0, None) == 1
    assert b"GRID" in L.torus_last_error() or b"INVALID" in L.torus_last_error()
    # host-buffer path: NULL comm / pointers are INVALID_ARG before anything is enqueued
    assert L.torus_allreduce_host(None, None, None, 10, 0, 1, 1, 1, None) == 1
    buf = ctypes.create_string_buffer(64)
    assert L.torus_allreduce_host(None, buf, buf, 10, 0, 1, 1, 1, None) == 1


def test_all_reduce_host_binding_validates_tensors():
    """TorusComm.all_reduce_host rejects a CUDA host tensor / CPU device tensor / short or
    mistyped device buffer before calling the library (marshalling only)."""
    import torch

    from paper_1811_05233_b200 import TorusComm
    comm = TorusComm.__new__(TorusComm)
    cpu = torch.zeros(16, dtype=torch.float16)
    with pytest.raises(ValueError):
        comm.all_reduce_host(cpu, cpu.clone())             # dev must be a CUDA tensor
    with pytest.raises(ValueError):
        comm.all_reduce_host(cpu[::2], cpu.clone())        # host must be contiguous


def test_strerror_names():
    L = _lib.load()
    for code, name in _lib.ERRORS.items():
        assert L.torus_strerror(code).decode() == name
    assert L.torus_strerror(0) == b"TORUS_OK"


def test_product_never_imports_oracle():
    """The oracle is test infrastructure only (task rule); the product must not touch it."""
    pkg = os.path.join(ROOT, "paper_1811_05233_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", txt, re.M), f
                assert "torus_oracle" not in txt, f
