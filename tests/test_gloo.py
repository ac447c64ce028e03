"""World-size-2 gloo tests (CPU) of the multi-process host logic around the CUDA path:
the IPC-handle exchange, its marshalling into the C array, and the all-ranks agreement
on communicator init (SURVEY.md Sec. 4 T3 host side).  No GPU is touched."""
import os
import socket
import traceback

import pytest

torch = pytest.importorskip("torch")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, errfile):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import ctypes

        import torch.distributed as dist

        from paper_1811_05233_b200 import torus
        from paper_1811_05233_b200._lib import torus_ipc_handle_t
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        n = ctypes.sizeof(torus_ipc_handle_t)
        mine = bytes([rank + 1]) * 64 + (0).to_bytes(8, "little") + (1 << 20).to_bytes(8, "little")
        assert len(mine) == n
        blobs = torus.exchange_blobs(mine, world)
        assert [b[0] for b in blobs] == [r + 1 for r in range(world)]       # rank order
        arr = torus.handles_array(blobs)
        for r in range(world):
            assert bytes(arr[r].bytes) == bytes([r + 1]) * 64 and arr[r].size == 1 << 20
        with pytest.raises(ValueError):
            torus.handles_array([b"short"])
        # all ranks succeed
        assert torus.agree_status(0, "", world) == []
        # rank 1 fails: every rank sees the failure (nobody keeps a half-built comm)
        bad = torus.agree_status(5 if rank == 1 else 0, "TORUS_ERR_PEER" if rank == 1 else "", world)
        assert [r for r, _ in bad] == [1] and bad[0][1][0] == 5
        # configuration fingerprints: equal -> [], rank 1 differs -> [1] everywhere
        cfg = (2, 2, 1, 148, 512 << 20, 0)
        assert torus.config_disagreement(cfg, world) == []
        other = cfg if rank == 0 else cfg[:3] + (74,) + cfg[4:]
        assert torus.config_disagreement(other, world) == [1]
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        with open(errfile, "a") as f:
            f.write(f"rank {rank}:\n{traceback.format_exc()}\n")
        raise


def test_handle_exchange_and_status_agreement_world2(tmp_path):
    import torch.multiprocessing as mp
    errfile = str(tmp_path / "err.txt")
    try:
        mp.spawn(_worker, args=(2, _port(), errfile), nprocs=2, join=True)
    except Exception as e:
        raise AssertionError(open(errfile).read() if os.path.exists(errfile) else str(e)) from None
