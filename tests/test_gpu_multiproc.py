"""Multi-process parity on real GPUs: one process per GPU, CUDA IPC + P2P over NVLink,
the product kernel vs the oracle, bit-exact.  Needs >= 2 GPUs
(run with `gpurun --gpus 2` / `--gpus 4`); skipped on a 1-GPU box.

Every rank generates every rank's seeded inputs (so it can run the oracle itself),
then the ranks barrier, launch together, synchronize, and only then compare -- so no
kernel ever spin-waits on a peer that is busy in the CPU oracle.
"""
import os
import socket
import traceback

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

TD = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16, "i32": torch.int32}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _to_dev(a, dtype, dev):
    if dtype == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).to(dev)
    return torch.from_numpy(a.copy()).to(dev)


def _from_dev(t, dtype):
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def _same(got, ref):
    w = {2: np.uint16, 4: np.uint32}[got.dtype.itemsize]
    if got.dtype == np.uint16:
        gn = ((got & 0x7F80) == 0x7F80) & ((got & 0x7F) != 0)
        rn = ((ref & 0x7F80) == 0x7F80) & ((ref & 0x7F) != 0)
    elif got.dtype in (np.float16, np.float32):
        gn, rn = np.isnan(got), np.isnan(ref)
    else:
        gn = rn = np.zeros(got.shape, bool)
    eq = (got.view(w) == ref.view(w)) | (gn & rn)
    return bool(eq.all()), int((~eq).sum())


def _worker(rank, world, port, cases, errfile):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import torch.distributed as dist

        import oracle
        import synthetic
        from paper_1811_05233_b200 import TorusComm
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        comms = {}
        for (X, Y, dtype, wire, op, D, dist_name) in cases:
            ring = X == 0  # (0, N, ...) marks the flat-ring baseline over all ranks
            hier = X < 0   # (-X, Y, ...) marks the hierarchical baseline on an X-by-Y grid
            key = (world, 1) if ring else ((-X, Y) if hier else (X, Y))
            if key not in comms:
                comms[key] = TorusComm.init(X=key[0], Y=key[1])
            comm = comms[key]
            ins = synthetic.make_all(dist_name, D, world, dtype, salt=D % 89)
            t = _to_dev(ins[rank], dtype, f"cuda:{rank}")
            torch.cuda.synchronize()
            dist.barrier()
            fn = comm.ring_all_reduce if ring else (comm.hier_all_reduce if hier else comm.all_reduce)
            fn(t, op=op, wire=TD[wire])
            torch.cuda.synchronize()
            assert comm.async_error() == 0, "watchdog"
            got = _from_dev(t, dtype)
            q = 16 // (2 if wire in ("f16", "bf16") else 4)
            if ring:
                ref = oracle.ring_allreduce(ins, dtype, wire=wire, op=op, policy="hop", q=q,
                                            round_elems=comm.ring_round_elems(TD[wire]))[rank]
                ok, nbad = _same(got, ref)
                assert ok, f"rank {rank} ring {dtype}/{wire} {op} D={D}: {nbad} mismatches"
                dist.barrier()
                continue
            if hier:
                ref = oracle.hier_allreduce(ins, -X, Y, dtype, wire=wire, op=op, policy="hop", q=q)[rank]
                ok, nbad = _same(got, ref)
                assert ok, f"rank {rank} hier {-X}x{Y} {dtype}/{wire} {op} D={D}: {nbad} mismatches"
                dist.barrier()
                continue
            R = comm.round_elems(TD[wire])
            if D <= 300_000:
                ref = oracle.torus_allreduce(ins, X, Y, dtype, wire=wire, op=op, q=q,
                                             round_elems=R)[rank]
                ok, nbad = _same(got, ref)
            else:  # full size: sampled outputs vs the oracle's closed form
                g = np.random.Generator(np.random.PCG64(rank))
                idx = np.unique(np.concatenate([g.integers(0, D, 3000), [0, D - 1]]))
                ref = oracle.torus_elements(ins, X, Y, idx, dtype, wire=wire, op=op, q=q,
                                            round_elems=R)
                ok, nbad = _same(got[idx], ref)
            assert ok, f"rank {rank} {X}x{Y} {dtype}/{wire} {op} D={D}: {nbad} mismatches"
            dist.barrier()
        for c in comms.values():
            dist.barrier()
            c.destroy()
        dist.destroy_process_group()
    except Exception:
        with open(errfile, "a") as f:
            f.write(f"rank {rank}:\n{traceback.format_exc()}\n")
        raise


def _run(world, cases, tmp_path, ll_max=None):
    """ll_max: (TORUS_LL_MAX_BYTES, TORUS_LL2_MAX_BYTES) for the spawned ranks (None =
    library defaults)."""
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    errfile = str(tmp_path / "errors.txt")
    keys = ("TORUS_LL_MAX_BYTES", "TORUS_LL2_MAX_BYTES")
    old = {k: os.environ.get(k) for k in keys}
    if ll_max is not None:
        for k, v in zip(keys, ll_max):
            os.environ[k] = str(v)
    try:
        mp.spawn(_worker, args=(world, _free_port(), cases, errfile), nprocs=world, join=True)
    except Exception as e:
        msg = open(errfile).read() if os.path.exists(errfile) else str(e)
        raise AssertionError(msg) from None
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


# LL paths off (multi-phase kernel at every size) / one-shot forced for every size below
# 1 MiB of wire per rank (NEXT-2) / two-shot forced below 1 MiB (N >= 3)
LL_MODES = pytest.mark.parametrize("ll_max", [(0, 0), (1 << 20, 0)], ids=["multiphase", "oneshot"])
LL_MODES_4 = pytest.mark.parametrize("ll_max", [(0, 0), (1 << 20, 0), (0, 1 << 20)],
                                     ids=["multiphase", "oneshot", "twoshot"])


PAIRS = [("f32", "f32"), ("f16", "f16"), ("bf16", "bf16"), ("i32", "i32"), ("f32", "f16"),
         ("f32", "bf16")]


def _cases(grids, sizes=(1, 4099, 200_003), ops=("sum", "mean")):
    out = []
    for (X, Y) in grids:
        for dtype, wire in PAIRS:
            for op in ops:
                for D in sizes:
                    dn = "full" if dtype == "i32" else ("wide" if D < 5000 else "normal")
                    out.append((X, Y, dtype, wire, op, D, dn))
    return out


@LL_MODES
def test_two_gpus(tmp_path, ll_max):
    _run(2, _cases([(2, 1), (1, 2), (0, 2)]), tmp_path, ll_max)


@LL_MODES_4
def test_four_gpus(tmp_path, ll_max):
    cases = _cases([(2, 2), (4, 1), (1, 4), (0, 4), (-2, 2)], ops=("mean",))
    cases += [(2, 2, "f16", "f16", "mean", 25_557_032, "grad")]  # config 2 shape on 2x2
    _run(4, cases, tmp_path, ll_max)


def _multi_worker(rank, world, port, errfile):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import torch.distributed as dist

        import oracle
        import synthetic
        from paper_1811_05233_b200 import TorusComm
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        comm = TorusComm.init(X=world, Y=1)
        # a ResNet-50-shaped bucket: the 40 smallest-to-mid layers (backprop order)
        sizes = synthetic.resnet50_param_numels()[::-1][:40]
        D = sum(sizes)
        for wire in ("f16", "bf16"):
            ins = synthetic.make_all("grad", D, world, "f32", salt=3)
            full = torch.from_numpy(ins[rank].copy()).cuda()
            parts = list(torch.split(full.clone(), sizes))
            parts = [p.contiguous() for p in parts]
            torch.cuda.synchronize()
            dist.barrier()
            comm.all_reduce_multi(parts, op="mean", wire=TD[wire])
            torch.cuda.synchronize()
            assert comm.async_error() == 0
            got = torch.cat(parts).cpu().numpy()
            ref = oracle.torus_allreduce(ins, world, 1, "f32", wire=wire, op="mean", q=8,
                                         round_elems=comm.round_elems(TD[wire]))[rank]
            ok, nbad = _same(got, ref)
            assert ok, f"rank {rank} multi {wire}: {nbad} mismatches"
            dist.barrier()
        dist.barrier()
        comm.destroy()
        dist.destroy_process_group()
    except Exception:
        with open(errfile, "a") as f:
            f.write(f"rank {rank}:\n{traceback.format_exc()}\n")
        raise


def test_multi_tensor_bucket_two_gpus(tmp_path):
    """NEXT-1: the bucketed API equals the all-reduce of the concatenated bucket."""
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    errfile = str(tmp_path / "errors.txt")
    try:
        mp.spawn(_multi_worker, args=(2, _free_port(), errfile), nprocs=2, join=True)
    except Exception as e:
        raise AssertionError(open(errfile).read() if os.path.exists(errfile) else str(e)) from None


def _nvls_worker(rank, world, port, errfile):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import torch.distributed as dist

        import oracle
        import synthetic
        from paper_1811_05233_b200 import TorusComm
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        comm = TorusComm.init(X=world, Y=1)
        comm.nvls_init(8 << 20)
        for dtype, wire, tol in (("f16", "f16", 1e-2), ("bf16", "bf16", 1e-2), ("f32", "f32", 1e-6),
                                 ("f32", "f16", 1e-2)):
            D = 1_000_003
            ins = synthetic.make_all("normal", D, world, dtype, salt=11)
            t = _to_dev(ins[rank], dtype, f"cuda:{rank}")
            torch.cuda.synchronize()
            dist.barrier()
            comm.nvls_all_reduce(t, op="mean", wire=TD[wire])  # 4 rounds of the 8 MiB staging
            torch.cuda.synchronize()
            assert comm.async_error() == 0
            got = synthetic.as_float64(_from_dev(t, dtype), dtype)
            ref = oracle.brute_sum_f64(ins, dtype, "mean")
            mag = sum(np.abs(synthetic.as_float64(a, dtype)) for a in ins) / world
            err = np.abs(got - ref) / (mag + 1e-30)
            assert (err <= tol).all(), f"rank {rank} nvls {dtype}/{wire}: max err {err.max()}"
            dist.barrier()
        dist.barrier()
        comm.destroy()
        dist.destroy_process_group()
    except Exception:
        with open(errfile, "a") as f:
            f.write(f"rank {rank}:\n{traceback.format_exc()}\n")
        raise


@pytest.mark.parametrize("world", [2, 4])
def test_nvls_variant_tolerance(tmp_path, world):
    """NEXT-4: in-switch reduction; the switch's order is unspecified, so the check is the
    north-star tolerance vs the f64 sum (1e-2 f16/bf16, 1e-6 f32, normalized by sum|x|)."""
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    errfile = str(tmp_path / "errors.txt")
    try:
        mp.spawn(_nvls_worker, args=(world, _free_port(), errfile), nprocs=world, join=True)
    except Exception as e:
        raise AssertionError(open(errfile).read() if os.path.exists(errfile) else str(e)) from None


def _mismatch_worker(rank, world, port, errfile):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import time
        import torch.distributed as dist
        from paper_1811_05233_b200 import TorusComm
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), TORUS_CHECK="1",
                          TORUS_TIMEOUT_MS="20000")
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        comm = TorusComm.init(X=world, Y=1)
        D = 1_000_000 + 8 * rank  # the ranks disagree on the count
        t = torch.ones(D, dtype=torch.float16, device=f"cuda:{rank}")
        dist.barrier()
        t0 = time.time()
        comm.all_reduce(t, op="sum")
        torch.cuda.synchronize()
        dt = time.time() - t0
        err = comm.async_error()
        assert err == 7, f"rank {rank}: async error {err}, expected TORUS_ERR_MISMATCH (7)"
        assert dt < 10.0, f"rank {rank}: took {dt:.1f} s (the check should abort, not time out)"
        dist.barrier()
        comm.destroy()  # poisoned comm: no collective barrier, resources freed
        dist.destroy_process_group()
    except Exception:
        with open(errfile, "a") as f:
            f.write(f"rank {rank}:\n{traceback.format_exc()}\n")
        raise


def test_header_check_detects_mismatch(tmp_path):
    """with TORUS_CHECK=1, ranks that disagree on the call
    (here the count) get TORUS_ERR_MISMATCH asynchronously instead of hanging."""
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    errfile = str(tmp_path / "errors.txt")
    try:
        mp.spawn(_mismatch_worker, args=(2, _free_port(), errfile), nprocs=2, join=True)
    except Exception as e:
        raise AssertionError(open(errfile).read() if os.path.exists(errfile) else str(e)) from None


def _stream_worker(rank, world, port, errfile, X, Y):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import torch.distributed as dist

        import oracle
        import synthetic
        from paper_1811_05233_b200 import TorusComm
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        comm = TorusComm.init(X=X, Y=Y)
        R16 = comm.round_elems(torch.float16)
        # every routing threshold (one-shot, two-shot, multi-phase) and a multi-round call,
        # back to back on one stream, no host synchronization in between
        sizes = [5, comm.ll_max_bytes() // 2, comm.ll_max_bytes() // 2 + 8, 3_000_001, 8, 25_557_032,
                 1_000, R16 + 12_345, 77, 9_000_000]
        sizes = [s for s in sizes if s > 0]
        ins = [synthetic.make_all("normal", D, world, "f16", salt=90 + k) for k, D in enumerate(sizes)]
        ts = [torch.from_numpy(a[rank].copy()).to(f"cuda:{rank}") for a in ins]
        torch.cuda.synchronize()
        dist.barrier()
        for t in ts:
            comm.all_reduce(t, op="mean")
        torch.cuda.synchronize()
        assert comm.async_error() == 0
        for k, (t, a) in enumerate(zip(ts, ins)):
            D = a[0].size
            if D > 3_000_000:
                g = np.random.Generator(np.random.PCG64(k))
                idx = np.unique(np.concatenate([g.integers(0, D, 2000), [0, D - 1]]))
                ref = oracle.torus_elements(a, X, Y, idx, "f16", op="mean", q=8, round_elems=R16)
                ok, nbad = _same(t.cpu().numpy()[idx], ref)
            else:
                ref = oracle.torus_allreduce(a, X, Y, "f16", op="mean", q=8, round_elems=R16)[rank]
                ok, nbad = _same(t.cpu().numpy(), ref)
            assert ok, f"rank {rank} call {k} D={D} ({comm.route(D, torch.float16)}): {nbad} mismatches"
        dist.barrier()
        comm.destroy()
        dist.destroy_process_group()
    except Exception:
        with open(errfile, "a") as f:
            f.write(f"rank {rank}:\n{traceback.format_exc()}\n")
        raise


@pytest.mark.parametrize("world,X,Y", [(2, 1, 2), (2, 2, 1), (4, 2, 2)])
def test_back_to_back_calls_across_routes(tmp_path, world, X, Y):
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    errfile = str(tmp_path / "errors.txt")
    try:
        mp.spawn(_stream_worker, args=(world, _free_port(), errfile, X, Y), nprocs=world, join=True)
    except Exception as e:
        raise AssertionError(open(errfile).read() if os.path.exists(errfile) else str(e)) from None


def _host_worker(rank, world, port, errfile):
    """torus_allreduce_host: pinned host buffer -> device -> all-reduce -> host, pipelined
    over pieces; each piece must equal the oracle on that piece (its own message)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import torch.distributed as dist

        import oracle
        import synthetic
        from paper_1811_05233_b200 import TorusComm
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        X, Y = (1, 2) if world == 2 else (2, 2)
        comm = TorusComm.init(X=X, Y=Y)
        for dtype, wire, D, piece in [("f16", "f16", 1_000_003, 262_144), ("f32", "f16", 600_001, 0),
                                      ("f32", "bf16", 300_007, 100_000), ("bf16", "bf16", 5_000, 1_024)]:
            ins = synthetic.make_all("normal", D, world, dtype, salt=D % 97)
            host = _to_dev(ins[rank], dtype, "cpu").pin_memory()
            dev = torch.empty(D + 13, dtype=TD[dtype], device=f"cuda:{rank}")
            torch.cuda.synchronize()
            dist.barrier()
            comm.all_reduce_host(host, dev, op="mean", wire=TD[wire], piece=piece)
            torch.cuda.synchronize()
            assert comm.async_error() == 0, "watchdog"
            got = host.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else host.numpy()
            q = 16 // (2 if wire in ("f16", "bf16") else 4)
            P = D if piece == 0 else piece
            for off in range(0, D, P):
                n = min(P, D - off)
                R = comm.round_elems(TD[wire])
                ref = oracle.torus_allreduce([a[off:off + n].copy() for a in ins], X, Y, dtype, wire=wire,
                                             op="mean", q=q, round_elems=R)[rank]
                ok, nbad = _same(got[off:off + n], ref)
                assert ok, f"rank {rank} host {dtype}/{wire} D={D} piece@{off}: {nbad} mismatches"
            dist.barrier()
        dist.barrier()
        comm.destroy()
        dist.destroy_process_group()
    except Exception:
        with open(errfile, "a") as f:
            f.write(f"rank {rank}:\n{traceback.format_exc()}\n")
        raise


@pytest.mark.parametrize("world", [2, 4])
def test_allreduce_host_pipelined(tmp_path, world):
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    errfile = str(tmp_path / "errors.txt")
    try:
        mp.spawn(_host_worker, args=(world, _free_port(), errfile), nprocs=world, join=True)
    except Exception as e:
        msg = open(errfile).read() if os.path.exists(errfile) else str(e)
        raise AssertionError(msg) from None


def _concurrent_worker(rank, world, port, errfile):
    """Two communicators with split CTA budgets (TorusComm.init(ctas=SMs/2)) running the
    LL128 kernel concurrently on two streams: both kernels must co-reside (their CTAs spin
    on peers) and both results must equal the oracle."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import torch.distributed as dist

        import oracle
        import synthetic
        from paper_1811_05233_b200 import TorusComm
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        X, Y = (1, 2) if world == 2 else (2, 2)
        sms = torch.cuda.get_device_properties(rank).multi_processor_count
        comms = [TorusComm.init(X=X, Y=Y, ctas=sms // 2) for _ in range(2)]
        streams = [torch.cuda.Stream() for _ in range(2)]
        D = 4_000_037  # 8 MB of f16: above the one-shot / two-shot thresholds at N = 2 and 4
        ins = [synthetic.make_all("normal", D, world, "f16", salt=s) for s in (5, 6)]
        assert comms[0].route(D, torch.float16) == "torus_ll128_kernel"
        for rep in range(3):
            ts = [_to_dev(ins[k][rank], "f16", f"cuda:{rank}") for k in range(2)]
            torch.cuda.synchronize()
            dist.barrier()
            for k in range(2):
                with torch.cuda.stream(streams[k]):
                    comms[k].all_reduce(ts[k], op="mean", stream=streams[k])
            torch.cuda.synchronize()
            for k in range(2):
                assert comms[k].async_error() == 0, "watchdog"
                ref = oracle.torus_allreduce(ins[k], X, Y, "f16", wire="f16", op="mean", q=8,
                                             round_elems=comms[k].round_elems(torch.float16))[rank]
                ok, nbad = _same(_from_dev(ts[k], "f16"), ref)
                assert ok, f"rank {rank} comm {k} rep {rep}: {nbad} mismatches"
            dist.barrier()
        for c in comms:
            dist.barrier()
            c.destroy()
        dist.destroy_process_group()
    except Exception:
        with open(errfile, "a") as f:
            f.write(f"rank {rank}:\n{traceback.format_exc()}\n")
        raise


@pytest.mark.parametrize("world", [2, 4])
def test_concurrent_comms_split_ctas(tmp_path, world):
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    errfile = str(tmp_path / "errors.txt")
    try:
        mp.spawn(_concurrent_worker, args=(world, _free_port(), errfile), nprocs=world, join=True)
    except Exception as e:
        msg = open(errfile).read() if os.path.exists(errfile) else str(e)
        raise AssertionError(msg) from None


def _oversub_worker(rank, world, port, ngpu, errfile):
    """The 8-rank 2x4 headline grid as 8 real processes on `ngpu` GPUs (8 / ngpu ranks per
    GPU, each comm capped to its share of the SMs so the spinning kernels co-reside): CUDA
    IPC between every pair of processes, NVLink between GPUs, the LL128 kernel at 2x4."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import torch.distributed as dist

        import oracle
        import synthetic
        from paper_1811_05233_b200 import TorusComm
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                          TORUS_LL_MAX_BYTES="0", TORUS_LL2_MAX_BYTES="0")
        dev = rank % ngpu
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        comm = TorusComm.init(X=2, Y=4, ctas=sms // (world // ngpu))
        assert comm.route(1_000_003, torch.float16) == "torus_ll128_kernel"
        for dtype, wire, D in [("f16", "f16", 1_000_003), ("f32", "f16", 300_007), ("bf16", "bf16", 200_003),
                               ("f16", "f16", synthetic.RESNET50_NUMEL)]:
            ins = synthetic.make_all("grad" if dtype == "f16" else "normal", D, world, dtype, salt=D % 83)
            t = _to_dev(ins[rank], dtype, f"cuda:{dev}")
            torch.cuda.synchronize()
            dist.barrier()
            comm.all_reduce(t, op="mean", wire=TD[wire])
            torch.cuda.synchronize()
            assert comm.async_error() == 0, "watchdog"
            got = _from_dev(t, dtype)
            q = 16 // (2 if wire in ("f16", "bf16") else 4)
            R = comm.round_elems(TD[wire])
            if D <= 1_000_003:
                ref = oracle.torus_allreduce(ins, 2, 4, dtype, wire=wire, op="mean", q=q, round_elems=R)[rank]
                ok, nbad = _same(got, ref)
            else:
                g = np.random.Generator(np.random.PCG64(rank))
                idx = np.unique(np.concatenate([g.integers(0, D, 4000), [0, D - 1]]))
                ref = oracle.torus_elements(ins, 2, 4, idx, dtype, wire=wire, op="mean", q=q, round_elems=R)
                ok, nbad = _same(got[idx], ref)
            assert ok, f"rank {rank} 2x4 {dtype}/{wire} D={D}: {nbad} mismatches"
            dist.barrier()
        dist.barrier()
        comm.destroy()
        dist.destroy_process_group()
    except Exception:
        with open(errfile, "a") as f:
            f.write(f"rank {rank}:\n{traceback.format_exc()}\n")
        raise


def test_eight_ranks_2x4_oversubscribed(tmp_path):
    """N = 8, 2x4 (BASELINE.json's headline grid) on the GPUs this box has (4 or 2)."""
    import torch.multiprocessing as mp
    ngpu = torch.cuda.device_count()
    if ngpu < 2 or 8 % ngpu:
        pytest.skip("needs 2, 4 or 8 GPUs")
    errfile = str(tmp_path / "errors.txt")
    try:
        mp.spawn(_oversub_worker, args=(8, _free_port(), ngpu, errfile), nprocs=8, join=True)
    except Exception as e:
        msg = open(errfile).read() if os.path.exists(errfile) else str(e)
        raise AssertionError(msg) from None
