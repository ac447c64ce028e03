"""One rank of a multi-GPU all-reduce run for profiling RANK 0 ALONE under ncu while the
other ranks run plainly (a multi-rank command must never be wrapped in ncu; one rank's
process can be).  Rendezvous is file-based, one "session" per run, so the plain run that
the GPU box's ncu wrapper performs before profiling pairs with a first session of the
peers and the profiled run with a second one.

  python tools/ncu_worker.py RANK WORLD X Y DIR [count] [calls]

Each session: init a gloo group through a FileStore in DIR/session_<k>, build a
TorusComm (X x Y), register the buffer, 3 warm-up calls, then `calls` timed calls (the
ncu command line selects which launch it measures), barrier, destroy."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def session_id(d, rank):
    """Rank 0: claim the next free session number; others: passed by the caller."""
    k = 0
    while True:
        try:
            fd = os.open(os.path.join(d, f"claim_{k}"), os.O_CREAT | os.O_EXCL | os.O_WRONLY)
            os.close(fd)
            return k
        except FileExistsError:
            k += 1


def run(rank, world, X, Y, d, count, calls, sid):
    import torch.distributed as dist
    import synthetic
    from paper_1811_05233_b200 import TorusComm
    sd = os.path.join(d, f"session_{sid}")
    os.makedirs(sd, exist_ok=True)
    store = dist.FileStore(os.path.join(sd, "store"), world)
    dist.init_process_group("gloo", store=store, rank=rank, world_size=world,
                            timeout=__import__("datetime").timedelta(seconds=120))
    torch.cuda.set_device(rank)
    comm = TorusComm.init(X=X, Y=Y)
    x = torch.from_numpy(synthetic.make("grad", count, rank, "f16")).cuda()
    comm.register(x)
    for _ in range(3):
        comm.all_reduce(x, op="mean")
    torch.cuda.synchronize()
    dist.barrier()
    for _ in range(calls):
        comm.all_reduce(x, op="mean")
    torch.cuda.synchronize()
    err = comm.async_error()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()
    print(f"rank {rank} session {sid}: {calls} calls, async_error={err}, route={comm.__class__.__name__}", flush=True)
    return err


if __name__ == "__main__":
    rank, world, X, Y = map(int, sys.argv[1:5])
    d = sys.argv[5]
    count = int(sys.argv[6]) if len(sys.argv) > 6 else 25_557_032
    calls = int(sys.argv[7]) if len(sys.argv) > 7 else 3
    os.makedirs(d, exist_ok=True)
    if rank == 0:
        sys.exit(1 if run(rank, world, X, Y, d, count, calls, session_id(d, rank)) else 0)
    # peers: serve sessions 0, 1, ... until one times out waiting for rank 0
    sid = 0
    while True:
        t0 = time.time()
        while not os.path.exists(os.path.join(d, f"claim_{sid}")):
            if time.time() - t0 > 90:
                sys.exit(0)
            time.sleep(0.2)
        run(rank, world, X, Y, d, count, calls, sid)
        sid += 1
