"""Trace one pull-kernel call on N real GPUs and summarise where the time goes.

  python tools/pull_trace.py N [X Y] [count]     (spawns N ranks; writes gpurun_out/pull_trace_*.npz)

Per CTA kind: start/end offsets, per-job waits: flags-seen -> operands-landed (TMA pull
latency incl. queueing), consumer time, consumer-done -> flags-raised (fence + stores),
and the gap between consecutive jobs' flag-seen stamps."""
import os
import socket
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
KINDS = ["S0", "R", "VR", "VA", "H", "SIG"]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, X, Y, D, out):
    os.environ["TORUS_TRACE"] = "1"
    import torch.distributed as dist
    import synthetic
    from paper_1811_05233_b200 import TorusComm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = TorusComm.init(X=X, Y=Y)
    x = torch.from_numpy(synthetic.make("grad", D, rank, "f16")).cuda()
    if os.environ.get("TRACE_REGISTER", "1") == "1":
        comm.register(x)
    for _ in range(5):
        comm.all_reduce(x, op="mean")
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    comm.all_reduce(x, op="mean")
    e1.record()
    torch.cuda.synchronize()
    tr, g, kinds = comm.pull_trace()
    np.savez(f"{out}_rank{rank}.npz", trace=tr[: g], kinds=np.array(kinds), us=e0.elapsed_time(e1) * 1e3)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


def summarise(out, world):
    for r in range(world):
        z = np.load(f"{out}_rank{r}.npz")
        tr, kinds, us = z["trace"].astype(np.int64), list(z["kinds"]), float(z["us"])
        t0 = tr[:, 63, 0][tr[:, 63, 0] > 0].min()
        print(f"rank {r}: call {us:.1f} us (events), CTA split {dict(zip(KINDS, kinds))}")
        b = 0
        for k, g in zip(KINDS, kinds):
            if g == 0:
                continue
            blk = tr[b:b + g]
            b += g
            st = (blk[:, 63, 0] - t0) / 1e3
            en = (blk[:, 63, 1] - t0) / 1e3
            j = blk[:, :63, :]
            valid = (j[:, :, 0] > 0) & (j[:, :, 1] > 0) & (j[:, :, 2] > 0)
            land = (j[:, :, 1] - j[:, :, 0])[valid] / 1e3
            cons = (j[:, :, 2] - j[:, :, 1])[valid] / 1e3
            sig_ok = valid & (j[:, :, 3] > 0)
            sig = (j[:, :, 3] - j[:, :, 2])[sig_ok] / 1e3
            st_ok = valid & (j[:, :, 4] > 0) & (j[:, :, 5] > 0)
            st_issue = (j[:, :, 4] - j[:, :, 2])[st_ok] / 1e3
            st_read = (j[:, :, 5] - j[:, :, 4])[st_ok] / 1e3
            st_pub = (j[:, :, 3] - j[:, :, 5])[st_ok & sig_ok] / 1e3
            first = (j[:, 0, 0] - t0)[j[:, 0, 0] > 0] / 1e3
            gaps = []
            for row in j[:, :, 0]:
                v = row[row > 0]
                if len(v) > 1:
                    gaps.extend(np.diff(v) / 1e3)
            pc = lambda a: "n/a" if len(a) == 0 else f"p10 {np.percentile(a,10):.2f} p50 {np.median(a):.2f} p90 {np.percentile(a,90):.2f}"
            print(f"  {k:2s} x{g:3d}: start {st.min():.1f}-{st.max():.1f} end {en.min():.1f}-{en.max():.1f} us; "
                  f"jobs/CTA {valid.sum(1).mean():.1f}; first flags-seen {pc(first)}")
            print(f"        land {pc(land)} | consume {pc(cons)} | signal {pc(sig)} | job gap {pc(np.array(gaps))}")
            print(f"        store issue {pc(st_issue)} | store read {pc(st_read)} | read->flags {pc(st_pub)}")


if __name__ == "__main__":
    import torch.multiprocessing as mp
    world = int(sys.argv[1])
    X, Y = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else ((1, 2) if world == 2 else (2, 2))
    D = int(sys.argv[4]) if len(sys.argv) > 4 else 25_557_032
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    out = os.path.join(ROOT, "gpurun_out", f"pull_trace_{X}x{Y}")
    mp.spawn(worker, args=(world, free_port(), X, Y, D, out), nprocs=world, join=True)
    summarise(out, world)
