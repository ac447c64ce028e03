"""NVLink / flag calibration through libtorus's probe kernel.
Run under torchrun on N GPUs; rank 0 prints one JSON line per measurement:
push / pull GB/s per rank (one direction, all peers at once, both directions busy),
local HBM copy, and the flag ping-pong one-way latency alpha."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_05233_b200 import TorusComm  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = TorusComm.init(X=world, Y=1, ws_bytes=1 << 30)
    s = torch.cuda.current_stream()
    nbytes = 51_114_064 * 2 * (world - 1) // world // 16 * 16  # 2(N-1)/N * S
    out = []
    only = os.environ.get("PROBE_ONLY")
    for mode, name in ((0, "push"), (1, "pull"), (4, "tma_push"), (5, "tma_pull"), (3, "local_copy"),
                       (10, "store16"), (11, "store32")):
        if only and name not in only.split(","):
            continue
        for ctas in ((16, 32, 64, 148, 296) if mode < 4 or mode >= 10 else (16, 32, 64, 148)):
            for _ in range(3):
                comm.probe(mode, nbytes, ctas=ctas)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            it = 20
            for _ in range(it):
                comm.probe(mode, nbytes, ctas=ctas)
            e1.record(s)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 1e3 / it], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            gbs = nbytes / t.item() / 1e9
            rec = {"probe": name, "ctas": ctas, "bytes": nbytes, "us": t.item() * 1e6,
                   "GBps_per_rank": gbs * (2 if mode == 3 else 1), "n": world}
            if rank == 0:
                print(json.dumps(rec), flush=True)
            dist.barrier()
    for mode, name in ((7, "fence_quiet"), (6, "fence_under_tma_push"), (8, "fence_in_cta_pushing"), (9, "fence_in_cta_pulling")):
        torch.cuda.synchronize()
        dist.barrier()
        ns = comm.probe(mode, nbytes, ctas=148)
        torch.cuda.synchronize()
        if rank == 0:
            print(json.dumps({"probe": name, "ns_per_fence": ns}), flush=True)
        dist.barrier()
    if world >= 2:
        torch.cuda.synchronize()
        dist.barrier()
        ns = comm.probe(2, 0, iters=2000)
        if rank == 0:
            print(json.dumps({"probe": "pingpong", "iters": 2000, "one_way_us": ns / 2000 / 2 / 1e3,
                              "async_error": comm.async_error()}), flush=True)
        torch.cuda.synchronize()
    dist.barrier()
    comm.destroy()
    if rank == 0:
        for o in out:
            print(json.dumps(o))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
