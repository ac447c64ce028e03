"""NVLS variant (NEXT-4) check under torchrun: setup, tolerance parity vs an f64 sum
(the switch's summation order is unspecified), and device time vs the torus and NCCL on
the 51 MB fp16 mean message.  Rank 0 prints JSON lines."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_1811_05233_b200 import TorusComm  # noqa: E402


def timeit(fn, iters=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3 / iters], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def main():
    world, rank, local = (int(os.environ[k]) for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    X, Y = {2: (1, 2), 4: (2, 2), 8: (2, 4)}.get(world, (world, 1))
    comm = TorusComm.init(X=X, Y=Y)
    D = synthetic.RESNET50_NUMEL
    comm.nvls_init(D * 2 + (4 << 20))
    out = []
    for dt, wire, tdt in (("f16", None, torch.float16), ("bf16", None, torch.bfloat16),
                          ("f32", None, torch.float32), ("f32", torch.float16, torch.float32)):
        x0 = torch.from_numpy(synthetic.make("grad" if dt != "bf16" else "normal", 1_000_003, rank,
                                             "f32")).cuda().to(tdt)
        ref = x0.double()
        dist.all_reduce(ref)
        ref /= world
        mag = x0.double().abs()
        dist.all_reduce(mag)
        mag /= world
        x = x0.clone()
        comm.nvls_all_reduce(x, op="mean", wire=wire)
        torch.cuda.synchronize()
        err = float(((x.double() - ref).abs() / (mag + 1e-30)).max())
        cs = x.view(torch.uint8).to(torch.int64).sum()
        allcs = [torch.zeros_like(cs) for _ in range(world)]
        dist.all_gather(allcs, cs)
        out.append({"check": f"{dt}/{wire}", "max_err_over_sum_abs": err,
                    "ranks_identical": all(int(c) == int(allcs[0]) for c in allcs),
                    "async_error": comm.async_error()})
    x = torch.from_numpy(synthetic.make("grad", D, rank, "f16")).cuda()
    S = D * 2
    bus = 2 * (world - 1) / world
    for name, fn in (("nvls", lambda: comm.nvls_all_reduce(x, op="mean")),
                     ("torus", lambda: comm.all_reduce(x, op="mean")),
                     ("nccl", lambda: dist.all_reduce(x, op=dist.ReduceOp.AVG))):
        t = timeit(fn)
        out.append({"impl": name, "n_gpus": world, "us": t * 1e6, "busbw": S / t / 1e9 * bus})
    dist.barrier()
    comm.destroy()
    if rank == 0:
        for o in out:
            print(json.dumps(o), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
