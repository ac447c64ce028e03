"""Stress check of the LL128 kernel's flag-in-data assumption on real GPUs: K calls with
fresh random inputs of varying sizes, each result compared bit for bit (on the GPU) with
the push kernel's result on the same inputs -- the push kernel is bit-exact vs the oracle
and does not depend on 128-byte line atomicity.  Under torchrun; rank 0 prints a summary.

  python -m torch.distributed.run --nproc-per-node N tools/ll128_stress.py [calls]"""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_05233_b200 import TorusComm  # noqa: E402


def comm_with(kernel, X, Y):
    old = os.environ.get("TORUS_KERNEL")
    os.environ["TORUS_KERNEL"] = kernel
    os.environ["TORUS_LL_MAX_BYTES"] = "0"
    os.environ["TORUS_LL2_MAX_BYTES"] = "0"
    try:
        return TorusComm.init(X=X, Y=Y)
    finally:
        if old is None:
            os.environ.pop("TORUS_KERNEL")
        else:
            os.environ["TORUS_KERNEL"] = old


def main():
    calls = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    world, rank, local = (int(os.environ[k]) for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    X, Y = {2: (1, 2), 4: (2, 2), 8: (2, 4)}[world]
    grids = [(X, Y)] + ([(world, 1)] if world > 2 else [(2, 1)])
    g = torch.Generator(device="cuda")
    bad, total_el, done = 0, 0, 0
    sizes = [25_557_032, 1_000_003, 7_777_777, 300_007, 12_345_678, 31, 4096 * 30 * 8]
    for gx, gy in grids:
        ll = comm_with("ll128", gx, gy)
        ps = comm_with("push", gx, gy)
        assert ll.route(25_557_032, torch.float16) == "torus_ll128_kernel"
        for k in range(calls):
            D = sizes[k % len(sizes)]
            dt = [torch.float16, torch.bfloat16, torch.float32][k % 3]
            g.manual_seed(1000 * k + 17 * rank)
            x = (torch.randn(D, device="cuda", generator=g) * 2 ** -7).to(dt)
            y = x.clone()
            ll.all_reduce(x, op="mean" if k % 2 else "sum")
            ps.all_reduce(y, op="mean" if k % 2 else "sum")
            torch.cuda.synchronize()
            ok = torch.equal(x.view(torch.uint8), y.view(torch.uint8))
            bad += 0 if ok else 1
            total_el += D
            done += 1
        assert ll.async_error() == 0 and ps.async_error() == 0
        ll.destroy()
        ps.destroy()
    t = torch.tensor([bad], device="cuda")
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"world": world, "grids": [f"{a}x{b}" for a, b in grids], "calls": done,
                          "elements_per_rank": total_el, "mismatching_calls_all_ranks": int(t.item())}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
