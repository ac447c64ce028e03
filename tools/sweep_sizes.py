"""Config 4: message-size sweep (4 KiB .. 1 GiB) of the torus all-reduce, the flat-ring
baseline kernel and NCCL all-reduce on the same tensors, under torchrun (one rank per
GPU).  Per size: device time per call (CUDA events, median of 5 batches, max over
ranks), algbw and busbw.  Rank 0 prints one JSON line per (size, impl)."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1811_05233_b200 import TorusComm  # noqa: E402

TD = {"f16": torch.float16, "bf16": torch.bfloat16, "f32": torch.float32}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default=None)
    ap.add_argument("--dtype", default="f16")
    ap.add_argument("--min-bytes", type=int, default=4096)
    ap.add_argument("--max-bytes", type=int, default=1 << 30)
    ap.add_argument("--impls", default="torus,ring,nccl")
    ap.add_argument("--ll-max", type=int, default=4 << 20)
    args = ap.parse_args()
    world, rank, local = (int(os.environ[k]) for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    X, Y = (map(int, args.grid.split("x")) if args.grid else {2: (1, 2), 4: (2, 2), 8: (2, 4)}[world])
    comm = TorusComm.init(X=X, Y=Y)
    # extra arms: "torus_mp" = multi-phase kernel at every size (one-shot path off);
    # "torus_mpc<G>" = the same with G CTAs; "torus_mpt<V>" = with V-vector tiles; "torus_ll" = one-shot path forced (--ll-max)
    extra = {}
    for impl in args.impls.split(","):
        env = {}
        if impl.startswith("torus_mp"):
            env["TORUS_LL_MAX_BYTES"] = "0"
            env["TORUS_LL2_MAX_BYTES"] = "0"
            if impl.startswith("torus_mpc"):
                env["TORUS_CTAS"] = impl[len("torus_mpc"):]
            elif impl.startswith("torus_mpt"):  # fixed tile (vectors); huge = one tile
                env["TORUS_TILE"] = impl[len("torus_mpt"):]
            elif impl.startswith("torus_mpm"):  # "torus_mpm<tiles>o<one_tile_max>"
                m, o = impl[len("torus_mpm"):].split("o")
                env["TORUS_MID_TILES"], env["TORUS_ONE_TILE_MAX"] = m, o
        elif impl == "torus_ll":
            env["TORUS_LL_MAX_BYTES"] = str(args.ll_max)
            env["TORUS_LL2_MAX_BYTES"] = "0"
        elif impl == "torus_ll2":  # two-shot forced up to --ll-max
            env["TORUS_LL_MAX_BYTES"] = "0"
            env["TORUS_LL2_MAX_BYTES"] = str(args.ll_max)
        else:
            continue
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        extra[impl] = TorusComm.init(X=X, Y=Y)
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    dt = TD[args.dtype]
    esz = torch.tensor([], dtype=dt).element_size()
    bus = 2.0 * (world - 1) / world
    impls = args.impls.split(",")
    nbytes = args.min_bytes
    while nbytes <= args.max_bytes:
        n = nbytes // esz
        x = torch.randn(n, device="cuda").to(dt) * 0.01
        for impl in impls:
            if impl == "torus":
                fn = lambda: comm.all_reduce(x, op="mean")  # noqa: E731
            elif impl in extra:
                fn = lambda c=extra[impl]: c.all_reduce(x, op="mean")  # noqa: E731
            elif impl == "ring":
                fn = lambda: comm.ring_all_reduce(x, op="mean")  # noqa: E731
            else:
                fn = lambda: dist.all_reduce(x, op=dist.ReduceOp.AVG)  # noqa: E731
            iters = max(3, min(200, int(2e9 // max(nbytes, 1) // 50)))
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            times = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(iters):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) / 1e3 / iters)
            t = torch.tensor([sorted(times)[2]], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t = t.item()
            if rank == 0:
                print(json.dumps({"impl": impl, "n_gpus": world, "grid": f"{X}x{Y}", "dtype": args.dtype,
                                  "bytes": nbytes, "us": t * 1e6, "algbw": nbytes / t / 1e9,
                                  "busbw": nbytes / t / 1e9 * bus}), flush=True)
            dist.barrier()
        del x
        nbytes *= 2
    if comm.async_error():
        print(json.dumps({"error": "async error"}))
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
