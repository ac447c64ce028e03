"""Config 5: layer-bucketed ResNet-50 gradients (161 tensors, f32 gradients, fp16 wire,
mean) through torus_allreduce_multi, buckets overlapped on per-bucket streams (one comm
per concurrent stream, CTA budgets split so all spinning kernels co-reside).  Buckets:
reverse registration order (backprop order), greedy caps 1 MiB then 25 MiB of fp16 bytes
(DDP's rule).  Under torchrun; rank 0 prints one JSON line."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_1811_05233_b200 import TorusComm  # noqa: E402


def buckets(sizes, first_cap=1 << 20, cap=25 << 20, esz=2):
    out, cur, cur_b, c = [], [], 0, first_cap
    for i, n in enumerate(sizes):
        cur.append(i)
        cur_b += n * esz
        if cur_b >= c:
            out.append(cur)
            cur, cur_b, c = [], 0, cap
    if cur:
        out.append(cur)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=2)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    world, rank, local = (int(os.environ[k]) for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    X, Y = {2: (1, 2), 4: (2, 2), 8: (2, 4)}.get(world, (world, 1))
    sizes = synthetic.resnet50_param_numels()[::-1]
    bks = buckets(sizes)
    K = min(args.streams, len(bks))
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    comms = [TorusComm.init(X=X, Y=Y, ctas=max(1, sms // K)) for _ in range(K)]
    streams = [torch.cuda.Stream() for _ in range(K)]
    grads = [torch.randn(n, device="cuda") * 2 ** -7 for n in sizes]
    for ci, c in enumerate(comms):  # reserve staging so timed calls never allocate
        c.reserve(max(sum(sizes[i] for i in b) for b in bks[ci::K]) * 2 + 4096)

    def step():
        ev = torch.cuda.Event()
        ev.record()
        for bi, b in enumerate(bks):
            k = bi % K
            streams[k].wait_event(ev)
            comms[k].all_reduce_multi([grads[i] for i in b], op="mean", wire=torch.float16,
                                      stream=streams[k])
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3 / args.steps], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # NCCL comparator: the same buckets, fp16-compressed like DDP's fp16 hook
    flat16 = [torch.empty(sum(sizes[i] for i in b), device="cuda", dtype=torch.float16) for b in bks]

    def nccl_step():
        for bi, b in enumerate(bks):
            flat16[bi].copy_(torch.cat([grads[i] for i in b]))
            dist.all_reduce(flat16[bi], op=dist.ReduceOp.AVG)
            off = 0
            for i in b:
                grads[i].copy_(flat16[bi][off:off + sizes[i]])
                off += sizes[i]

    for _ in range(args.warmup):
        nccl_step()
    torch.cuda.synchronize()
    dist.barrier()
    e0.record()
    for _ in range(args.steps):
        nccl_step()
    e1.record()
    torch.cuda.synchronize()
    tn = torch.tensor([e0.elapsed_time(e1) / 1e3 / args.steps], device="cuda", dtype=torch.float64)
    dist.all_reduce(tn, op=dist.ReduceOp.MAX)
    # one flat f32 buffer of the same elements through the torus with fp16 wire (the
    # bound a fused bucket call should approach), and NCCL on pre-flattened buckets: f32
    # (DDP's bucket views, no compression) and fp16 (collective only, no cast cost)
    flat32 = torch.randn(sum(sizes), device="cuda") * 2 ** -7
    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0.record()
        for _ in range(args.steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        x = torch.tensor([e0.elapsed_time(e1) / 1e3 / args.steps], device="cuda", dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        return x.item()
    t_flat = timed(lambda: comms[0].all_reduce(flat32, op="mean", wire=torch.float16))
    bk32 = [torch.randn(sum(sizes[i] for i in b), device="cuda") for b in bks]
    t_nccl32 = timed(lambda: [dist.all_reduce(x, op=dist.ReduceOp.AVG) for x in bk32])
    t_nccl16 = timed(lambda: [dist.all_reduce(x, op=dist.ReduceOp.AVG) for x in flat16])
    S = sum(sizes) * 2
    bus = 2 * (world - 1) / world
    err = max(c.async_error() for c in comms)
    routes = [comms[0].route(sum(sizes[i] for i in b), torch.float32, torch.float16) for b in bks]
    for c in comms:
        c.destroy()
    if rank == 0:
        print(json.dumps({"config": "resnet50 layer-bucketed f32 grads, fp16 wire, mean",
                          "n_gpus": world, "grid": f"{X}x{Y}", "buckets": [len(b) for b in bks],
                          "bucket_elems": [sum(sizes[i] for i in b) for b in bks], "streams": K,
                          "us_per_step": t.item() * 1e6, "busbw_fp16": S / t.item() / 1e9 * bus,
                          "flat_single_call_us": t_flat * 1e6,
                          "ratio_to_flat": t.item() / t_flat,
                          "routes": routes,
                          "nccl_fp16_hook_us": tn.item() * 1e6,
                          "nccl_bucket_f32_us": t_nccl32 * 1e6, "nccl_bucket_fp16_collective_only_us": t_nccl16 * 1e6,
                          "nccl_busbw_fp16": S / tn.item() / 1e9 * bus, "async_error": err}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
