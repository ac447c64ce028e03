"""Per-iteration device timeline of the torus kernel (TORUS_TRACE=1), under torchrun.
Rank 0 prints, for CTA 0 and averaged over CTAs, what the control warp and the workers
spend each pipeline iteration on (us)."""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

os.environ["TORUS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_1811_05233_b200 import TorusComm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default=None)
    ap.add_argument("--count", type=int, default=synthetic.RESNET50_NUMEL)
    args = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    X, Y = (map(int, args.grid.split("x")) if args.grid else ({2: (1, 2), 4: (2, 2), 8: (2, 4)}[world]))
    comm = TorusComm.init(X=X, Y=Y)
    x = torch.from_numpy(synthetic.make("grad", args.count, rank, "f16")).cuda()
    for _ in range(10):
        comm.all_reduce(x, op="mean")
    torch.cuda.synchronize()
    dist.barrier()
    comm.all_reduce(x, op="mean")
    torch.cuda.synchronize()
    tr = comm.trace().astype(np.int64)  # [G, 64, 8]
    dist.barrier()
    if rank == 0:
        G = tr.shape[0]
        valid = tr[:, :, 0] > 0
        iters = int(valid[0].sum())
        t0 = tr[:, 0, 0].min()
        rel = (tr - t0) / 1e3
        print(json.dumps({"grid": f"{X}x{Y}", "ctas": G, "iters": iters,
                          "kernel_span_us": float(rel[:, :iters, 6].max())}))
        for it in range(iters):
            r = rel[:, it, :]
            m = lambda x: round(float(x.mean()), 2)
            prev6 = rel[:, it - 1, 6] if it > 0 else rel[:, it, 5]
            print(json.dumps({
                "it": it, "ctl_start": m(r[:, 0]), "poll": m(r[:, 1] - r[:, 0]),
                "done_wait": m(r[:, 2] - r[:, 1]), "raise": m(r[:, 4] - r[:, 3]),
                "wk_start": m(r[:, 5]), "wk_idle": m(r[:, 5] - prev6), "wk_busy": m(r[:, 6] - r[:, 5]),
                "wk_busy_max": round(float((r[:, 6] - r[:, 5]).max()), 2)}))
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
