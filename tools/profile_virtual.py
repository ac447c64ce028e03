"""Single-GPU run of the product torus kernel on a virtual X-by-Y grid (all ranks in one
cooperative launch) at the full ResNet-50 size -- the configuration ncu can capture
(a multi-process run cannot be replayed by ncu).  Prints device time per call."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_1811_05233_b200 import VirtualTorus  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="2x4")
    ap.add_argument("--count", type=int, default=synthetic.RESNET50_NUMEL)
    ap.add_argument("--calls", type=int, default=5)
    ap.add_argument("--ctas", type=int, default=16)
    args = ap.parse_args()
    X, Y = map(int, args.grid.split("x"))
    vt = VirtualTorus(X, Y, device=0, ctas=args.ctas)
    ts = [torch.from_numpy(synthetic.make("grad", args.count, r, "f16")).cuda() for r in range(X * Y)]
    for _ in range(2):
        vt.all_reduce(ts, op="mean")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.calls):
        vt.all_reduce(ts, op="mean")
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / args.calls
    S = args.count * 2
    print(json.dumps({"grid": args.grid, "virtual_ranks": X * Y, "ctas_per_rank": vt.ctas(),
                      "us_per_call": us, "launches_per_call": vt.launches(args.count, torch.float16),
                      "note": "all ranks on ONE GPU: HBM-bound emulation, not an NVLink number",
                      "async_error": vt.async_error()}))
    vt.destroy()


if __name__ == "__main__":
    main()
