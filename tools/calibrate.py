"""NVLink calibration on the GPU box (SURVEY.md 8(d) "Calibration"): peer copy GB/s
between GPU 0 and GPU 1, one direction and both directions at once, via
cudaMemcpyPeerAsync (torch cross-device copy).  Single process, >= 2 visible GPUs."""
import json
import sys

import torch


def main(nbytes=51_114_064, iters=50):
    n = torch.cuda.device_count()
    out = {"gpus": n}
    if n < 2:
        print(json.dumps(out)); return
    a0 = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    b1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    a1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda:1")
    b0 = torch.empty(nbytes, dtype=torch.uint8, device="cuda:0")
    s0 = torch.cuda.Stream(device=0)
    s1 = torch.cuda.Stream(device=1)
    for _ in range(5):
        with torch.cuda.stream(s0):
            b1.copy_(a0, non_blocking=True)
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s0):
        e0.record(s0)
        for _ in range(iters):
            b1.copy_(a0, non_blocking=True)
        e1.record(s0)
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    t = e0.elapsed_time(e1) / 1e3 / iters
    out["uni_GBps"] = nbytes / t / 1e9
    # both directions at once
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0, g1 = torch.cuda.Event(enable_timing=True, ), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s0):
        f0.record(s0)
        for _ in range(iters):
            b1.copy_(a0, non_blocking=True)
        f1.record(s0)
    with torch.cuda.device(1), torch.cuda.stream(s1):
        g0.record(s1)
        for _ in range(iters):
            b0.copy_(a1, non_blocking=True)
        g1.record(s1)
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    out["bidir_GBps_per_direction"] = [nbytes / (f0.elapsed_time(f1) / 1e3 / iters) / 1e9,
                                       nbytes / (g0.elapsed_time(g1) / 1e3 / iters) / 1e9]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
