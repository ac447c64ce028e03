"""N = 1 cast round trip under the bench's rotation protocol (no L2 flush; NB buffers of
the full workload in rotation, so every call reads a cold buffer and inherits the dirty
lines the previous call left): the castscale kernel variants against torch's own copy of
the same bytes (read 102 MB + write 102 MB).  One JSON line per variant.
Usage (GPU box): python tools/cast_probe.py [calls [variant ...]]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_1811_05233_b200 import TorusComm  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 200
D = synthetic.RESNET50_NUMEL
x0 = torch.from_numpy(synthetic.make("grad", D, 0, "f32")).cuda()
NB = 4
ring = [x0.clone() for _ in range(NB)]
comm = TorusComm.init(X=1, Y=1)


def timed(fn, n):
    for i in range(10):
        fn(i)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for i in range(n):
        ev[i][0].record()
        fn(i)
        ev[i][1].record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return {"mean_us": round(sum(t) / n, 2), "p50_us": round(t[n // 2], 2), "min_us": round(t[0], 2)}


def report(name, r):
    r["name"] = name
    r["gbs_alg"] = round(2 * 4 * D / (r["mean_us"] * 1e-6) / 1e9, 1)
    print(json.dumps(r), flush=True)


# variants: "tma:<NB>x<cps>", "ldg:<U>x<BLK>x<cps>", "cache:<load>,<store>" (see torus_kernels.cu)
specs = sys.argv[2:] or ["tma:6x1", "tma:4x1", "ldg:1x512x0", "ldg:2x256x0", "ldg:4x256x4"]
variants = []
for sp in specs:
    kind, arg = sp.split(":")
    env = {"tma": {"TORUS_CS_KERNEL": "tma", "TORUS_CS_TMA": arg}, "ldg": {"TORUS_CS": arg},
           "cache": {"TORUS_CS_CACHE": arg}}[kind]
    variants.append((sp, env))
for name, env in variants:
    saved = {k: os.environ.get(k) for k in ("TORUS_CS_TMA", "TORUS_CS_KERNEL", "TORUS_CS", "TORUS_CS_CACHE")}
    for k in saved:
        os.environ.pop(k, None)
    os.environ.update(env)
    report(name, timed(lambda i: comm.all_reduce(ring[i % NB], wire=torch.float16), calls))
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
# torch's copy of the same bytes: read one buffer, write another (rotating pairs)
report("torch copy_", timed(lambda i: ring[(i + 1) % NB].copy_(ring[i % NB]), calls))
# torch copy in place of a pair that was just... (read+write the same buffer: x.mul_(1))
report("torch mul_(1) in place", timed(lambda i: ring[i % NB].mul_(1.0), calls))
comm.destroy()
