"""Quick single-GPU parity sweep of the pull kernel on virtual grids (development aid;
tests/test_gpu_parity.py is the gate).  Usage: python tools/pull_check.py [X Y ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synthetic  # noqa: E402
from paper_1811_05233_b200 import VirtualTorus  # noqa: E402

TD = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16, "i32": torch.int32}


def dev(a, dt):
    if dt == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(a.copy()).cuda()


def host(t, dt):
    if dt == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


os.environ.setdefault("TORUS_LL_MAX_BYTES", "0")
os.environ.setdefault("TORUS_LL2_MAX_BYTES", "0")
grids = [(2, 1), (1, 2), (2, 2), (2, 4), (4, 2), (3, 3)]
if len(sys.argv) > 2:
    v = list(map(int, sys.argv[1:]))
    grids = list(zip(v[::2], v[1::2]))
bad = 0
for X, Y in grids:
    vt = VirtualTorus(X, Y, device=0)
    N = X * Y
    print(f"grid {X}x{Y} route(1M f16) = {vt.route(1 << 20, torch.float16)} ctas={vt.ctas()}", flush=True)
    for dt, w in (("f16", "f16"), ("f32", "f32"), ("i32", "i32"), ("bf16", "bf16"), ("f32", "f16")):
        R = vt.round_elems(TD[w])
        for D in (1, 7, 1000, 4099, 200_003, 1_000_001):
            ins = synthetic.make_all("full" if dt == "i32" else "normal", D, N, dt, salt=D % 13)
            ts = [dev(a, dt) for a in ins]
            t0 = time.time()
            vt.all_reduce(ts, op="mean", wire=TD[w])
            torch.cuda.synchronize()
            err = vt.async_error()
            ref = oracle.torus_allreduce(ins, X, Y, dt, wire=w, op="mean", q=16 // (2 if w in ("f16", "bf16") else 4),
                                         round_elems=R)
            nbad = 0
            for r in range(N):
                g = host(ts[r], dt)
                wd = {2: np.uint16, 4: np.uint32}[g.dtype.itemsize]
                eq = g.view(wd) == ref[r].view(wd)
                if g.dtype != np.uint16 and g.dtype.kind == "f":
                    eq |= np.isnan(g) & np.isnan(ref[r])
                nbad += int((~eq).sum())
            status = "OK" if nbad == 0 and err == 0 else f"FAIL nbad={nbad} err={err}"
            if nbad or err:
                bad += 1
            print(f"  {X}x{Y} {dt}/{w} D={D}: {status} ({time.time() - t0:.2f}s)", flush=True)
            if err:
                break
        if vt.async_error():
            break
    vt.destroy()
print("ALL OK" if bad == 0 else f"{bad} FAILURES")
