"""Small single-GPU run of every route on a virtual 2x2 grid (and the N=1 cast pass), for
compute-sanitizer (racecheck / synccheck).  Each call is checked against the oracle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synthetic  # noqa: E402
from paper_1811_05233_b200 import VirtualTorus  # noqa: E402

cases = [("ll128", {"TORUS_KERNEL": "ll128", "TORUS_LL_MAX_BYTES": "0", "TORUS_LL2_MAX_BYTES": "0"}),
         ("pull", {"TORUS_KERNEL": "pull", "TORUS_LL_MAX_BYTES": "0", "TORUS_LL2_MAX_BYTES": "0"}),
         ("push", {"TORUS_KERNEL": "push", "TORUS_LL_MAX_BYTES": "0", "TORUS_LL2_MAX_BYTES": "0"}),
         ("ll", {"TORUS_LL_MAX_BYTES": str(1 << 20), "TORUS_LL2_MAX_BYTES": "0"}),
         ("ll2", {"TORUS_LL_MAX_BYTES": "0", "TORUS_LL2_MAX_BYTES": str(1 << 20)})]
D = int(os.environ.get("SAN_D", "40000"))
for name, env in cases:
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    vt = VirtualTorus(2, 2, device=0, ctas=8, ws_bytes=64 << 20)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    ins = synthetic.make_all("normal", D, 4, "f16")
    ts = [torch.from_numpy(a.copy()).cuda() for a in ins]
    vt.all_reduce(ts, op="mean")
    torch.cuda.synchronize()
    ref = oracle.torus_allreduce(ins, 2, 2, "f16", op="mean", q=8, round_elems=vt.round_elems(torch.float16))
    ok = all(np.array_equal(t.cpu().numpy().view(np.uint16), r.view(np.uint16)) for t, r in zip(ts, ref))
    print(f"{name}: route {vt.route(D, torch.float16)} bit-exact={ok} async_error={vt.async_error()}", flush=True)
    vt.destroy()
vt = VirtualTorus(1, 1, device=0)
x = torch.from_numpy(synthetic.make("normal", 100_003, 0, "f32")).cuda()
vt.all_reduce([x], op="mean", wire=torch.float16)
torch.cuda.synchronize()
print("castscale: ok", flush=True)
vt.destroy()
