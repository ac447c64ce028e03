"""Run bench.py once per environment setting and print one compact line per run.

  python tools/sweep_env.py N "ENV=a ENV2=b" "ENV=c" ...   [-- extra bench args]

Each run: --steps 50 --warmup 5, no NCCL / e2e / oracle legs unless extra args say so.
Lines go to stdout and are appended to gpurun_out/sweep.jsonl."""
import json
import os
import random
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = int(sys.argv[1])
rest = sys.argv[2:]
extra = []
if "--" in rest:
    i = rest.index("--")
    rest, extra = rest[:i], rest[i + 1:]
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
for spec in rest:
    env = dict(os.environ)
    for kv in spec.split():
        k, v = kv.split("=", 1)
        env[k] = v
    args = ["--gpus", str(n), "--steps", "50", "--warmup", "5", "--no-nccl", "--no-e2e", "--no-cpu"] + extra
    if n == 1:
        cmd = [sys.executable, "bench.py"] + args
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr", "127.0.0.1", f"--master-port={29500 + random.randint(0, 999)}",
               "bench.py"] + args
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    line = [l for l in p.stdout.splitlines() if l.startswith("{")]
    if p.returncode != 0 or not line:
        print(f"{spec:60s} FAILED rc={p.returncode} {p.stderr[-300:]!r}", flush=True)
        continue
    d = json.loads(line[-1])
    out = {"n": n, "env": spec, "extra": " ".join(extra), "us": d["us_per_call"], "us_min": d["us_per_call_min"],
           "us_p50": d.get("us_per_call_p50"), "us_p90": d.get("us_per_call_p90"), "us_max": d.get("us_per_call_max"),
           "busbw": d["busbw"], "kernel": d["roofline"].get("kernel"), "sanity": d["sanity"]}
    print(f"{spec:60s} {d['us_per_call']:8.1f} us  busbw {d['busbw']:6.1f}  min {d['us_per_call_min']:7.1f}  "
          f"p50 {d.get('us_per_call_p50', 0):7.1f} p90 {d.get('us_per_call_p90', 0):7.1f} max {d.get('us_per_call_max', 0):8.1f}  "
          f"{d['roofline'].get('kernel')} ok={d['sanity'].get('ranks_identical')}", flush=True)
    with open(os.path.join(ROOT, "gpurun_out", "sweep.jsonl"), "a") as f:
        f.write(json.dumps(out) + "\n")
