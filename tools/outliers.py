"""Per-call device times of back-to-back all-reduce calls (with the bench's L2 eviction
between calls) to find sporadic slow calls.  Under torchrun; rank 0 prints a summary and
the indices / times of calls slower than 1.5x the median (max over ranks per call)."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic  # noqa: E402
from paper_1811_05233_b200 import TorusComm  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 400
count = int(sys.argv[2]) if len(sys.argv) > 2 else synthetic.RESNET50_NUMEL
evict = os.environ.get("EVICT", "1") == "1"
world, rank, local = (int(os.environ[k]) for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
X, Y = {2: (1, 2), 4: (2, 2)}[world]
comm = TorusComm.init(X=X, Y=Y)
x = torch.from_numpy(synthetic.make("grad", count, rank, "f16")).cuda()
comm.register(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
clean = torch.zeros(64 << 20, dtype=torch.int32, device="cuda")
for _ in range(10):
    comm.all_reduce(x)
torch.cuda.synchronize()
dist.barrier()
dist.all_reduce(torch.zeros(1, device="cuda"))  # release the GPUs together (host skew)
if os.environ.get("PRIME", "0") == "1":  # one untimed call right before the timed ones
    comm.all_reduce(x)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(calls)]
for i in range(calls):
    if evict:
        flush.fill_(i & 255)
        clean.max()
    ev[i][0].record()
    comm.all_reduce(x)
    ev[i][1].record()
torch.cuda.synchronize()
t = torch.tensor([a.elapsed_time(b) * 1e3 for a, b in ev], device="cuda", dtype=torch.float64)
dist.all_reduce(t, op=dist.ReduceOp.MAX)
if rank == 0:
    v = t.cpu().tolist()
    med = sorted(v)[len(v) // 2]
    slow = [(i, round(s, 1)) for i, s in enumerate(v) if s > 1.5 * med]
    print(json.dumps({"route": comm.route(count, torch.float16), "calls": calls, "median_us": round(med, 1),
                      "mean_us": round(sum(v) / len(v), 1), "max_us": round(max(v), 1), "n_slow": len(slow),
                      "slow": slow[:40], "evict": evict}))
comm.destroy()
dist.destroy_process_group()
