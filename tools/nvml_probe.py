"""Which NVML NVLink counters does this box expose?  Reads every candidate field (per link
and aggregate) before and after a 1 GiB peer copy GPU0 -> GPU1 and prints the deltas."""
import pynvml as p
import torch

FIELDS = {"THROUGHPUT_DATA_TX": 138, "THROUGHPUT_DATA_RX": 139, "THROUGHPUT_RAW_TX": 140,
          "THROUGHPUT_RAW_RX": 141, "COUNT_XMIT_PACKETS": 201, "COUNT_XMIT_BYTES": 202,
          "COUNT_RCV_PACKETS": 203, "COUNT_RCV_BYTES": 204}
SCOPES = list(range(18)) + [0xFFFFFFFF]


def read(h):
    out = {}
    for name, fid in FIELDS.items():
        vals = p.nvmlDeviceGetFieldValues(h, [(fid, s) for s in SCOPES])
        out[name] = [(v.nvmlReturn, int(v.value.ullVal)) for v in vals]
    return out


p.nvmlInit()
hs = [p.nvmlDeviceGetHandleByIndex(i) for i in range(2)]
a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
b = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:1")
torch.cuda.synchronize(0)
before = [read(h) for h in hs]
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize(0)
torch.cuda.synchronize(1)
after = [read(h) for h in hs]
for g in range(2):
    for name in FIELDS:
        rc = [r for r, _ in after[g][name]]
        d = [a2 - b2 for (_, a2), (_, b2) in zip(after[g][name], before[g][name])]
        print(f"gpu{g} {name}: rc={sorted(set(rc))} delta_per_scope={d}")
