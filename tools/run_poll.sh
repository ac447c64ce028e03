#!/bin/bash
O=gpurun_out
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for S in 64 0 256; do
  TORUS_POLL_SLEEP=$S TORUS_LL_MAX_BYTES=0 timeout 200 $P --master-port $((29500 + RANDOM % 300)) tools/trace.py --grid 2x2 --count 2048 > $O/poll${S}_trace.jsonl 2>/dev/null
  TORUS_POLL_SLEEP=$S timeout 300 $P --master-port $((29500 + RANDOM % 300)) bench.py --gpus 4 --no-e2e > $O/poll${S}_bench.log 2>&1
done
