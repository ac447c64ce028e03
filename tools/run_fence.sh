#!/bin/bash
O=gpurun_out
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for FE in 0 1; do
  for G in 2x2 4x1; do
    TORUS_FENCE_EARLY=$FE timeout 300 $P --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 200 --no-e2e --grid $G > $O/fe${FE}_$G.log 2>&1
  done
done
TORUS_FENCE_EARLY=1 timeout 200 $P --master-port 29799 tools/trace.py --grid 2x2 > $O/trace_fe1_2x2.jsonl 2>/dev/null
