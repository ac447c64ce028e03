#!/bin/bash
O=gpurun_out
export TORUS_LL_MAX_BYTES=0
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for G in 2x2 4x1; do
  timeout 200 $P --master-port $((29500 + RANDOM % 300)) tools/trace.py --grid $G --count 2048 > $O/trace_small_$G.jsonl 2>$O/trace_small_$G.err
done
