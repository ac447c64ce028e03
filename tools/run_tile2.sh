#!/bin/bash
O=gpurun_out
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for R in 1 2; do
for G in 2x2 4x1; do
for T in 0 2700; do
  TORUS_TILE=$T timeout 300 $P 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py --gpus 4 --grid $G --no-e2e --no-nccl --no-cpu --steps 300 > $O/tile2_${G}_${T}_r$R.log 2>&1
done; done; done
