#!/bin/bash
O=gpurun_out
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for T in 0 1200 1500 2200 2700 5400; do
  TORUS_TILE=$T timeout 300 $P 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py --gpus 4 --no-e2e --no-nccl --no-cpu --steps 300 > $O/tile_${T}_n4.log 2>&1
done
for T in 0 2700 5400 10800; do
  TORUS_TILE=$T timeout 300 $P 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py --gpus 2 --no-e2e --no-nccl --no-cpu --steps 300 > $O/tile_${T}_n2.log 2>&1
done
