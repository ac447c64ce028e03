#!/bin/bash
O=gpurun_out
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for R in 1 2; do
for V in base u2f2 u2f1 u1f1 u3f2; do
  if [ $V = base ]; then L=paper_1811_05233_b200/libtorus.so; else L=build_variants/libtorus_$V.so; fi
  for N in 4 2; do
    TORUS_LIB_PATH=$PWD/$L timeout 300 $P $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py --gpus $N --no-e2e --no-nccl --no-cpu --steps 300 > $O/unroll2_${V}_n${N}_r$R.log 2>&1
  done
done
done
