#!/bin/bash
O=gpurun_out
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
timeout 500 $P 4 --master-addr 127.0.0.1 --master-port 29694 tools/sweep_sizes.py --grid 2x2 --min-bytes 262144 --max-bytes 16777216 --ll-max 8388608 --impls torus_ll,torus_ll2,torus_mp,nccl > $O/ll2b_n4_2x2.jsonl 2>&1
timeout 500 $P 4 --master-addr 127.0.0.1 --master-port 29695 tools/sweep_sizes.py --grid 4x1 --min-bytes 262144 --max-bytes 16777216 --ll-max 8388608 --impls torus_ll,torus_ll2,torus_mp,nccl > $O/ll2b_n4_4x1.jsonl 2>&1
