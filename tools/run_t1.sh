#!/bin/bash
O=gpurun_out
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
timeout 400 $P 4 --master-addr 127.0.0.1 --master-port 29671 tools/sweep_sizes.py --grid 2x2 --min-bytes 2097152 --max-bytes 67108864 --impls torus,torus_mp,torus_mpt1000000,nccl > $O/t1_n4.jsonl 2>&1
timeout 400 $P 2 --master-addr 127.0.0.1 --master-port 29672 tools/sweep_sizes.py --grid 1x2 --min-bytes 2097152 --max-bytes 67108864 --impls torus,torus_mp,torus_mpt1000000,nccl > $O/t1_n2.jsonl 2>&1
