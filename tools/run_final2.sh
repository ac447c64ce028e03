#!/bin/bash
O=gpurun_out
tools/run_final.sh
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
timeout 500 $P 4 --master-addr 127.0.0.1 --master-port 29696 tools/sweep_sizes.py --grid 2x2 --min-bytes 4096 --max-bytes 134217728 --impls torus,nccl > $O/f2_sizes_n4.jsonl 2>&1
timeout 500 $P 2 --master-addr 127.0.0.1 --master-port 29697 tools/sweep_sizes.py --grid 1x2 --min-bytes 4096 --max-bytes 134217728 --impls torus,nccl > $O/f2_sizes_n2.jsonl 2>&1
