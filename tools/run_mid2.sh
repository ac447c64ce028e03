#!/bin/bash
O=gpurun_out
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
timeout 500 $P 4 --master-addr 127.0.0.1 --master-port 29691 tools/sweep_sizes.py --grid 2x2 --min-bytes 4194304 --max-bytes 134217728 --impls torus_mp,torus_mpm2o4096,torus_mpm1o8192,torus_mpm2o8192,torus_mpm3o16384,nccl > $O/mid2_n4.jsonl 2>&1
timeout 500 $P 2 --master-addr 127.0.0.1 --master-port 29692 tools/sweep_sizes.py --grid 1x2 --min-bytes 4194304 --max-bytes 134217728 --impls torus_mp,torus_mpm2o4096,torus_mpm2o8192,torus_mpm3o16384,nccl > $O/mid2_n2.jsonl 2>&1
