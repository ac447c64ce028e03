#!/bin/bash
O=gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/nd_gpu_tests.txt 2>&1
echo "rc=$?" >> $O/nd_gpu_tests.txt
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
timeout 400 $P 4 --master-addr 127.0.0.1 --master-port 29681 tools/sweep_sizes.py --grid 2x2 --min-bytes 4096 --max-bytes 134217728 --impls torus,nccl > $O/nd_sizes_n4.jsonl 2>&1
timeout 400 $P 2 --master-addr 127.0.0.1 --master-port 29682 tools/sweep_sizes.py --grid 1x2 --min-bytes 4096 --max-bytes 134217728 --impls torus,nccl > $O/nd_sizes_n2.jsonl 2>&1
