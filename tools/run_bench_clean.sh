#!/bin/bash
O=gpurun_out
timeout 300 python bench.py > $O/bc_n1.log 2>&1
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
timeout 300 $P 2 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 2 > $O/bc_n2.log 2>&1
timeout 300 $P 4 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 4 > $O/bc_n4.log 2>&1
