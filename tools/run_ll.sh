#!/bin/bash
# one-shot small-message kernel: parity (1 GPU virtual + 2/4 GPU) and the size sweep
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ll or interleaved" > $O/ll_parity.txt 2>&1
echo "parity rc=$?" >> $O/ll_parity.txt
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -k "oneshot" > $O/ll_multiproc.txt 2>&1
echo "multiproc rc=$?" >> $O/ll_multiproc.txt
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
timeout 300 $P 4 --master-addr 127.0.0.1 --master-port 29631 tools/sweep_sizes.py --grid 2x2 --max-bytes 8388608 --impls torus,torus_mp,nccl > $O/ll_sizes_n4.jsonl 2>&1
timeout 300 $P 4 --master-addr 127.0.0.1 --master-port 29632 tools/sweep_sizes.py --grid 4x1 --max-bytes 8388608 --impls torus,torus_mp,nccl > $O/ll_sizes_n4_4x1.jsonl 2>&1
timeout 300 $P 2 --master-addr 127.0.0.1 --master-port 29633 tools/sweep_sizes.py --grid 1x2 --max-bytes 8388608 --impls torus,torus_mp,nccl > $O/ll_sizes_n2.jsonl 2>&1
