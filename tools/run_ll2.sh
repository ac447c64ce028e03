#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ll2 or interleaved" > $O/ll2_parity.txt 2>&1
echo "rc=$?" >> $O/ll2_parity.txt
grep -q "rc=0" $O/ll2_parity.txt || exit 1
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -k "four and twoshot" > $O/ll2_multiproc.txt 2>&1
echo "rc=$?" >> $O/ll2_multiproc.txt
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
TORUS_LL2_MAX_BYTES=8388608 timeout 400 $P 4 --master-addr 127.0.0.1 --master-port 29693 tools/sweep_sizes.py --grid 2x2 --min-bytes 1048576 --max-bytes 16777216 --impls torus,torus_mp,nccl > $O/ll2_sizes_n4.jsonl 2>&1
