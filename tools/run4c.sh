#!/bin/bash
O=gpurun_out
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest4c.log 2>&1; echo rc=$? >> $O/pytest4c.log
timeout 300 $P --master-port 29631 bench.py --gpus 4 --steps 200 --no-e2e --algo ring > $O/d4_ring.log 2>&1
TORUS_TILE=1920 timeout 300 $P --master-port 29632 bench.py --gpus 4 --steps 200 > $O/d4_torus.log 2>&1
timeout 300 $P --master-port 29633 tools/bench_buckets.py --streams 1 > $O/d4_buckets1.log 2>&1
timeout 300 $P --master-port 29634 tools/bench_buckets.py --streams 2 > $O/d4_buckets2.log 2>&1
timeout 900 $P --master-port 29635 tools/sweep_sizes.py > $O/sizes_n4.jsonl 2> $O/sizes_n4.err
