#!/bin/bash
O=gpurun_out
run() { local name=$1; shift; env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 200 --no-e2e $EXTRA > $O/c4_$name.log 2>&1; }
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest4b.log 2>&1; echo rc=$? >> $O/pytest4b.log
EXTRA=""
run 2x2_t1920 TORUS_TILE=1920
run 2x2_t3840 TORUS_TILE=3840
run 2x2_t7680 TORUS_TILE=7680
run 2x2_nocopy TORUS_TILE=1920 TORUS_COPY=0
EXTRA="--grid 4x1"; run 4x1 TORUS_TILE=3840
EXTRA="--grid 1x4"; run 1x4 TORUS_TILE=3840
