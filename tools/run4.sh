#!/bin/bash
# 4-GPU measurement pass (run under gpurun --gpus 4).  Outputs in gpurun_out/.
O=gpurun_out
run() {  # run NAME ENV... -- ARGS
  local name=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
      --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 \
      --steps 200 --no-e2e $EXTRA > $O/b4_$name.log 2>&1
}
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest4.log 2>&1; echo rc=$? >> $O/pytest4.log
EXTRA=""
run 2x2_t3840 TORUS_TILE=3840
run 2x2_t1920 TORUS_TILE=1920
run 2x2_t7680 TORUS_TILE=7680
EXTRA="--grid 1x4"; run 1x4 TORUS_TILE=3840
EXTRA="--grid 4x1"; run 4x1 TORUS_TILE=3840
EXTRA=""; run nccl_nonvls NCCL_NVLS_ENABLE=0
EXTRA=""; run nccl_ring NCCL_ALGO=Ring
timeout 300 python bench.py --steps 100 > $O/b1_final.log 2>&1
