#!/bin/bash
# One documented driver for multi-GPU measurement calls under gpurun (replaces the
# round-1 one-off run*.sh launchers).  Usage (on the GPU box, from the repo root):
#   tools/run_gpu.sh bench  N TAG [bench.py args...]   -> gpurun_out/TAG.json (+ .log)
#   tools/run_gpu.sh tests  EXPR TAG                    -> pytest -m gpu -k EXPR  -> gpurun_out/TAG.txt
set -u
mode=$1; shift
mkdir -p gpurun_out
case "$mode" in
  bench)
    n=$1; tag=$2; shift 2
    port=$((29500 + RANDOM % 1000))
    if [ "$n" = 1 ]; then
      python bench.py --gpus 1 "$@" > gpurun_out/$tag.log 2>&1
    else
      python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $port bench.py --gpus $n "$@" > gpurun_out/$tag.log 2>&1
    fi
    rc=$?
    grep '^{' gpurun_out/$tag.log > gpurun_out/$tag.json
    echo "== $tag rc=$rc"; tail -c 1500 gpurun_out/$tag.json; echo
    ;;
  tests)
    expr=$1; tag=$2
    timeout 3000 python -m pytest tests -m gpu -x -q -k "$expr" > gpurun_out/$tag.txt 2>&1
    echo "== $tag rc=$?"; tail -15 gpurun_out/$tag.txt
    ;;
esac
