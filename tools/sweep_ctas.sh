#!/bin/bash
# usage: tools/sweep_ctas.sh NGPUS "16 32 64 ..." [extra bench args]   (run on the GPU box)
N=$1; shift; LIST=$1; shift
for C in $LIST; do
  if [ "$N" = 1 ]; then
    timeout 300 python bench.py --gpus 1 --ctas $C --no-cpu --no-e2e "$@" | tail -1
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29500 + C)) bench.py --gpus $N --ctas $C --no-e2e "$@" 2>/dev/null | tail -1
  fi
done
