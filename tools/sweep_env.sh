#!/bin/bash
# usage: tools/sweep_env.sh NGPUS "CTAS:TILE ..." [extra bench args]   (run on the GPU box)
N=$1; shift; LIST=$1; shift
P=29600
for CT in $LIST; do
  C=${CT%%:*}; TL=${CT##*:}; P=$((P+1))
  if [ "$N" = 1 ]; then
    TORUS_TILE=$TL timeout 300 python bench.py --gpus 1 --ctas $C --no-cpu --no-e2e "$@" | tail -1
  else
    TORUS_TILE=$TL timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $P bench.py --gpus $N --ctas $C --no-e2e "$@" 2>/dev/null | tail -1
  fi
done
