#!/bin/bash
# A/B of library builds (TORUS_LIB_PATH) on the per-call outlier tool: N=2 (1x2) and N=4
# (2x2), 400 back-to-back calls each with L2 eviction, all builds interleaved, twice.
# Usage: tools/r02_ab.sh TAG A.so B.so [C.so ...]  -> gpurun_out/TAG.txt
tag=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in "$@"; do
    for n in 2 4; do
      echo -n "$(basename $lib) n=$n rep=$rep " >> gpurun_out/$tag.txt
      TORUS_LIB_PATH=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
        --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) tools/outliers.py 400 \
        2>/dev/null | grep '^{' >> gpurun_out/$tag.txt
    done
  done
done
cat gpurun_out/$tag.txt
