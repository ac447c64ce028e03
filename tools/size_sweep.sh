#!/bin/bash
# Size sweep of the multi-phase kernels (push vs pull) at N GPUs: fp16 mean, one bench
# line per (kernel, size).  Usage: tools/size_sweep.sh N TAG [sizes in elements...]
n=$1; tag=$2; shift 2
sizes=${@:-4194304 8388608 16777216 25557032 33554432 67108864}
for cnt in $sizes; do
  for k in push pull; do
    TORUS_KERNEL=$k TORUS_LL_MAX_BYTES=0 TORUS_LL2_MAX_BYTES=0 python tools/sweep_env.py $n "K=$k" -- --count $cnt --out gpurun_out/$tag.jsonl
  done
done
