#!/bin/bash
# Routing thresholds with the LL128 kernel as the multi-phase route: one-shot (N=2) and
# two-shot (N=4) LL kernels vs LL128 at 1-16 MB, plus the grid sweep at N=4.
for cnt in 524288 1048576 2097152 3145728 4194304 8388608; do
  python tools/sweep_env.py 4 "TORUS_LL_MAX_BYTES=0 TORUS_LL2_MAX_BYTES=0" "TORUS_LL_MAX_BYTES=0 TORUS_LL2_MAX_BYTES=33554432" "TORUS_LL2_MAX_BYTES=0" -- --count $cnt --steps 100 --out gpurun_out/r02_thr_n4.jsonl
done
for cnt in 524288 1048576 2097152 3145728 4194304; do
  python tools/sweep_env.py 2 "TORUS_LL_MAX_BYTES=0" "TORUS_LL_MAX_BYTES=33554432" -- --count $cnt --steps 100 --out gpurun_out/r02_thr_n2.jsonl
done
for g in 1x4 2x2 4x1; do python tools/sweep_env.py 4 "G=$g" -- --grid $g --steps 200; done
