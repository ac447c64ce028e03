#!/bin/bash
# One-GPU profiling pass (run under gpurun): plain runs first, then ncu on the same
# command lines (B200_PROFILING.md).  Outputs land in gpurun_out/.
set -x
O=gpurun_out
python bench.py --steps 100 --warmup 10 > $O/bench_n1.json 2> $O/bench_n1.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_n1.csv \
    python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1
python tools/profile_virtual.py > $O/profile_virtual.json 2> $O/profile_virtual.err && \
ncu --set full --clock-control none --import-source on -k regex:torus_kernel -s 1 -c 1 \
    -o $O/prof_torus_virtual2x4 python tools/profile_virtual.py --calls 2 > $O/ncu_torus.log 2>&1
python bench.py --steps 10 --warmup 5 --no-cpu --no-e2e > $O/bench_cs_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:castscale -s 5 -c 1 \
    -o $O/prof_castscale python bench.py --steps 10 --warmup 5 --no-cpu --no-e2e > $O/ncu_cs.log 2>&1
ls -la $O
