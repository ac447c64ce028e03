#!/bin/bash
# N = 1 validation + profile of the shipped cast kernel (run under gpurun, one GPU):
# parity tests of the N = 1 path, smoke, two bench lines, then ONE ncu --set full capture
# of castscale_kernel on the same bench command line.  Outputs in gpurun_out/.
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x -k "single_rank or multi_tensor_single" > $O/r02_n1_tests.txt 2>&1
echo "tests rc=$?"; tail -1 $O/r02_n1_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/r02_n1_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/r02_n1_smoke.txt
for i in 1 2; do python bench.py --steps 100 --warmup 5 > $O/r02_n1_bench_$i.json 2> $O/r02_n1_bench_$i.err; echo "bench rc=$?"; done
python bench.py --steps 10 --warmup 5 --no-cpu --no-e2e > $O/r02_n1_bench_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:castscale_kernel -s 5 -c 1 \
    -o $O/r02_prof_castscale python bench.py --steps 10 --warmup 5 --no-cpu --no-e2e > $O/r02_ncu_cs.log 2>&1
echo "ncu rc=$?"; ls $O/r02_prof_castscale* 2>/dev/null
