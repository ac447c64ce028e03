#!/bin/bash
# One-GPU round-end style call: the GPU test suite, smoke, the default bench line, the
# ncu launch list of the same bench command, and one ncu --set full capture of the N=1
# kernel (castscale_tma_kernel) for the roofline traffic figure.
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > $O/r02_gpu_suite_n1.txt 2>&1; echo "== suite rc=$?"; tail -3 $O/r02_gpu_suite_n1.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/r02_smoke_n1.txt 2>&1; echo "== smoke rc=$?"; tail -2 $O/r02_smoke_n1.txt
python bench.py --steps 20 --warmup 5 > $O/r02_bench_n1.json 2> $O/r02_bench_n1.err; echo "== bench rc=$?"; tail -c 600 $O/r02_bench_n1.json
python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/r02_bench_n1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_n1.csv \
    python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > $O/r02_ncu_launches.log 2>&1; echo "== ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:castscale -s 5 -c 1 \
    -o $O/r02_prof_castscale_tma python bench.py --steps 10 --warmup 5 --no-cpu --no-e2e > $O/r02_ncu_cs.log 2>&1; echo "== ncu full rc=$?"
ls -la $O/*.ncu-rep
