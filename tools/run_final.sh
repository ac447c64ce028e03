#!/bin/bash
# round-end evidence: full GPU suite, smoke, bench lines at N = 1, 2, 4 (+ reference arm)
O=gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > $O/final_gpu_tests.txt 2>&1
echo "rc=$?" >> $O/final_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/final_smoke.txt 2>&1
timeout 300 python bench.py > $O/final_bench_n1.log 2>&1
timeout 300 python bench.py --impl reference > $O/final_bench_ref_n1.log 2>&1
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
timeout 300 $P 2 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 2 > $O/final_bench_n2.log 2>&1
timeout 300 $P 4 --master-addr 127.0.0.1 --master-port 29662 bench.py --gpus 4 > $O/final_bench_n4.log 2>&1
