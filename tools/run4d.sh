#!/bin/bash
O=gpurun_out
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
for V in 512 256; do
  L=$PWD/paper_1811_05233_b200/libtorus.so; [ $V = 256 ] && L=$PWD/paper_1811_05233_b200/libtorus_t256.so
  TORUS_LIB_PATH=$L timeout 300 $P --master-port $((29650 + V % 97)) bench.py --gpus 4 --steps 200 --no-e2e > $O/e4_${V}_2x2.log 2>&1
  TORUS_LIB_PATH=$L timeout 300 $P --master-port $((29660 + V % 97)) bench.py --gpus 4 --steps 200 --no-e2e --grid 4x1 > $O/e4_${V}_4x1.log 2>&1
done
TORUS_LIB_PATH=$PWD/paper_1811_05233_b200/libtorus_t256.so timeout 600 python -m pytest tests/test_gpu_multiproc.py -x -q -k four > $O/pytest_t256.log 2>&1; echo rc=$? >> $O/pytest_t256.log
