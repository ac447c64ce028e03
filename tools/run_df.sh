#!/bin/bash
# dataflow scheduler: parity on one GPU, then 2x2 / 1x2 bench vs lockstep over tile counts
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "df" > $O/df_parity.txt 2>&1
echo "rc=$?" >> $O/df_parity.txt
grep -q "rc=0" $O/df_parity.txt || exit 1
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
for SC in lockstep df; do
  for AT in 3 4 6 8 12; do
    [ $SC = lockstep ] && [ $AT -gt 4 ] && continue
    TORUS_SCHED=$SC TORUS_AUTO_TILES=$AT timeout 300 $P 4 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py --gpus 4 --no-e2e --no-nccl --no-cpu --steps 200 > $O/df_${SC}_t${AT}_n4.log 2>&1
    TORUS_SCHED=$SC TORUS_AUTO_TILES=$AT timeout 300 $P 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 300)) bench.py --gpus 2 --no-e2e --no-nccl --no-cpu --steps 200 > $O/df_${SC}_t${AT}_n2.log 2>&1
  done
done
