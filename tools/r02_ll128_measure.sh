#!/bin/bash
# LL128-default measurement call (4 GPUs): ncu NVLink/DRAM bytes of torus_ll128_kernel on
# rank 0 at 1x2 and 2x2, bench lines at N=2 and N=4, the grid sweep at N=4, fp16 size sweeps.
O=gpurun_out
tools/ncu_rank0.sh 2 1 2 torus_ll128_kernel r02_ncu_ll128_1x2 2>&1 | tail -3
tools/ncu_rank0.sh 4 2 2 torus_ll128_kernel r02_ncu_ll128_2x2 2>&1 | tail -3
tools/run_gpu.sh bench 2 r02_ll128_bench_n2 --steps 200 --warmup 20
tools/run_gpu.sh bench 4 r02_ll128_bench_n4 --steps 200 --warmup 20
for g in 1x4 4x1; do tools/run_gpu.sh bench 4 r02_ll128_grid_$g --steps 100 --warmup 10 --no-cpu --no-e2e --grid $g; done
for n in 4 2; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29650 + n)) \
    tools/sweep_sizes.py --dtype f16 --min-bytes 4096 --max-bytes $((256 << 20)) --impls torus,nccl > $O/r02_ll128_sizes_f16_n$n.jsonl 2> $O/r02_ll128_sizes_f16_n$n.err
  echo "== sizes n=$n rc=$?"
done
