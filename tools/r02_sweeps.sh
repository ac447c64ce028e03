#!/bin/bash
# Round-2 measurement protocol (one call, 4 GPUs): BASELINE.json configs[2] (grid sweep)
# and configs[3] (size sweep fp16/bf16/f32 at 2 and 4 GPUs vs NCCL), plus the 2x4 routing
# check at N = 4 (per-CTA slice equal to the 8-GPU 2x4 one).  All under the same bench /
# sweep protocol: CUDA events on the launching stream, max over ranks, L2 evicted.
O=gpurun_out
# --- 2x4 routing validated at N=4: D such that the 2x2 per-CTA slice is 2698 vectors ---
python tools/sweep_env.py 4 "ROUTE=auto" "TORUS_ONE_TILE_MAX=0" "TORUS_MID_TILES=2" "TORUS_TILE=900" "TORUS_TILE=600" -- --count 12778516 --grid 2x2 --out $O/r02_route2x4_at_n4.jsonl
# --- grid sweep at the north-star message (fp16, 51.1 MB), with NCCL ---
for g in 1x4 2x2 4x1; do
  tools/run_gpu.sh bench 4 r02_grid_$g --steps 100 --warmup 10 --no-cpu --no-e2e --grid $g
done
tools/run_gpu.sh bench 4 r02_grid_ring4 --steps 100 --warmup 10 --no-cpu --no-e2e --no-nccl --algo ring
tools/run_gpu.sh bench 4 r02_grid_hier2x2 --steps 100 --warmup 10 --no-cpu --no-e2e --no-nccl --algo hier --grid 2x2
# --- size sweeps, three wire types, 2 and 4 GPUs, torus vs ring vs NCCL ---
for dt in f16 bf16 f32; do
  for n in 4 2; do
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) \
      tools/sweep_sizes.py --dtype $dt --min-bytes 4096 --max-bytes $((256 << 20)) --impls torus,nccl > $O/r02_sizes_${dt}_n$n.jsonl 2> $O/r02_sizes_${dt}_n$n.err
    echo "== sizes $dt n=$n rc=$?"; tail -2 $O/r02_sizes_${dt}_n$n.jsonl
  done
done
