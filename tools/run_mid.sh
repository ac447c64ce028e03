#!/bin/bash
# mid-size (512 KB - 8 MB): one-shot forced vs multi-phase at several CTA counts vs NCCL
O=gpurun_out
P="python -m torch.distributed.run --nnodes=1 --nproc-per-node"
timeout 400 $P 4 --master-addr 127.0.0.1 --master-port 29641 tools/sweep_sizes.py --grid 2x2 --min-bytes 524288 --max-bytes 8388608 --ll-max 4194304 --impls torus_ll,torus_mp,torus_mpc64,torus_mpc32,torus_mpc16,nccl > $O/mid_n4_2x2.jsonl 2>&1
timeout 400 $P 4 --master-addr 127.0.0.1 --master-port 29642 tools/sweep_sizes.py --grid 4x1 --min-bytes 524288 --max-bytes 8388608 --ll-max 4194304 --impls torus_ll,torus_mp,torus_mpc64,torus_mpc32,nccl > $O/mid_n4_4x1.jsonl 2>&1
timeout 400 $P 2 --master-addr 127.0.0.1 --master-port 29643 tools/sweep_sizes.py --grid 1x2 --min-bytes 524288 --max-bytes 8388608 --ll-max 8388608 --impls torus_ll,torus_mp,torus_mpc64,torus_mpc32,nccl > $O/mid_n2.jsonl 2>&1
