#!/bin/bash
# 32-byte-lane LL128 check (4 GPUs): GPU suite with TORUS_LL128_LANE=32 and with the
# default, the LL128-vs-push stress with 32-byte lanes, then 16- vs 32-byte lanes (and the
# previous build) interleaved on the bench at N=2 and N=4.
O=gpurun_out; P=$PWD/paper_1811_05233_b200
TORUS_LL128_LANE=32 timeout 900 python -m pytest tests -m gpu -q -x > $O/r02_lane32_suite.txt 2>&1; echo "suite32 rc=$?"; tail -1 $O/r02_lane32_suite.txt
timeout 900 python -m pytest tests -m gpu -q -x > $O/r02_lane16_suite.txt 2>&1; echo "suite16 rc=$?"; tail -1 $O/r02_lane16_suite.txt
TORUS_LL128_LANE=32 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29633 tools/ll128_stress.py 600 2>/dev/null | grep "^{" | tee $O/r02_lane32_stress_n4.json
for n in 2 4; do
  V="TORUS_LIB_PATH=$P/libtorus_base.so TORUS_LL128_LANE=16|TORUS_LL128_LANE=16|TORUS_LL128_LANE=32"
  IFS='|' read -ra A <<< "$V"
  python tools/sweep_env.py $n "${A[@]}" "${A[@]}" "${A[@]}" > $O/r02_lane_ab_n$n.txt 2>&1
  cut -c1-100 $O/r02_lane_ab_n$n.txt
done
