#!/bin/bash
# ncu on rank 0 of an N-GPU run (the other ranks plain): single-pass metrics of the
# multi-phase kernel -- duration, DRAM bytes, NVLink tx/rx bytes (user data and total).
# Application replay: every ncu pass reruns rank 0 as a new session the peers serve, so
# no pass replays a kernel whose peers have already finished.
#   tools/ncu_rank0.sh N X Y KERNEL_REGEX TAG [count]
# env TORUS_KERNEL etc. pass through.  Output: gpurun_out/TAG.csv (+ TAG.log)
set -u
n=$1; X=$2; Y=$3; kre=$4; tag=$5; count=${6:-25557032}
d=$(mktemp -d /tmp/ncu_sess.XXXX)
export TORUS_TIMEOUT_MS=${TORUS_TIMEOUT_MS:-5000}
for r in $(seq 1 $((n - 1))); do
  python tools/ncu_worker.py $r $n $X $Y $d $count 3 > gpurun_out/$tag.rank$r.log 2>&1 &
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes_data_protocol.sum
ncu --metrics $M --clock-control none --replay-mode application -k "regex:$kre" -s 3 -c 1 --csv --log-file gpurun_out/$tag.csv \
    python tools/ncu_worker.py 0 $n $X $Y $d $count 3 > gpurun_out/$tag.log 2>&1
echo "ncu rc=$?"
wait
tail -5 gpurun_out/$tag.log; cat gpurun_out/$tag.csv | tail -20
