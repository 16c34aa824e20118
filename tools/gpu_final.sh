#!/bin/bash
# End-of-session batch: round measurements, NEXT-row measurements, launch lists, QR-update capture.
set -u
bash tools/gpu_round.sh
bash tools/gpu_domain.sh
O=gpurun_out/r
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $O/ncu_plain_c3f0.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_f0.csv $CMD > $O/ncu_launch.log 2>&1
CMD2="python bench.py --fqr 1.0 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD2 > $O/ncu_plain_c3f1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_f1.csv $CMD2 > $O/ncu_launch1.log 2>&1
O2=gpurun_out/r2
mkdir -p $O2
C2="python tools/prof_case.py 32768 256 1.0 1"
$C2 > $O2/plain_qr.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_qr_update3" -s 200 -c 4 -o $O2/c3_qr $C2 > $O2/ncu_qr.log 2>&1
