#!/bin/bash
# ncu evidence for the round (1 GPU; each ncu command preceded by the same command without ncu)
set -u
O=gpurun_out/r
mkdir -p $O
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > $O/ncu_plain_c3f0.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_f0.csv $CMD > $O/ncu_launch.log 2>&1
CMD2="python bench.py --fqr 1.0 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD2 > $O/ncu_plain_c3f1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3_f1.csv $CMD2 > $O/ncu_launch1.log 2>&1
CMD3="python tools/prof_case.py 16384 256 0.0 1"
$CMD3 > $O/ncu_plain_lu.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_dgemm" -s 40 -c 3 -o $O/full_lu $CMD3 > $O/ncu_full_lu.log 2>&1
CMD4="python tools/prof_case.py 16384 256 1.0 1"
$CMD4 > $O/ncu_plain_qr.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_qr_update3|k_geqrt_tc|k_ttqrt_tc" -s 40 -c 6 -o $O/full_qr $CMD4 > $O/ncu_full_qr.log 2>&1
