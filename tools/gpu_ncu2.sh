#!/bin/bash
# representative single launches of the dominant kernels at the bench configuration (C3, N=32768)
set -u
O=gpurun_out/r2
mkdir -p $O
C1="python tools/prof_case.py 32768 256 0.0 1"
$C1 > $O/plain_lu.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_dgemm" -s 60 -c 2 -o $O/c3_lu $C1 > $O/ncu_lu.log 2>&1
C2="python tools/prof_case.py 32768 256 1.0 1"
$C2 > $O/plain_qr.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_qr_update3" -s 200 -c 4 -o $O/c3_qr $C2 > $O/ncu_qr.log 2>&1
