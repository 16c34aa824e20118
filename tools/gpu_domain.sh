#!/bin/bash
# NEXT f1 measurements: diagonal-domain vs tile pivoting on C2 (N=16384, normal seed 1), D=2, and
# the all-LU C3 pattern with domain pivoting (tall-panel GETRF at scale).  Outputs gpurun_out/d/.
set -u
O=gpurun_out/d
mkdir -p $O
for a in 1 3e4; do
  for ps in tile domain; do
    timeout 900 python bench.py --config C2 --criterion max --alpha $a --domains 2 --pivot-scope $ps \
      --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/c2_max${a}_${ps}.log 2>&1
  done
done
timeout 900 python bench.py --pivot-scope domain --domains 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/c3_f0_domain.log 2>&1
timeout 900 python bench.py --pivot-scope domain --domains 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/c3_f0_lupp.log 2>&1
