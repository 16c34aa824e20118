# Bulk-fed QR-update ring + QR solve DAG: GPU suite, QR bench lines (hqr4/8/16), ncu of a big TSMQR.
set -u
O=gpurun_out/r2m
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4.log 2>&1
timeout 900 $B --fqr 1.0 --tree hqr8 > $O/c3f1_hqr8.log 2>&1
timeout 900 $B --fqr 1.0 --tree hqr16 > $O/c3f1_hqr16.log 2>&1
timeout 900 $B --fqr 1.0 > $O/c3f1_greedy.log 2>&1
timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr4 > $O/c2_hqr4.log 2>&1
timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr8 > $O/c2_hqr8.log 2>&1
timeout 900 $B --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --tree hqr4 > $O/c5r_hqr4.log 2>&1
timeout 900 $B --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --tree hqr8 > $O/c5r_hqr8.log 2>&1
python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/plain_pc.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tsmqr3" -s 1 -c 1 -o $O/full_tsmqr_big python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/full_tsmqr_big.log 2>&1
