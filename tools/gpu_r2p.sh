# TMA-fed QR-update ring: GPU suite + A/B bench lines + ncu of a big TSMQR launch.
set -u
O=gpurun_out/r2p
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4.log 2>&1
HLQ_QR_TMA=0 timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4_notma.log 2>&1
timeout 900 $B --fqr 1.0 --tree hqr8 > $O/c3f1_hqr8.log 2>&1
timeout 900 $B --fqr 1.0 > $O/c3f1_greedy.log 2>&1
timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr4 > $O/c2_hqr4.log 2>&1
timeout 900 $B --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --tree hqr4 > $O/c5r_hqr4.log 2>&1
python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/plain_pc.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tsmqr3" -s 1 -c 1 -o $O/full_tsmqr_tma python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/full_tsmqr_tma.log 2>&1
