# QR panel / QR-update producer changes: full GPU suite, QR-heavy bench lines, ncu of BIG update
# launches and the panel kernels; C5-recipe V-divergence diagnostic at N = 8192.
set -u
O=gpurun_out/r2j
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --fqr 1.0 --tree hqr4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1_hqr4.log 2>&1
timeout 900 python bench.py --fqr 1.0 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1.log 2>&1
timeout 900 python bench.py --config C2 --criterion max --alpha 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c2_max1.log 2>&1
timeout 900 python bench.py --config C2 --criterion max --alpha 1 --tree hqr4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c2_max1_hqr4.log 2>&1
timeout 900 python bench.py --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --tree hqr4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c5r_hqr4.log 2>&1
M="--clock-control none"
python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/plain_pc.log 2>&1 && \
timeout 900 ncu --set full $M --import-source on -k regex:"k_tsmqr3" -s 1 -c 1 -o $O/full_tsmqr_big python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/full_tsmqr_big.log 2>&1
timeout 900 ncu --set full $M --import-source on -k regex:"k_unmqr3" -s 1 -c 1 -o $O/full_unmqr_big python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/full_unmqr_big.log 2>&1
python tools/prof_case.py 16384 256 1.0 1 > $O/plain_pcg.log 2>&1 && \
timeout 900 ncu --set full $M --import-source on -k regex:"k_ttmqr3" -s 1 -c 1 -o $O/full_ttmqr_big python tools/prof_case.py 16384 256 1.0 1 > $O/full_ttmqr_big.log 2>&1
timeout 900 ncu --set full $M --import-source on -k regex:"k_ttqrt_tc|k_geqrt_tc" -s 2 -c 2 -o $O/full_panel python tools/prof_case.py 16384 256 1.0 1 > $O/full_panel.log 2>&1
timeout 900 python tools/parity_diag2.py 8192 320 2 > $O/c5r_diag_8192.txt 2>&1
