# Verification + evidence: GPU suite, ncu of the new kernels, C5 at full size (hqr4 + panel DAG).
set -u
O=gpurun_out/r2o
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
M="--clock-control none"
B1="python bench.py --fqr 1.0 --tree hqr4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$B1 > $O/plain_b1.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum $M --csv --log-file $O/launches_c3_f1_hqr4.csv $B1 > $O/launches_c3_f1_hqr4.log 2>&1
python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/plain_pc.log 2>&1 && \
timeout 900 ncu --set full $M --import-source on -k regex:"k_qr_panel_dag" -s 3 -c 1 -o $O/full_panel_dag python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/full_panel_dag.log 2>&1
python tools/prof_case.py 32768 256 0.0 1 > $O/plain_pc0.log 2>&1 && \
timeout 900 ncu --set full $M --import-source on -k regex:"k_dgemm_tma" -s 40 -c 2 -o $O/full_dgemm_tma8 python tools/prof_case.py 32768 256 0.0 1 > $O/full_dgemm_tma8.log 2>&1
timeout 2400 python bench.py --config C5 --criterion max --alpha 1 --domains 2 --tree hqr4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c5_full_hqr4.log 2>&1
