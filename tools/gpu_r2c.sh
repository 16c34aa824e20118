# background: full-size parity of the QR-heavy runs with the QR-aware noise floor (CPU oracles);
# foreground: GPU tests and benches of the round's new kernels
set -u
O=gpurun_out/r2c
P=gpurun_out/parity2
mkdir -p $O $P
cp profiles/r02/parity/*.json $P/ 2>/dev/null
OPENBLAS_NUM_THREADS=4 HLQ_ORACLE_THREADS=4 timeout 3300 python tools/parity_full.py C3_f1 --floor-parallel --out $P > $P/log_c3f1.txt 2>&1 &
OPENBLAS_NUM_THREADS=4 HLQ_ORACLE_THREADS=4 timeout 3300 python tools/parity_full.py C5r --floor-parallel --out $P > $P/log_c5r.txt 2>&1 &
OPENBLAS_NUM_THREADS=2 HLQ_ORACLE_THREADS=2 timeout 3300 python tools/parity_full.py C2_max1 C4A_max C4A_sum C4B_max C4B_sum C4B_mumps C4C_max C4C_sum C4C_mumps --floor-parallel --out $P > $P/log_small.txt 2>&1 &
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=10 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f0.log 2>&1
HLQ_DGEMM_TMA=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f0_notma.log 2>&1
timeout 600 python bench.py --fqr 1.0 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1.log 2>&1
timeout 600 python bench.py --fqr 1.0 --tree hqr4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1_hqr4.log 2>&1
wait
