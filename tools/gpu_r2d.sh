set -u
O=gpurun_out/r2d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "hqr or random or step_log" -p no:cacheprovider > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
timeout 900 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -k "block_cyclic" -p no:cacheprovider > $O/pytest_fuzzdist.log 2>&1; echo "rc=$?" >> $O/pytest_fuzzdist.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f0.log 2>&1
HLQ_DGEMM_TMA=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f0_notma.log 2>&1
timeout 600 python bench.py --fqr 1.0 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1.log 2>&1
timeout 600 python bench.py --fqr 1.0 --tree hqr4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1_hqr4.log 2>&1
timeout 600 python bench.py --fqr 1.0 --tree hqr8 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1_hqr8.log 2>&1
