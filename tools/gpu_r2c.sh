set -u
O=gpurun_out/r2c
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=10 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f0.log 2>&1
HLQ_DGEMM_TMA=0 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f0_notma.log 2>&1
timeout 600 python bench.py --fqr 1.0 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1.log 2>&1
timeout 600 python bench.py --fqr 1.0 --tree hqr4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1_hqr4.log 2>&1
