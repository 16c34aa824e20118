set -u
O=gpurun_out/r2b
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f0.log 2>&1
