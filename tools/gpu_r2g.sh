# Round-2 session-2 status run: smoke, full GPU suite, bench lines (headline + QR-heavy + trees).
set -u
O=gpurun_out/r2g
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench_default.log 2>&1
timeout 900 python bench.py --fqr 1.0 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1.log 2>&1
timeout 900 python bench.py --fqr 1.0 --tree hqr4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1_hqr4.log 2>&1
timeout 900 python bench.py --config C2 --criterion max --alpha 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c2_max1.log 2>&1
timeout 900 python bench.py --config C2 --criterion max --alpha 1 --tree hqr4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c2_max1_hqr4.log 2>&1
timeout 900 python bench.py --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --tree hqr4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c5r_hqr4.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
