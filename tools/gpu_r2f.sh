set -u
O=gpurun_out/r2f
mkdir -p $O
timeout 600 python tools/tma_check2.py > $O/tma_schur.txt 2>&1
timeout 600 python tools/tma_check3.py > $O/tma_pattern.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "hqr or c1_max or forced" -p no:cacheprovider > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f0.log 2>&1
timeout 900 python bench.py --config C2 --criterion max --alpha 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c2_max1.log 2>&1
timeout 900 python bench.py --config C2 --criterion max --alpha 1 --tree hqr4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c2_max1_hqr4.log 2>&1
timeout 900 python bench.py --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c5r.log 2>&1
timeout 900 python bench.py --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --tree hqr4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c5r_hqr4.log 2>&1
