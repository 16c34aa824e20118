set -u
O=gpurun_out/tma5
mkdir -p $O
timeout 600 python tools/tma_check2.py > $O/tma_schur.txt 2>&1
timeout 600 python tools/tma_check3.py > $O/tma_pattern.txt 2>&1
timeout 600 python tools/tma_check.py 8192 256 > $O/tma_8192.txt 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f0.log 2>&1
