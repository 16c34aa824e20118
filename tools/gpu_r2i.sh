# Grid domain pivoting + variant tests; cuBLAS vs library Schur update on the C3 step-1 shape.
set -u
O=gpurun_out/r2i
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_multiproc.py tests/test_gpu_variants.py -m gpu -q -p no:cacheprovider > $O/pytest_dist_var.log 2>&1; echo "rc=$?" >> $O/pytest_dist_var.log
timeout 300 python tools/cublas_rank_update.py > $O/cublas_rank_update.jsonl 2>&1
timeout 300 python tools/schur_bench.py > $O/schur_bench.jsonl 2>&1
HLQ_TMA_CONS=8 timeout 300 python tools/schur_bench.py > $O/schur_bench_cons8.jsonl 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_cons4.log 2>&1
HLQ_TMA_CONS=8 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_cons8.log 2>&1
HLQ_TMA_CONS=8 HLQ_TMA_TPC=8 timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_cons8_tpc8.log 2>&1
