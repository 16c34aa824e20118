# LU solve: parallel partial-flag waits + reciprocal back-substitution chain; suite subset + timings.
set -u
O=gpurun_out/r2q
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_fuzz.py -m gpu -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 $B > $O/c3f0.log 2>&1
HB="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
python tools/prof_hbm.py 32768 256 lu > $O/plain_hl.log 2>&1 && \
timeout 900 ncu --metrics $HB --clock-control none --csv -k regex:"k_solve_rows" --log-file $O/hbm_solve_32768.csv python tools/prof_hbm.py 32768 256 lu > $O/hbm_solve.log 2>&1
