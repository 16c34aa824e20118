# Solve flags on their own lines + T zeroing + DAG default: GPU suite, headline, QR lines, solve HBM.
set -u
O=gpurun_out/r2l
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.log 2>&1
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4.log 2>&1
timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr4 > $O/c2_hqr4.log 2>&1
HB="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed"
python tools/prof_hbm.py 32768 256 lu > $O/plain_hl.log 2>&1 && \
timeout 900 ncu --metrics $HB --clock-control none --csv -k regex:"k_solve_rows" --log-file $O/hbm_solve_32768.csv python tools/prof_hbm.py 32768 256 lu > $O/hbm_solve.log 2>&1
