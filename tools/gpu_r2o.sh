# Solve timings: the DAG op body (latency-pipelined vs the step-by-step kernels' body), LU solve.
set -u
O=gpurun_out/r2o
mkdir -p $O
for body in 1 0; do
  export HLQ_QR_SOLVE_DAG_BODY=$body
  timeout 600 python tools/solve_times.py C2 16384 256 max hqr4 >> $O/solve_times.txt 2>&1
  timeout 600 python tools/solve_times.py C3 32768 256 1.0 hqr4 >> $O/solve_times.txt 2>&1
  timeout 600 python tools/solve_times.py C3 32768 256 1.0 greedy >> $O/solve_times.txt 2>&1
  timeout 600 python tools/solve_times.py C5 32768 320 max hqr4 >> $O/solve_times.txt 2>&1
done
unset HLQ_QR_SOLVE_DAG_BODY
timeout 600 python tools/solve_times.py C3 32768 256 0.0 >> $O/solve_times.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > $O/pytest_sub.log 2>&1; echo "rc=$?" >> $O/pytest_sub.log
