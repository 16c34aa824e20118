# QR solve DAG (no prefetch) + LU solve one-ahead prefetch: suite + solve-class timings.
set -u
O=gpurun_out/r2n
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 $B > $O/c3f0.log 2>&1
timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4.log 2>&1
HLQ_QR_SOLVE_DAG=0 timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4_nosdag.log 2>&1
timeout 900 $B --fqr 1.0 > $O/c3f1_greedy.log 2>&1
timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr4 > $O/c2_hqr4.log 2>&1
HLQ_QR_SOLVE_DAG=0 timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr4 > $O/c2_hqr4_nosdag.log 2>&1
