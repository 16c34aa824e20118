# Narrow QR-update shape for the lookahead column (HLQ_QR_NARROW): parity subset with it on, A/B lines.
set -u
O=gpurun_out/r2q
mkdir -p $O
HLQ_QR_NARROW=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_variants.py -m gpu -q -x -p no:cacheprovider > $O/pytest_narrow.log 2>&1; echo "rc=$?" >> $O/pytest_narrow.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for nv in 1 0; do
  export HLQ_QR_NARROW=$nv
  timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr4 > $O/c2_hqr4_n$nv.log 2>&1
  timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4_n$nv.log 2>&1
  timeout 900 $B --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --tree hqr4 > $O/c5r_hqr4_n$nv.log 2>&1
  timeout 900 $B --config C2 --criterion max --alpha 1 > $O/c2_greedy_n$nv.log 2>&1
done
