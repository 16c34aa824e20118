# Lookahead column on the panel stream (HLQ_LA_SP) + pipelined diagonal solves: GPU suite, A/B lines.
set -u
O=gpurun_out/r2n
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
for la in 1 0; do
  export HLQ_LA_SP=$la
  timeout 900 $B > $O/c3f0_la$la.log 2>&1
  timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4_la$la.log 2>&1
  timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr4 > $O/c2_hqr4_la$la.log 2>&1
  timeout 900 $B --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --tree hqr4 > $O/c5r_hqr4_la$la.log 2>&1
  timeout 900 $B --fqr 0.5 > $O/c3f05_la$la.log 2>&1
done
unset HLQ_LA_SP
for G in 2 8 16; do
  HLQ_SOLVE_G=$G timeout 900 $B --steps 2 > $O/c3f0_solveG$G.log 2>&1
done
