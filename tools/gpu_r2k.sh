# QR panel as one dependency-DAG launch + accumulator-interleaved QR update: GPU suite, A/B bench lines.
set -u
O=gpurun_out/r2k
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4_dag.log 2>&1
HLQ_QR_DAG=0 timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4_nodag.log 2>&1
HLQ_QR_REORD=1 timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4_dag_reord.log 2>&1
timeout 900 $B --fqr 1.0 --tree hqr8 > $O/c3f1_hqr8_dag.log 2>&1
timeout 900 $B --fqr 1.0 > $O/c3f1_greedy_dag.log 2>&1
timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr4 > $O/c2_hqr4_dag.log 2>&1
HLQ_QR_DAG=0 timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr4 > $O/c2_hqr4_nodag.log 2>&1
timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr8 > $O/c2_hqr8_dag.log 2>&1
timeout 900 $B --config C2 --criterion max --alpha 1 > $O/c2_greedy_dag.log 2>&1
timeout 900 $B --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --tree hqr4 > $O/c5r_hqr4_dag.log 2>&1
timeout 900 $B --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --tree hqr8 > $O/c5r_hqr8_dag.log 2>&1
