# Final-state check: GPU suite, smoke, the default bench line (with e2e and the CPU baseline), QR-heavy lines.
set -u
O=gpurun_out/r2p
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench_default.log 2>&1
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4.log 2>&1
timeout 900 $B --fqr 1.0 --tree hqr8 > $O/c3f1_hqr8.log 2>&1
timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr4 > $O/c2_hqr4.log 2>&1
timeout 900 $B --config C5 --N 32768 --criterion max --alpha 1 --domains 2 --tree hqr4 > $O/c5r_hqr4.log 2>&1
timeout 900 $B --fqr 0.5 --tree hqr4 > $O/c3f05_hqr4.log 2>&1
