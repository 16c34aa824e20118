# After the last refactor (no behaviour change): parity + variants subset, smoke, one short bench line.
set -u
O=gpurun_out/r2u
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_abi.py -m gpu -q -p no:cacheprovider > $O/pytest_sub.log 2>&1; echo "rc=$?" >> $O/pytest_sub.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3f0.log 2>&1
