# Round end: the GPU suite, smoke and the default bench line at HEAD.
set -u
O=gpurun_out/r2t
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench_default.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.log 2>&1
