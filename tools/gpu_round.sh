#!/bin/bash
# Round measurement batch (run on the GPU box from the repo root): tests, smoke, bench lines,
# ncu launch list and full captures.  Outputs under gpurun_out/r/.
set -u
O=gpurun_out/r
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_c3_f0.log 2>&1
timeout 600 python bench.py --fqr 1.0 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_c3_f1.log 2>&1
timeout 600 python bench.py --fqr 0.5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c3_f05.log 2>&1
timeout 600 python bench.py --dist --steps 3 --warmup 3 --no-e2e > $O/bench_dist_c3.log 2>&1
timeout 900 python bench.py --config C5 --N 32768 --criterion max --alpha 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c5r.log 2>&1
timeout 900 python bench.py --config C2 --criterion max --alpha 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c2_max1.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.log 2>&1
timeout 900 python bench.py --config C2 --criterion max --alpha 1 --lu-variant A2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c2_max1_a2.log 2>&1
timeout 900 python bench.py --lu-variant A2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f0_a2.log 2>&1
timeout 900 python bench.py --fqr 1.0 --lu-variant A2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c3_f1_a2.log 2>&1
