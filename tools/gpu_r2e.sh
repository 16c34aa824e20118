set -u
O=gpurun_out/r2e
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=10 -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
bash tools/gpu_ncu_r2.sh
