# Last job of the round: ncu evidence at the final kernels (tools/gpu_ncu_r2b.sh), then C5 at full size.
set -u
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_variants_final.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_variants_final.log
bash tools/gpu_ncu_r2b.sh
O=gpurun_out/r2r
mkdir -p $O
timeout 1800 python bench.py --config C5 --criterion max --alpha 1 --domains 2 --tree hqr4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/c5_full_hqr4.log 2>&1
