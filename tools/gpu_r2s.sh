# V-noise curves: the growth of a rounding-level perturbation through the steps of an all-QR run,
# oracle variants vs the GPU (128 steps, like C3).
set -u
O=gpurun_out/r2s
mkdir -p $O
export HLQ_ORACLE_THREADS=5 OPENBLAS_NUM_THREADS=2
timeout 900 python tools/vnoise_curve.py 8192 64 hqr4 --out $O/vnoise_8192_64_hqr4.json > $O/vnoise_8192_64_hqr4.log 2>&1
timeout 900 python tools/vnoise_curve.py 8192 64 greedy --out $O/vnoise_8192_64_greedy.json > $O/vnoise_8192_64_greedy.log 2>&1
timeout 2400 python tools/vnoise_curve.py 16384 128 hqr4 --out $O/vnoise_16384_128_hqr4.json > $O/vnoise_16384_128_hqr4.log 2>&1
