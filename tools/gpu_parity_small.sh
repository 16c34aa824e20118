set -u
mkdir -p gpurun_out/parity_small
timeout 900 python tools/parity_full.py small_C3_f0 small_C3_f1 small_C5r small_C2_max1 small_C2_mumps4 C4A_mumps C4C_max --out gpurun_out/parity_small > gpurun_out/parity_small/log.txt 2>&1; echo "rc=$?" >> gpurun_out/parity_small/log.txt
