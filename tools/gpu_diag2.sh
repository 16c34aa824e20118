set -u
O=gpurun_out/diag2
mkdir -p $O
timeout 900 python tools/parity_diag2.py 8192 320 2 > $O/c5r_8192.txt 2>&1
timeout 1500 python tools/parity_diag2.py 16384 320 2 > $O/c5r_16384.txt 2>&1
