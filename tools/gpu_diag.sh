set -u
O=gpurun_out/diag
mkdir -p $O
timeout 900 python tools/parity_diag.py 8192 256 > $O/diag_8192.txt 2>&1
timeout 1500 python tools/parity_diag.py 16384 256 > $O/diag_16384.txt 2>&1
