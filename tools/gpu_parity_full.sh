# Full-size parity records (tools/parity_full.py), four oracle processes in parallel on the box's
# host cores; outputs under gpurun_out/parity/.
set -u
O=gpurun_out/parity
mkdir -p $O
(nproc; free -g) > $O/host.txt
OPENBLAS_NUM_THREADS=8 HLQ_ORACLE_THREADS=4 timeout 9000 python tools/parity_full.py C3_f0 --out $O > $O/log_c3f0.txt 2>&1 &
OPENBLAS_NUM_THREADS=4 HLQ_ORACLE_THREADS=6 timeout 9000 python tools/parity_full.py C3_f1 --out $O > $O/log_c3f1.txt 2>&1 &
OPENBLAS_NUM_THREADS=4 HLQ_ORACLE_THREADS=6 timeout 9000 python tools/parity_full.py C5r --out $O > $O/log_c5r.txt 2>&1 &
OPENBLAS_NUM_THREADS=4 HLQ_ORACLE_THREADS=4 timeout 9000 python tools/parity_full.py C2_mumps4 C2_max1 C4A_max C4A_sum C4A_mumps C4B_max C4B_sum C4B_mumps C4C_max C4C_sum C4C_mumps --out $O > $O/log_small.txt 2>&1 &
wait
free -g >> $O/host.txt
