# Full-size parity records at the final kernels (tools/parity_full.py), five oracle processes in
# parallel on the box's host cores; outputs under gpurun_out/parity2/.
set -u
O=gpurun_out/parity2
mkdir -p $O
(nproc; free -g) > $O/host.txt
T=3400
OPENBLAS_NUM_THREADS=4 HLQ_ORACLE_THREADS=4 timeout $T python tools/parity_full.py C3_f0 --floor-parallel --out $O > $O/log_c3f0.txt 2>&1 &
OPENBLAS_NUM_THREADS=3 HLQ_ORACLE_THREADS=4 timeout $T python tools/parity_full.py C3_f1 --floor-parallel --out $O > $O/log_c3f1.txt 2>&1 &
OPENBLAS_NUM_THREADS=3 HLQ_ORACLE_THREADS=4 timeout $T python tools/parity_full.py C3_f1@hqr4 --floor-parallel --out $O > $O/log_c3f1_hqr4.txt 2>&1 &
OPENBLAS_NUM_THREADS=3 HLQ_ORACLE_THREADS=4 timeout $T python tools/parity_full.py C5r@hqr4 --out $O > $O/log_c5r_hqr4.txt 2>&1 &
OPENBLAS_NUM_THREADS=3 HLQ_ORACLE_THREADS=3 timeout $T python tools/parity_full.py C2_max1 C2_max1@hqr4 C2_mumps4 C4A_max C4A_sum C4A_mumps C4B_max C4B_sum C4B_mumps C4C_max C4C_sum C4C_mumps --out $O > $O/log_small.txt 2>&1 &
wait
free -g >> $O/host.txt
