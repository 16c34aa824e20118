# Round-2 session-2 evidence run: full-size parity of the QR-heavy configs (oracle on the host
# cores, in the background) beside ncu captures of the dominant kernels and the HBM-bound ones.
set -u
O=gpurun_out/r2h
P=gpurun_out/parity2
mkdir -p $O $P
(nproc; free -g) > $P/host.txt
cp profiles/r02/parity/C5r.json profiles/r02/parity/C2_max1.json $P/  # decision vectors for the parallel floor runs
OPENBLAS_NUM_THREADS=4 HLQ_ORACLE_THREADS=4 timeout 4200 python tools/parity_full.py C3_f1 --floor-parallel --out $P > $P/log_c3f1.txt 2>&1 &
OPENBLAS_NUM_THREADS=4 HLQ_ORACLE_THREADS=4 timeout 4200 python tools/parity_full.py C5r C2_max1 --floor-parallel --out $P > $P/log_c5r.txt 2>&1 &
M="--clock-control none"
B0="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$B0 > $O/plain_b0.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum $M --csv --log-file $O/launches_c3_f0.csv \
  $B0 > $O/launches_c3_f0.log 2>&1
python tools/prof_case.py 32768 256 0.0 1 > $O/plain_pc0.log 2>&1 && timeout 900 ncu --set full $M --import-source on -k regex:"k_dgemm_tma" -s 40 -c 2 -o $O/full_dgemm_tma \
  python tools/prof_case.py 32768 256 0.0 1 > $O/full_dgemm_tma.log 2>&1
python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/plain_pc1.log 2>&1 && timeout 900 ncu --set full $M --import-source on -k regex:"k_tsmqr3|k_unmqr3|k_ttmqr3" -s 12 -c 6 -o $O/full_qrupd_hqr4 \
  python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/full_qrupd_hqr4.log 2>&1
timeout 900 ncu --set full $M --import-source on -k regex:"k_tsqrt_tc|k_geqrt_tc|k_ttqrt_tc" -s 12 -c 6 -o $O/full_qrpanel_hqr4 \
  python tools/prof_case.py 16384 256 1.0 1 hqr4 > $O/full_qrpanel_hqr4.log 2>&1
B1="python bench.py --fqr 1.0 --tree hqr4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$B1 > $O/plain_b1.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum $M --csv --log-file $O/launches_c3_f1_hqr4.csv \
  $B1 > $O/launches_c3_f1_hqr4.log 2>&1
HB="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed"
for N in 32768 16384; do
  python tools/prof_hbm.py $N 256 crit > $O/plain_hc$N.log 2>&1 && python tools/prof_hbm.py $N 256 lu > $O/plain_hl$N.log 2>&1 && python tools/prof_hbm.py $N 256 qr > $O/plain_hq$N.log 2>&1
  timeout 900 ncu --metrics $HB $M --csv -k regex:"k_panel_stats|k_tile_norm_max|k_colpart_max|k_final_scan|k_solve_rows|k_decide" \
    --log-file $O/hbm_crit_$N.csv python tools/prof_hbm.py $N 256 crit > $O/hbm_crit_$N.log 2>&1
  timeout 900 ncu --metrics $HB $M --csv -k regex:"k_colpart_max|k_solve_rows|k_final_scan" \
    --log-file $O/hbm_lu_$N.csv python tools/prof_hbm.py $N 256 lu > $O/hbm_lu_$N.log 2>&1
  timeout 900 ncu --metrics $HB $M --csv -k regex:"k_qr_apply_vec|k_solve_rows" \
    --log-file $O/hbm_qr_$N.csv python tools/prof_hbm.py $N 256 qr > $O/hbm_qr_$N.log 2>&1
done
wait
