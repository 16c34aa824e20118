# Round-2 profiles (one GPU): launch lists of the bench commands, --set full captures of the
# dominant kernels, DRAM bytes + duration of the HBM-bound kernels (row d).  Outputs gpurun_out/ncu2.
set -u
O=gpurun_out/ncu2
mkdir -p $O
M="--clock-control none"
# (1) launch list of the headline bench command (one timed step) -- shares, not absolute times
timeout 1500 ncu --metrics gpu__time_duration.sum $M --csv --log-file $O/launches_c3_f0.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches_c3_f0.log 2>&1
# (2) --set full of representative launches: the TMA Schur DGEMM, the TRSMs, the persistent solve
timeout 900 ncu --set full $M --import-source on -k regex:"k_dgemm_tma" -s 40 -c 2 -o $O/full_dgemm_tma \
  python tools/prof_case.py 32768 256 0.0 1 > $O/full_dgemm_tma.log 2>&1
timeout 900 ncu --set full $M --import-source on -k regex:"k_trsm" -s 40 -c 2 -o $O/full_trsm \
  python tools/prof_case.py 32768 256 0.0 1 > $O/full_trsm.log 2>&1
timeout 900 ncu --set full $M --import-source on -k regex:"k_solve_rows" -c 2 -o $O/full_solve \
  python tools/prof_hbm.py 32768 256 lu > $O/full_solve.log 2>&1
# (3) HBM kernels: DRAM bytes and duration per launch (C3 and C2 sizes)
HB="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed"
for N in 32768 16384; do
  timeout 900 ncu --metrics $HB $M --csv -k regex:"k_panel_stats|k_tile_norm_max|k_colpart_max|k_final_scan|k_solve_rows|k_decide" \
    --log-file $O/hbm_crit_$N.csv python tools/prof_hbm.py $N 256 crit > $O/hbm_crit_$N.log 2>&1
  timeout 900 ncu --metrics $HB $M --csv -k regex:"k_colpart_max|k_solve_rows|k_final_scan" \
    --log-file $O/hbm_lu_$N.csv python tools/prof_hbm.py $N 256 lu > $O/hbm_lu_$N.log 2>&1
  timeout 900 ncu --metrics $HB $M --csv -k regex:"k_qr_apply_vec|k_solve_rows" \
    --log-file $O/hbm_qr_$N.csv python tools/prof_hbm.py $N 256 qr > $O/hbm_qr_$N.log 2>&1
done
