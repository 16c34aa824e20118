# Round-2 profiles of the final kernels (one GPU): launch list of the headline bench command, DRAM
# bytes + duration of the solve kernels (row d), --set full of the two solve kernels.  gpurun_out/ncu3.
set -u
O=gpurun_out/ncu3
mkdir -p $O
M="--clock-control none"
timeout 1500 ncu --metrics gpu__time_duration.sum $M --csv --log-file $O/launches_c3_f0.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches_c3_f0.log 2>&1
HB="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed"
for N in 32768 16384; do
  timeout 900 ncu --metrics $HB $M --csv -k regex:"k_colpart_max|k_solve_rows|k_final_scan" \
    --log-file $O/hbm_lu_$N.csv python tools/prof_hbm.py $N 256 lu > $O/hbm_lu_$N.log 2>&1
  timeout 900 ncu --metrics $HB $M --csv -k regex:"k_qr_solve_dag|k_qr_apply_vec|k_solve_rows" \
    --log-file $O/hbm_qr_$N.csv python tools/prof_hbm.py $N 256 qr hqr4 > $O/hbm_qr_$N.log 2>&1
done
timeout 900 ncu --set full $M --import-source on -k regex:"k_solve_rows" -c 2 -o $O/full_solve \
  python tools/prof_hbm.py 32768 256 lu > $O/full_solve.log 2>&1
timeout 900 ncu --set full $M --import-source on -k regex:"k_qr_solve_dag" -c 1 -o $O/full_qr_solve \
  python tools/prof_hbm.py 16384 256 qr hqr4 > $O/full_qr_solve.log 2>&1
python tools/hbm_summary.py $O/hbm_*.csv > $O/hbm_kernels.txt 2>&1
python tools/launch_summary.py $O/launches_c3_f0.csv > $O/launches_c3_f0_summary.txt 2>&1
gzip -f $O/launches_c3_f0.csv
