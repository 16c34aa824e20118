cd $GRAFT_REPO_ROOT
python tools/prof_case.py 8192 256 1.0 1 > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k regex:k_ttqrt_tc -s 20 -c 1 -o gpurun_out/tt python tools/prof_case.py 8192 256 1.0 1 > gpurun_out/ncu_tt.log 2>&1
ncu -i gpurun_out/tt.ncu-rep --page source --csv --print-source sass > gpurun_out/tt_src.csv 2>&1
