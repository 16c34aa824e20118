#!/bin/bash
# Per-kernel launch times (ncu, serialised, cold cache) of one small all-QR / all-LU case:
#   bash tools/launch_times.sh N nb fqr out.csv
set -u
python tools/prof_case.py $1 $2 $3 1 > /dev/null 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $4 \
    python tools/prof_case.py $1 $2 $3 1 > /dev/null 2>&1
