# C5-recipe Householder sign question: GPU determinism across scheduling variants, the recipe at small
# sizes with the same ragged tile, and the full-size record with the oracle's small-alpha log and the
# flipped rows' indices.
set -u
O=gpurun_out/r2m
mkdir -p $O
timeout 900 python tools/gpu_determinism.py --out $O/determinism.json > $O/determinism.log 2>&1
timeout 900 python tools/sign_probe.py --out $O/sign_probe.jsonl 5 9 17 25 > $O/sign_probe.log 2>&1
timeout 3300 python tools/parity_full.py C5r --out $O/parity > $O/parity_c5r.log 2>&1
