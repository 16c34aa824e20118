# QR update: CTA dephasing experiment (HLQ_QR_DEPHASE ns) on C3 all-QR hqr4 and C2.
set -u
O=gpurun_out/r2r
mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
for d in 0 250 500 1000; do
  HLQ_QR_DEPHASE=$d timeout 900 $B --fqr 1.0 --tree hqr4 > $O/c3f1_hqr4_d$d.log 2>&1
done
for d in 0 500; do
  HLQ_QR_DEPHASE=$d timeout 900 $B --config C2 --criterion max --alpha 1 --tree hqr4 > $O/c2_hqr4_d$d.log 2>&1
done
