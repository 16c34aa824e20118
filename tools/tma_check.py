"""TMA Schur DGEMM vs the cp.async kernel: the factorizations must be bit-identical (same DMMA
accumulation order).  python tools/tma_check.py N nb"""
import os
import subprocess
import sys

import numpy as np

N, nb = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 3:  # child: factor and dump
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import hlq_inputs as I
    import paper_1401_5522_b200 as H
    n = (N + nb - 1) // nb
    A = torch.empty(N * N, dtype=torch.float64, device="cuda")
    H.hlq_generate_uniform(A, N, N, N, 3, 0, N)
    f = H.hlq_factor_ex(A, N, nb, 0, 1.0, forced=np.zeros(n, dtype=np.uint8))
    torch.cuda.synchronize()
    np.save(sys.argv[3], A.cpu().numpy())
    sys.exit(0)
outs = []
for tma in ("1", "0"):
    p = f"/tmp/tma_{tma}.npy"
    subprocess.run([sys.executable, __file__, str(N), str(nb), p], check=True,
                   env={**os.environ, "HLQ_DGEMM_TMA": tma})
    outs.append(np.load(p).reshape(N, N).T)
a, b = outs
print("bit-identical:", np.array_equal(a, b), "max abs diff", float(np.nanmax(np.abs(a - b))))
bad = np.argwhere(~(a == b))
if bad.size:
    print("first differing (row, col):", bad[:5].tolist(), "count", len(bad))
    r, c = bad[0]
    print("tile", r // nb, c // nb)
