"""Diagnostic for the C5 recipe at reduced N: GPU vs oracle vs oracle variant, per step R (up to
row signs) and V differences.  python tools/parity_diag2.py N nb D"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hlq_inputs as I  # noqa: E402
import paper_1401_5522_b200 as H  # noqa: E402
from oracle import hlq_oracle as O  # noqa: E402

N, nb, D = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
spec = os.environ.get("SPEC", "1")
n = (N + nb - 1) // nb
A = I.uniform_matrix(2, N)
fo = O.hybrid_factor(A, nb, O.CRIT_MAX, 1.0, D=D)
fv = O.hybrid_factor(A, nb, O.CRIT_MAX, 1.0, D=D, forced=fo.dec, variant=1)
dA = H.to_colmajor(A)
f = H.hlq_factor_ex(dA, N, nb, 0, 1.0, tree_domains=D)
F = H.from_colmajor(dA)
dA2 = H.to_colmajor(A)
f2 = H.hlq_factor_ex(dA2, N, nb, 0, 1.0, tree_domains=D, forced=fo.dec)
F2 = H.from_colmajor(dA2)
print("dec", "".join("LQ"[d] for d in f.decisions()), "==oracle", np.array_equal(f.decisions(), fo.dec))
print(f"eps_F gpu {O.factor_diff(F, fo.A):.3e}  gpu(forced, no speculation) {O.factor_diff(F2, fo.A):.3e}  "
      f"variant {O.factor_diff(fv.A, fo.A):.3e}  gpu-vs-gpu(forced) {O.factor_diff(F, F2):.3e}")
G = fo.A
for k in range(n):
    r0, r1 = k * nb, min((k + 1) * nb, N)
    def rdiff(X):
        sx = np.where(np.diag(X[r0:r1, r0:r1]) < 0, -1.0, 1.0)
        sg = np.where(np.diag(G[r0:r1, r0:r1]) < 0, -1.0, 1.0)
        a = np.triu(X[r0:r1, r0:]) * sx[:, None]
        b_ = np.triu(G[r0:r1, r0:]) * sg[:, None]
        return np.linalg.norm(a - b_) / np.linalg.norm(b_), int(np.sum(sx != sg))
    rg, fg = rdiff(F)
    rv, fvv = rdiff(fv.A)
    Vg = np.linalg.norm(F[r1:, r0:r1] - G[r1:, r0:r1]) / max(np.linalg.norm(G[r1:, r0:r1]), 1e-300)
    Vv = np.linalg.norm(fv.A[r1:, r0:r1] - G[r1:, r0:r1]) / max(np.linalg.norm(G[r1:, r0:r1]), 1e-300)
    print(f"step {k:3d} {'LQ'[fo.dec[k]]}: R gpu {rg:.2e} (flips {fg}) variant {rv:.2e} (flips {fvv}) | V gpu {Vg:.2e} variant {Vv:.2e}")
