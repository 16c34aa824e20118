"""Diagnostic: where do the GPU's and the oracle's packed factors differ?  All-QR C3 recipe at N.
Prints the relative difference per tile row block of R (rows of step k) and per V tile column."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hlq_inputs as I  # noqa: E402
import paper_1401_5522_b200 as H  # noqa: E402
from oracle import hlq_oracle as O  # noqa: E402

N, nb = int(sys.argv[1]), int(sys.argv[2])
tree = sys.argv[3] if len(sys.argv) > 3 else "greedy"
n = N // nb
A = I.uniform_matrix(3, N)
forced = np.ones(n, dtype=np.uint8)
dA = H.to_colmajor(A)
kw = {} if tree == "greedy" else {"tree": 1, "ts_group": int(tree[3:])}
f = H.hlq_factor_ex(dA, N, nb, 0, 1.0, forced=forced, **kw)
F = H.from_colmajor(dA)
dA2 = H.to_colmajor(A)
f2 = H.hlq_factor_ex(dA2, N, nb, 0, 1.0, forced=forced, **kw)
print("gpu run-to-run identical:", np.array_equal(F, H.from_colmajor(dA2)), flush=True)
t = time.time()
fo = O.hybrid_factor(A, nb, forced=forced, tree=tree)
print(f"oracle {time.time() - t:.0f}s eps_F {O.factor_diff(F, fo.A):.3e}", flush=True)
G = fo.A
for k in range(n):
    rk = slice(k * nb, (k + 1) * nb)
    Rg, Ro = np.triu(F[rk, k * nb:]), np.triu(G[rk, k * nb:])
    dR = np.linalg.norm(Rg - Ro) / np.linalg.norm(Ro)
    # R up to row signs
    sg = np.sign(np.diag(F[rk, rk]) * np.diag(G[rk, rk]))
    dRs = np.linalg.norm(Rg * sg[:, None] - Ro) / np.linalg.norm(Ro)
    Vg, Vo = F[(k + 1) * nb:, rk], G[(k + 1) * nb:, rk]
    dV = np.linalg.norm(Vg - Vo) / max(np.linalg.norm(Vo), 1e-300) if Vo.size else 0.0
    flips = int(np.sum(sg < 0))
    print(f"step {k:3d}: R rows rel diff {dR:.2e} (up to row signs {dRs:.2e}, sign flips {flips}), "
          f"V column block {dV:.2e}", flush=True)
