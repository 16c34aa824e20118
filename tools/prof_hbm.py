"""One factorization + solve for the HBM-bound kernels' ncu captures (row d):
    python tools/prof_hbm.py N nb mode [hqrA]
mode "crit": Max criterion alpha = 1.2e4 (panel statistics, LU/QR mix, the decision kernels);
mode "lu": forced all LU (k_colpart_max, the persistent LU solve); mode "qr": forced all QR
(the Q^T replay DAG k_qr_solve_dag in the solve; optional HQR tree with TS groups of A).  Uniform seed 3 input generated on the device."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hlq_inputs as I  # noqa: E402
import paper_1401_5522_b200 as H  # noqa: E402

N, nb, mode = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
tree = sys.argv[4] if len(sys.argv) > 4 else "greedy"
kw = dict(tree=H.TREE_HQR, ts_group=int(tree[3:])) if tree.startswith("hqr") else {}
n = (N + nb - 1) // nb
A = torch.empty(N * N, dtype=torch.float64, device="cuda")
H.hlq_generate_uniform(A, N, N, N, 3, 0, N)
b = torch.empty(N, dtype=torch.float64, device="cuda")
H.hlq_generate_uniform(b, N, 1, N, 3, N * N, N)
if mode == "crit":
    f = H.hlq_factor_ex(A, N, nb, H.CRIT_MAX, 1.2e4)
else:
    f = H.hlq_factor_ex(A, N, nb, H.CRIT_MAX, 1.0,
                        forced=I.bernoulli_pattern(30, n, 0.0 if mode == "lu" else 1.0), **kw)
x = f.solve(b)
torch.cuda.synchronize()
print("ok", "".join("LQ"[d] for d in f.decisions()))
