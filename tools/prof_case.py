"""One small factorization for ncu captures: python tools/prof_case.py N nb fqr [reps [tree]]
(fqr = forced QR-step fraction of the C3 Bernoulli pattern; uniform seed 3 input on the device;
tree = greedy (default) or hqrA, TS groups of A tiles)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hlq_inputs as I  # noqa: E402
import paper_1401_5522_b200 as H  # noqa: E402

N, nb, fqr = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
tree = sys.argv[5] if len(sys.argv) > 5 else "greedy"
topt = {} if tree == "greedy" else {"tree": 1, "ts_group": int(tree[3:] or 4)}
n = (N + nb - 1) // nb
A0 = torch.empty(N * N, dtype=torch.float64, device="cuda")
H.hlq_generate_uniform(A0, N, N, N, 3, 0, N)
A = torch.empty_like(A0)
forced = I.bernoulli_pattern(30, n, fqr)
for _ in range(reps):
    A.copy_(A0)
    f = H.hlq_factor_ex(A, N, nb, 0, 1.0, forced=forced, **topt)
    f.free()
torch.cuda.synchronize()
print("ok")
