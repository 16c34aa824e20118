"""One Schur update, TMA vs cp.async kernel, bitwise (no other stream running)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1401_5522_b200 as H
for N in (2048, 8192, 16384):
    for k0 in (0, 256 * 7):
        A0 = torch.empty(N * N, dtype=torch.float64, device="cuda")
        H.hlq_generate_uniform(A0, N, N, N, 3, 0, N)
        A1 = A0.clone()
        r0 = H.hlq_test_schur(A0, N, N, k0, 256, True)
        r1 = H.hlq_test_schur(A1, N, N, k0, 256, False)
        d = (A0 != A1).sum().item()
        print(N, k0, "tma ran" if r0 == 1 else "tma NOT run", "differing entries:", d, flush=True)
        if d:
            idx = torch.nonzero((A0 != A1).view(N, N))[:3].tolist()  # (col, row) storage order
            print("   first (col,row):", idx)
