import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1401_5522_b200 as H
N = 2048
for rep in range(3):
    A0 = torch.empty(N * N, dtype=torch.float64, device="cuda")
    H.hlq_generate_uniform(A0, N, N, N, 3, 0, N)
    A1 = A0.clone()
    H.hlq_test_schur(A0, N, N, 0, 256, True)
    H.hlq_test_schur(A1, N, N, 0, 256, False)
    a = A0.view(N, N).cpu().numpy().T
    b = A1.view(N, N).cpu().numpy().T
    bad = np.argwhere(a != b)
    print("rep", rep, "differing", len(bad))
    tiles = {}
    for r, c in bad:
        key = ((r - 256) // 64, (c - 256) // 64)
        tiles.setdefault(key, []).append(((r - 256) % 64, (c - 256) % 64))
    for key, v in sorted(tiles.items())[:6]:
        rows = sorted(set(x for x, _ in v)); cols = sorted(set(y for _, y in v))
        print("  tile", key, "rows", rows[:20], "ncols", len(cols), "cols", cols[:8], "...", cols[-4:])
    if len(bad):
        r, c = bad[0]
        print("  sample got", a[r, c], "want", b[r, c])
