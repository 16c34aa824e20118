"""Fig. 2-style alpha sweep on the GPU through the product path: for each criterion and
alpha, the LU-step fraction, HPL3, growth and the factor+solve rate (2N^3/3 basis and true flops).
Random uniform input (seed 0).  python tools/alpha_sweep.py [N] [nb] > out.json"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_5522_b200 as H  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 256
A0 = torch.empty(N * N, dtype=torch.float64, device="cuda")
b = torch.empty(N, dtype=torch.float64, device="cuda")
H.hlq_generate_uniform(A0, N, N, N, 0, 0, N)
H.hlq_generate_uniform(b, N, 1, N, 0, N * N, N)
A = torch.empty_like(A0)
x = torch.empty_like(b)
alphas = {"max": [1.0, 1e2, 1e3, 3e3, 1e4, 3e4, 1e5, math.inf],
          "sum": [1.0, 1e3, 1e4, 1e5, 3e5, 1e6, 1e7, math.inf],
          "mumps": [0.5, 1.0, 1.5, 2.0, 2.1, 3.0, 4.0, math.inf]}
crits = {"max": H.CRIT_MAX, "sum": H.CRIT_SUM, "mumps": H.CRIT_MUMPS}
out = {"N": N, "nb": nb, "input": "uniform[-0.5,0.5) seed 0", "rows": []}
for cname, al in alphas.items():
    for alpha in al:
        best = None
        for rep in range(2):  # first run warms up
            A.copy_(A0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f = H.hlq_factor_ex(A, N, nb, crits[cname], alpha)
            f.solve(b, x)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
            info = f.info()
            dec = f.decisions()
            f.free()
        res = H.hlq_residual(A0, N, N, x, b)
        out["rows"].append({"criterion": cname, "alpha": alpha, "lu_fraction": float(1 - dec.mean()),
                            "hpl3": res["hpl3"], "growth": info["growth"], "ms": best,
                            "tflops_2n3_3": info["fake_flops"] / (best * 1e-3) / 1e12,
                            "true_tflops": info["true_flops"] / (best * 1e-3) / 1e12})
print(json.dumps(out, indent=1))
