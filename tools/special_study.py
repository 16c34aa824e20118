"""Stability on the paper's formula-defined special matrices (Table III / Fig. 3), on the
GPU through the product path: HPL3 and QR-step fraction for Max (alpha = 6000) and MUMPS (alpha = 2.1)
as in P:953, the all-LU path (alpha = inf, tile-local pivoting: the analogue of LU NoPiv) and the
all-QR path (alpha = 0: the HQR analogue).  python tools/special_study.py [N] [nb] > out.json"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hlq_inputs as I  # noqa: E402
import paper_1401_5522_b200 as H  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 128
runs = [("max_6000", H.CRIT_MAX, 6000.0), ("mumps_2.1", H.CRIT_MUMPS, 2.1),
        ("all_lu", H.CRIT_MAX, math.inf), ("all_qr", H.CRIT_MAX, 0.0)]
out = {"N": N, "nb": nb, "rows": []}
for name in I.SPECIAL_BY_FORMULA:
    A = I.special_matrix(name, N)
    b = I.uniform_rhs(6, N)
    dA0 = H.to_colmajor(A)
    db = torch.from_numpy(b).cuda()
    row = {"matrix": name}
    for lab, crit, alpha in runs:
        dA = dA0.clone()
        f = H.hlq_factor_ex(dA, N, nb, crit, alpha)
        x = f.solve(db)
        res = H.hlq_residual(dA0, N, N, x, db)
        row[lab] = {"hpl3": res["hpl3"], "qr_fraction": float(f.decisions().mean()),
                    "growth": f.growth(), "status": f.status}
        f.free()
    ref = row["all_qr"]["hpl3"]
    for lab, _, _ in runs:
        h = row[lab]["hpl3"]
        row[lab]["ratio_to_all_qr"] = (h / ref) if (ref and math.isfinite(h)) else None
    out["rows"].append(row)
print(json.dumps(out, indent=1))
