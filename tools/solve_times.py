#!/usr/bin/env python
"""Repeated solve timings on one factorization (CUDA events on the solve's stream):
python tools/solve_times.py CONFIG N nb [fqr|max] [tree] -- prints min / median / max ms of 12 solves."""
import statistics
import sys

import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hlq_inputs as I
import paper_1401_5522_b200 as H

cfg, N, nb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
mode = sys.argv[4] if len(sys.argv) > 4 else "max"
tree = sys.argv[5] if len(sys.argv) > 5 else "greedy"
A, b, _ = I.config_system(cfg, N)
dA = H.to_colmajor(A)
n = (N + nb - 1) // nb
kw = {}
if tree.startswith("hqr"):
    kw.update(tree=H.TREE_HQR, ts_group=int(tree[3:]))
if mode == "max":
    f = H.hlq_factor_ex(dA, N, nb, H.CRIT_MAX, 1.0, **kw)
else:
    f = H.hlq_factor_ex(dA, N, nb, H.CRIT_MAX, 1.0, forced=I.bernoulli_pattern(30, n, float(mode)), **kw)
db = torch.from_numpy(np.ascontiguousarray(b)).cuda()
x = torch.empty_like(db)
ts = []
for it in range(14):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f.solve(db, x)
    e1.record()
    torch.cuda.synchronize()
    if it >= 2:
        ts.append(e0.elapsed_time(e1))
print(cfg, N, nb, mode, tree, os.environ.get("HLQ_QR_SOLVE_DAG_BODY", "1"),
      "solve ms min %.2f med %.2f max %.2f" % (min(ts), statistics.median(ts), max(ts)),
      " ".join("%.1f" % t for t in ts), flush=True)
