#!/usr/bin/env python
"""Householder sign-decision probe (test infrastructure: oracle/, the input module, the C ABI).

The C5-recipe parity record (profiles/r02/parity/C5r.json) has 42 rows of step 85's R negated on
the GPU relative to the oracle.  This probe runs the same recipe (normal input, nb = 320, D = 2,
greedy tree, Max alpha = 1) at sizes N = 320 t + 128 (the same ragged last tile of 128 rows) and
reports, per size: the rows of R whose sign differs (step and row index), eps_F, eps_R, and the
oracle's reflectors with |alpha| < 1e-6 ||(alpha, x)|| (LARFG_LOG) -- a sign decision near its
discontinuity.

  python tools/sign_probe.py [--nb 320] [--rag 128] [--D 2] [--tree greedy] t [t ...]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402

import hlq_inputs as I  # noqa: E402
from oracle import hlq_oracle as O  # noqa: E402
from parity_full import r_part_diff  # noqa: E402


def flipped_rows(F, G, N, nb):
    out = {}
    for k in range((N + nb - 1) // nb):
        r0, r1 = k * nb, min((k + 1) * nb, N)
        df, dg = np.diag(F[r0:r1, r0:r1]), np.diag(G[r0:r1, r0:r1])
        idx = np.nonzero(np.sign(df) != np.sign(dg))[0]
        if idx.size:
            out[str(k)] = {"rows": idx.tolist(), "gpu_diag": df[idx].tolist(),
                           "oracle_diag": dg[idx].tolist()}
    return out


def main():
    import torch
    import paper_1401_5522_b200 as H
    ap = argparse.ArgumentParser()
    ap.add_argument("t", nargs="+", type=int)
    ap.add_argument("--nb", type=int, default=320)
    ap.add_argument("--rag", type=int, default=128)
    ap.add_argument("--D", type=int, default=2)
    ap.add_argument("--tree", default="greedy")
    ap.add_argument("--config", default="C5")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sign_probe.jsonl"))
    a = ap.parse_args()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    for t in a.t:
        N, nb = a.nb * t + a.rag, a.nb
        A, b, _ = I.config_system(a.config, N)
        O.LARFG_LOG = []
        t0 = time.perf_counter()
        fo = O.hybrid_factor(A, nb, O.CRIT_MAX, 1.0, D=a.D, tree=a.tree)
        ts = time.perf_counter() - t0
        log = O.LARFG_LOG
        O.LARFG_LOG = None
        dA = H.to_colmajor(A)
        kw = dict(tree_domains=a.D)
        if a.tree.startswith("hqr"):
            kw.update(tree=H.TREE_HQR, ts_group=int(a.tree[3:]))
        f = H.hlq_factor_ex(dA, N, nb, O.CRIT_MAX, 1.0, **kw)
        torch.cuda.synchronize()
        dec = f.decisions()
        f.free()
        F = H.from_colmajor(dA)
        rec = {"N": N, "nb": nb, "D": a.D, "tree": a.tree, "oracle_s": round(ts, 1),
               "decisions": "".join("LQ"[d] for d in fo.dec),
               "decisions_identical": bool(np.array_equal(dec, fo.dec)),
               "eps_F": O.factor_diff(F, fo.A), "eps_R": r_part_diff(F, fo.A, N, nb),
               "flipped": flipped_rows(F, fo.A, N, nb),
               "oracle_small_alpha": [(k, al, nr) for k, al, nr in log][:200],
               "oracle_small_alpha_count": len(log)}
        print(json.dumps(rec), flush=True)
        with open(a.out, "a") as fh:
            fh.write(json.dumps(rec) + "\n")
        del dA, F


if __name__ == "__main__":
    main()
