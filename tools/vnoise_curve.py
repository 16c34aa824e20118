#!/usr/bin/env python
"""Per-step noise curves of an all-QR factorization (test infrastructure: oracle/, the input module,
the C ABI).  For one (N, nb, tree) it factors the same matrix with the oracle, with its two noise
variants (1: reversed summation in the trailing updates; 2: that plus reversed summation of the
reflector norms inside the panel kernels) and on the GPU, and records for every step k the relative
difference to the oracle of
    V_k : the reflector tiles of step k (column block k below the diagonal tile row), and
    R_k : the rows of block k from column k*nb on, rows normalised to a nonnegative diagonal,
so that the growth of a rounding-level perturbation through the steps (the V tiles of a tree QR
are determined only up to an ill-conditioned rotation) can be compared between
"another rounding of the oracle" and "the GPU".

  python tools/vnoise_curve.py N nb tree [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import hlq_inputs as I  # noqa: E402
from oracle import hlq_oracle as O  # noqa: E402


def curves(F, G, N, nb):
    n = (N + nb - 1) // nb
    v, r, flips = [], [], []
    for k in range(n):
        r0, r1 = k * nb, min((k + 1) * nb, N)
        dv = np.linalg.norm(F[r1:, r0:r1] - G[r1:, r0:r1])
        nv = np.linalg.norm(G[r1:, r0:r1])
        v.append(float(dv / nv) if nv > 0 else 0.0)
        df, dg = np.diag(F[r0:r1, r0:r1]), np.diag(G[r0:r1, r0:r1])
        sf, sg = np.where(df < 0, -1.0, 1.0), np.where(dg < 0, -1.0, 1.0)
        Rf, Rg = np.triu(F[r0:r1, r0:]) * sf[:, None], np.triu(G[r0:r1, r0:]) * sg[:, None]
        nr = np.linalg.norm(Rg)
        r.append(float(np.linalg.norm(Rf - Rg) / nr) if nr > 0 else 0.0)
        flips.append(int(np.sum(sf != sg)))
    return {"V": v, "R": r, "flips": flips}


def _oracle(args):
    N, nb, tree, variant, path = args
    A = I.config_system("C3", N)[0]
    n = (N + nb - 1) // nb
    forced = np.ones(n, dtype=np.uint8)
    t0 = time.perf_counter()
    F = O.hybrid_factor(A, nb, O.CRIT_MAX, 1.0, forced=forced, variant=variant, tree=tree).A
    np.save(path, F)
    return time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("N", type=int)
    ap.add_argument("nb", type=int)
    ap.add_argument("tree")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    N, nb, tree = a.N, a.nb, a.tree
    out = a.out or os.path.join(ROOT, "gpurun_out", f"vnoise_{N}_{nb}_{tree}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    tmp = [out + f".v{v}.npy" for v in (0, 1, 2)]
    with mp.get_context("fork").Pool(3) as pool:
        secs = pool.map(_oracle, [(N, nb, tree, v, tmp[v]) for v in (0, 1, 2)])
    import torch
    import paper_1401_5522_b200 as H
    A = I.config_system("C3", N)[0]
    n = (N + nb - 1) // nb
    dA = H.to_colmajor(A)
    kw = dict(tree=H.TREE_HQR, ts_group=int(tree[3:])) if tree.startswith("hqr") else {}
    f = H.hlq_factor_ex(dA, N, nb, H.CRIT_MAX, 1.0, forced=np.ones(n, dtype=np.uint8), **kw)
    torch.cuda.synchronize()
    f.free()
    Fg = H.from_colmajor(dA)
    F0 = np.load(tmp[0])
    rec = {"N": N, "nb": nb, "tree": tree, "n": n, "oracle_s": secs,
           "gpu": curves(Fg, F0, N, nb),
           "variant1": curves(np.load(tmp[1]), F0, N, nb),
           "variant2": curves(np.load(tmp[2]), F0, N, nb),
           "eps_F": {"gpu": O.factor_diff(Fg, F0),
                     "variant1": O.factor_diff(np.load(tmp[1]), F0),
                     "variant2": O.factor_diff(np.load(tmp[2]), F0)}}
    for t in tmp:
        os.remove(t)

    def rate(c):  # geometric growth per step of the V difference over the steps where it is resolved
        ks = [k for k, x in enumerate(c["V"]) if 1e-14 < x < 1e-2]
        if len(ks) < 8:
            return None
        lo, hi = ks[0], ks[-1]
        return math.exp((math.log(c["V"][hi]) - math.log(c["V"][lo])) / max(1, hi - lo))
    rec["V_growth_per_step"] = {k: rate(rec[k]) for k in ("gpu", "variant1", "variant2")}
    json.dump(rec, open(out, "w"))
    pick = list(range(0, n, max(1, n // 16)))
    print(json.dumps({"N": N, "nb": nb, "tree": tree, "eps_F": rec["eps_F"],
                      "V_growth_per_step": rec["V_growth_per_step"], "steps": pick,
                      "V_gpu": [rec["gpu"]["V"][k] for k in pick],
                      "V_variant1": [rec["variant1"]["V"][k] for k in pick],
                      "V_variant2": [rec["variant2"]["V"][k] for k in pick],
                      "R_gpu_max": max(rec["gpu"]["R"]), "R_variant2_max": max(rec["variant2"]["R"]),
                      "oracle_s": secs}), flush=True)


if __name__ == "__main__":
    main()
