#!/usr/bin/env python
"""Per-step NVLink volume and time model of the 2D block-cyclic factorization (row e)
for C5 (N = 131072, nb = 320, D = 2, Max alpha = 1: every step but the last is QR) on a P x Q grid.

Nothing here is measured on more than one GPU (this run has one); the model combines
  * the exchange schedule of dist.cu (X1 statistics allgather, X2 domain-head allgather, X3 panel
    package broadcast, X4 head-row allgather) with its exact payload sizes,
  * the guide's measured NVLink figures (B200_PROFILING.md: 770 GB/s peer copy per direction) and
    an assumed per-collective latency,
  * the single-GPU kernel rates measured on this pool (QR update class, panel kernels at nb = 320),
and sums, per step k, max(update of step k on the busiest rank, panel stage of step k+1 incl. its
exchanges) -- the lookahead-1 schedule of the library.  The same formulas at P = Q = 1 reproduce the
measured one-GPU C5 time (calibration) and give the predicted scaling efficiency.

  python tools/dist_model.py [--P 2 --Q 4] [--json out.json]
"""
from __future__ import annotations

import argparse
import json
import math

# ---- measured on one B200 (profiles/r01, profiles/r02; nb = 320)
QR_UPDATE_TF = 18.6       # QR trailing-update class, true Table-I flops / s (C5 full size, 1 GPU)
LU_UPDATE_TF = 30.0       # LU Schur update class (C3)
T_GEQRT_MS = 1.10         # k_geqrt_tc per launch at nb = 320 (all tiles of a column in parallel)
T_TTQRT_MS = 0.867        # k_ttqrt_tc per launch (one tree level, all pairs in parallel)
T_PANEL_STATS_MS = 0.05   # criterion statistics + GETRF + decide hidden behind the QR panel
# ---- NVLink / NCCL (B200_PROFILING.md measured peer copy; latency assumed)
LINK_GBS = 770.0
COLL_LAT_US = 25.0


def step_model(N, nb, P, Q, D, k, qr=True):
    n = -(-N // nb)
    m = n - k - 1                         # sub-diagonal tiles of step k
    tb = nb * nb * 8                      # bytes of one tile
    tT = 32 * nb * 8                      # bytes of one ib x nb T factor
    # busiest rank: tile rows / columns of the trailing matrix it owns (block-cyclic)
    rows_p = -(-(m + 1) // P)
    cols_q = -(-m // Q) if m > 0 else 0
    # ---- compute
    if qr:
        upd_flops = 4.0 * rows_p * cols_q * nb ** 3      # Table I: 4 nb^3 per (eliminated tile, column)
        upd_ms = upd_flops / (QR_UPDATE_TF * 1e12) * 1e3
        md = -(-(m + 1) // max(D, 1))                     # tiles of one domain in this column
        levels = math.ceil(math.log2(md)) if md > 1 else 0
        inter = math.ceil(math.log2(min(D, m + 1))) if m + 1 > 1 else 0
        panel_ms = T_GEQRT_MS + (levels + inter) * T_TTQRT_MS + T_PANEL_STATS_MS
    else:
        upd_flops = 2.0 * rows_p * cols_q * nb ** 3
        upd_ms = upd_flops / (LU_UPDATE_TF * 1e12) * 1e3
        panel_ms = 0.6
    # ---- exchanges (bytes leaving / arriving at one rank)
    if P * Q == 1:
        return dict(m=m, upd_ms=upd_ms, panel_ms=panel_ms, x_ms=0.0, x4_ms=0.0, bytes=0)
    loc_panel = -(-(m + 1) // P)                          # panel tiles on one rank of column qk
    x1 = (loc_panel + 2 * nb) * 8 + (tb + 4 * nb if P > 1 else 0)    # norms, maxes, W + ipiv
    x2 = (tb if qr else 0) * (1 if P > 1 else 0)          # the local domain head's R
    x3 = loc_panel * (tb + (2 * tT if qr else 0)) + 2 * tb + 64      # panel tiles, T's, merges, d_k
    x4 = nb * cols_q * nb * 8                             # head rows of the local trailing columns
    lat = COLL_LAT_US / 1e3
    ms = lambda b: b / (LINK_GBS * 1e9) * 1e3             # noqa: E731
    x_panel = (lat + ms(x1 * (P - 1))) * (P > 1) + (lat + ms(x2 * (P - 1))) * (P > 1) \
        + (lat + ms(x3)) * (Q > 1)                        # on the panel critical path
    x4_ms = (lat + ms(x4 * (P - 1))) * (P > 1)            # overlapped with the update
    return dict(m=m, upd_ms=upd_ms, panel_ms=panel_ms, x_ms=x_panel, x4_ms=x4_ms,
                bytes=x1 * (P - 1) + x2 * (P - 1) + x3 + x4 * (P - 1))


def run_model(N, nb, P, Q, D):
    n = -(-N // nb)
    total = 0.0
    bytes_tot = 0
    exposed_panel = 0.0
    rows = []
    for k in range(n):
        s = step_model(N, nb, P, Q, D, k, qr=(k < n - 1))
        nxt = step_model(N, nb, P, Q, D, k + 1, qr=(k + 1 < n - 1)) if k + 1 < n else None
        crit = (nxt["panel_ms"] + nxt["x_ms"]) if nxt else 0.0
        upd = s["upd_ms"] + s["x4_ms"] * 0.0  # X4 overlaps the update's other column blocks
        t = max(upd, crit)
        if k == 0:
            t += s["panel_ms"] + s["x_ms"]
        exposed_panel += max(0.0, crit - upd)
        total += t
        bytes_tot += s["bytes"]
        if k % 41 == 0 or k == n - 1:
            rows.append({"k": k, "m": s["m"], "update_ms": round(s["upd_ms"], 3),
                         "panel_next_ms": round(crit, 3), "exch_MB": round(s["bytes"] / 1e6, 2),
                         "step_ms": round(t, 3)})
    return total / 1e3, bytes_tot, exposed_panel / 1e3, rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=131072)
    ap.add_argument("--nb", type=int, default=320)
    ap.add_argument("--P", type=int, default=2)
    ap.add_argument("--Q", type=int, default=4)
    ap.add_argument("--D", type=int, default=2)
    ap.add_argument("--json")
    a = ap.parse_args()
    t1, _, e1, _ = run_model(a.N, a.nb, 1, 1, a.D)
    tg, bts, eg, rows = run_model(a.N, a.nb, a.P, a.Q, a.D)
    G = a.P * a.Q
    out = {
        "config": {"N": a.N, "nb": a.nb, "D": a.D, "grid": f"{a.P}x{a.Q}", "all_steps": "QR but the last"},
        "assumptions": {"qr_update_tf_per_gpu": QR_UPDATE_TF, "t_geqrt_ms": T_GEQRT_MS,
                        "t_ttqrt_ms": T_TTQRT_MS, "link_GBps": LINK_GBS,
                        "collective_latency_us": COLL_LAT_US},
        "one_gpu_model_s": round(t1, 2),
        "grid_model_s": round(tg, 2),
        "ideal_s": round(t1 / G, 2),
        "predicted_efficiency": round(t1 / (G * tg), 3),
        "exposed_panel_s": round(eg, 2),
        "nvlink_bytes_per_rank_GB": round(bts / 1e9, 2),
        "nvlink_time_at_link_bw_s": round(bts / (LINK_GBS * 1e9), 3),
        "steps_sampled": rows,
    }
    print(json.dumps(out, indent=1))
    if a.json:
        json.dump(out, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
