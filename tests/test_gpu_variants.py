"""Schedule and kernel-shape variants must not change the factorization (-m gpu).

The speculative QR panel (HLQ_SPEC_QR) only moves the QR branch's panel work to a second stream and a
copy of the panel (its kernels run while d_k is undecided and exit once it is LU), the TMA-fed Schur update
(default) and the cp.async kernel (HLQ_DGEMM_TMA=0) accumulate every element's K products in the
same order; the QR panel as one dependency-DAG launch (default) or level by level (HLQ_QR_DAG=0)
runs the same kernels' arithmetic, and so does the solve's Q^T replay as one DAG launch per run of
QR steps (default) or step by step (HLQ_QR_SOLVE_DAG=0), and the lookahead column's update on the
panel stream (default) or in front of the rest on the update stream (HLQ_LA_SP=0): all must give bit-identical factors and x,
decisions and QR-step T factors -- under A1 and A2, Max and MUMPS, one and two QR-tree domains.  The environment is read once per process, so each variant
runs in its own interpreter."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import hlq_inputs as I, paper_1401_5522_b200 as H
N, nb = 1008, 128  # ragged last tile (112 rows), TMA-eligible (N, nb multiples of 16)
A = I.normal_system(1, N)[0]
U = I.uniform_matrix(3, N)
out = {{}}
# (name, matrix, criterion, alpha, options): mixed LU/QR decisions under A1 and A2, MUMPS, and two
# QR-tree domains (the speculative QR panel writes the T factors of QR steps directly)
cases = (("max1", A, H.CRIT_MAX, 1.0, {{}}), ("max3e4", A, H.CRIT_MAX, 3e4, {{}}),
         ("lu", A, H.CRIT_MAX, float("inf"), {{}}),
         ("a2_mix", U, H.CRIT_MAX, 1.2e4, dict(lu_variant=H.LU_A2)),
         ("mumps", A, H.CRIT_MUMPS, 2.1, {{}}),
         ("dom2", U, H.CRIT_MAX, 1.2e4, dict(tree_domains=2)),
         ("hqr4", U, H.CRIT_MAX, 1.2e4, dict(tree=H.TREE_HQR, ts_group=4)),
         ("hqr3_qr", A, H.CRIT_MAX, 0.0, dict(tree=H.TREE_HQR, ts_group=3, tree_domains=2)))
for name, M, crit, alpha, kw in cases:
    dA = H.to_colmajor(M)
    f = H.hlq_factor_ex(dA, N, nb, crit, alpha, **kw)
    out[name + "_F"] = H.from_colmajor(dA)
    d = f.decisions()
    out[name + "_d"] = d
    n = len(d)
    T = [f.T(i, k, kind) for k in range(n) if d[k] == 1 for i in range(k, n) for kind in (0, 1)]
    out[name + "_T"] = np.array(T) if T else np.zeros(0)
    out[name + "_x"] = f.solve(torch.from_numpy(I.uniform_rhs(7, N)).cuda()).cpu().numpy()
    f.free()
np.savez({path!r}, **out)
'''


def _run(env_extra, path):
    env = dict(os.environ)
    env.update(env_extra)
    code = SCRIPT.format(root=ROOT, path=path)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


@pytest.mark.parametrize("env", [{"HLQ_SPEC_QR": "0"}, {"HLQ_DGEMM_TMA": "0"},
                                 {"HLQ_TMA_CONS": "4"}, {"HLQ_QR_DAG": "0"},
                                 {"HLQ_QR_SOLVE_DAG": "0"}, {"HLQ_QR_SOLVE_DAG_BODY": "0"},
                                 {"HLQ_LA_SP": "0"}])
def test_variant_is_bit_identical(tmp_path, env):
    base = _run({}, str(tmp_path / "base.npz"))
    var = _run(env, str(tmp_path / "var.npz"))
    for key in base.files:
        assert np.array_equal(base[key], var[key]), key
