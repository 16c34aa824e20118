"""Schedule and kernel-shape variants must not change the factorization (-m gpu).

The speculative QR panel (HLQ_SPEC_QR) only moves the QR branch's panel work to a second stream and a
copy of the panel, and the DGEMM warp grid (HLQ_DGEMM_TILE) only changes which CTA computes which
output tile (every element still accumulates its K products in the same order): both must give
bit-identical factors and decisions.  The environment is read once per process, so each variant
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
N, nb = 1000, 128
A = I.normal_system(1, N)[0]
out = {{}}
for name, crit, alpha in (("max1", H.CRIT_MAX, 1.0), ("max3e4", H.CRIT_MAX, 3e4), ("lu", H.CRIT_MAX, float("inf"))):
    dA = H.to_colmajor(A)
    f = H.hlq_factor_ex(dA, N, nb, crit, alpha)
    out[name + "_F"] = H.from_colmajor(dA)
    out[name + "_d"] = f.decisions()
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


@pytest.mark.parametrize("env", [{"HLQ_SPEC_QR": "0"}, {"HLQ_DGEMM_TILE": "4x2"}])
def test_variant_is_bit_identical(tmp_path, env):
    base = _run({}, str(tmp_path / "base.npz"))
    var = _run(env, str(tmp_path / "var.npz"))
    for key in base.files:
        assert np.array_equal(base[key], var[key]), key
