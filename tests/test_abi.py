"""-m "not gpu": the C-ABI library loads and exports every symbol include/hlq.h declares; the
ctypes structures match the C layout; argument errors are reported without touching a GPU."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hlq.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hlq_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def built():
    import __graft_entry__ as g
    g.build()
    return g.LIB


def test_every_declared_symbol_is_exported(built):
    lib = ctypes.CDLL(built)
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_struct_layout_matches_binding(built):
    import paper_1401_5522_b200 as H
    so, si, ver = H.hlq_abi()
    assert so == ctypes.sizeof(H.HlqOptions) and si == ctypes.sizeof(H.HlqInfo) and ver == 1
    o = H.hlq_default_options()
    assert o.struct_size == so and o.ib == 32 and o.tie_rel_tol == 1e-10 and o.blocking == 1


def test_argument_errors_without_gpu(built):
    import paper_1401_5522_b200 as H
    lib = H.lib
    h = ctypes.c_void_p()
    # NULL A, bad N, bad nb, bad criterion, NaN alpha: LAPACK-style negative codes
    assert lib.hlq_factor(None, 8, 2, 0, 1.0, ctypes.byref(h)) == -1
    dummy = ctypes.c_void_p(0x1000)
    assert lib.hlq_factor(dummy, 0, 2, 0, 1.0, ctypes.byref(h)) == -2
    assert lib.hlq_factor(dummy, 8, 0, 0, 1.0, ctypes.byref(h)) == -3
    assert lib.hlq_factor(dummy, 4096, 321, 0, 1.0, ctypes.byref(h)) == -3  # HLQ_MAX_NB = 320
    # options: unknown LU variant; A2 needs ib = 32 and the exact inverse norm
    for fields in ({"lu_variant": 2}, {"lu_variant": 1, "ib": 16},
                   {"lu_variant": 1, "invnorm_estimate": 1}, {"pivot_scope": 2},
                   {"pivot_scope": 1, "lu_variant": 1}, {"ib": 16}, {"ib": 8}, {"ib": 33}):
        opt = H.hlq_default_options()
        for k, v in fields.items():
            setattr(opt, k, v)
        assert lib.hlq_factor_ex(dummy, 8, 2, 0, 1.0, ctypes.byref(opt), ctypes.byref(h)) == -6
    assert lib.hlq_factor(dummy, 8, 2, 5, 1.0, ctypes.byref(h)) == -4
    assert lib.hlq_factor(dummy, 8, 2, 0, float("nan"), ctypes.byref(h)) == -5
    assert lib.hlq_factor(dummy, 8, 2, 0, -1.0, ctypes.byref(h)) == -5
    assert lib.hlq_solve(None, None, None) == -1
    assert lib.hlq_status_string(2) == b"exact zero on the final U/R diagonal"


def test_product_path_has_no_oracle_or_cpu_fallback():
    pkg = os.path.join(ROOT, "paper_1401_5522_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert not re.search(r"(import|from)\s+oracle|hlq_oracle|hlqo_", txt), fn
                assert "numpy.linalg" not in txt and "scipy" not in txt, fn


def test_binding_validates_arguments_before_the_call(built):
    """The binding refuses what the C side cannot check (host-side, no GPU needed): a non-CUDA or
    wrong-dtype matrix, a matrix smaller than lda*(N-1)+N, per-step vectors of the wrong length,
    ref_dec without ref_margin."""
    import numpy as np
    import torch
    import paper_1401_5522_b200 as H
    with pytest.raises(H.HlqError, match="float64 CUDA"):
        H.hlq_factor_ex(torch.zeros(64, dtype=torch.float64), 8, 4)
    with pytest.raises(H.HlqError, match="float64 CUDA"):
        H.hlq_factor_ex(torch.zeros(64, dtype=torch.float32), 8, 4)
    opt = H.hlq_default_options()
    with pytest.raises(H.HlqError):
        H._step_vectors(opt, 2, np.zeros(3), None, None, [])
    with pytest.raises(H.HlqError, match="together"):
        H._step_vectors(opt, 2, None, np.zeros(2), None, [])
    with pytest.raises(H.HlqError):
        H._step_vectors(opt, 2, None, np.zeros(2), np.zeros(1), [])
    keep = []
    H._step_vectors(opt, 2, np.array([0, 1]), np.array([1, 0]), np.array([0.5, -0.5]), keep)
    assert len(keep) == 3 and opt.forced and opt.ref_dec and opt.ref_margin
