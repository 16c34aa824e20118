"""The special matrices the paper defines by formula (Table III), pinned to closed forms
and library routines (input generators: no method arithmetic)."""
import numpy as np
import pytest
from scipy.linalg import hilbert, toeplitz

import hlq_inputs as I


def test_hilb_is_scipy_hilbert_and_lotkin_first_row():
    np.testing.assert_array_equal(I.special_matrix("hilb", 12), hilbert(12))
    L = I.special_matrix("lotkin", 12)
    np.testing.assert_array_equal(L[0], np.ones(12))
    np.testing.assert_array_equal(L[1:], hilbert(12)[1:])


def test_house_and_orthogo_are_orthogonal():
    H = I.special_matrix("house", 50)
    np.testing.assert_allclose(H.T @ H, np.eye(50), atol=1e-14)
    np.testing.assert_allclose(H, H.T, atol=0)
    O = I.special_matrix("orthogo", 40)
    np.testing.assert_allclose(O @ O, np.eye(40), atol=1e-13)  # symmetric and orthogonal


def test_parter_is_toeplitz_and_ris_hankel_structure():
    P = I.special_matrix("parter", 9)
    i, j = np.indices((9, 9))
    np.testing.assert_array_equal(P, toeplitz(P[:, 0], P[0, :]))
    np.testing.assert_allclose(P, 1.0 / (i - j + 0.5))
    R = I.special_matrix("ris", 9)
    np.testing.assert_allclose(R, 0.5 / (9 - (i + 1) - (j + 1) + 1.5))
    Hk = I.special_matrix("hankel", 9)
    for s in range(17):  # constant anti-diagonals
        vals = [Hk[a, s - a] for a in range(9) if 0 <= s - a < 9]
        assert np.all(np.array(vals) == vals[0])


def test_lehmer_inverse_is_tridiagonal():
    Le = I.special_matrix("lehmer", 10)
    np.testing.assert_array_equal(Le, Le.T)
    Li = np.linalg.inv(Le)
    assert np.abs(np.triu(Li, 2)).max() < 1e-10
    assert np.all(np.linalg.eigvalsh(Le) > 0)


def test_compan_eigenvalues_are_polynomial_roots():
    C = I.special_matrix("compan", 8, seed=3)
    p = np.random.default_rng(3).standard_normal(9)
    ev = np.sort_complex(np.linalg.eigvals(C))
    np.testing.assert_allclose(ev, np.sort_complex(np.roots(p)), rtol=1e-8, atol=1e-10)


def test_demmel_row_scaling():
    D = I.special_matrix("demmel", 16)
    scale = 10.0 ** (14.0 * np.arange(16) / 16)
    R = D / scale[:, None]
    np.testing.assert_allclose(np.diag(R), 1.0 + np.diag(R - np.eye(16)), atol=0)
    assert np.abs(R - np.eye(16)).max() <= 1e-7


def test_unknown_special_matrix_is_refused():
    with pytest.raises(ValueError):
        I.special_matrix("foster", 10)  # named by the paper, not defined by it
