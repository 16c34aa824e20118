"""Pins for the CPU oracle (-m "not gpu"): each oracle function is checked against something other
than itself -- LAPACK routines (scipy.linalg.lapack), numpy dense formulas, the paper's worked example
and bounds, brute force on tiny tiled matrices.  See DESIGN.md "Oracle pins"."""
import itertools
import math
import os

import numpy as np
import pytest
import scipy.linalg as sl
import scipy.linalg.lapack as lapack

import hlq_inputs as I
from oracle import hlq_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(1234)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ---------------------------------------------------------------- P1: tile kernels
def test_norm1_hand_values():
    assert O.norm1(np.array([[1.0, -2.0], [3.0, 4.0]])) == 6.0
    assert O.norm1(np.eye(5)) == 1.0
    T = RNG.standard_normal((7, 7))
    assert O.norm1(T) == pytest.approx(np.linalg.norm(T, 1), rel=1e-15)


@pytest.mark.parametrize("b", [1, 2, 5, 16, 64])
def test_getrf_matches_lapack_dgetrf(b):
    for _ in range(3):
        T = RNG.standard_normal((b, b))
        W, ipiv, zp = O.getrf(T)
        lu, piv, info = lapack.dgetrf(T)
        assert not zp and info == 0
        np.testing.assert_array_equal(ipiv, piv)
        assert rel(W, lu) < 1e-13


def test_getrf_forced_swap_and_zero_pivot():
    W, ipiv, zp = O.getrf(np.array([[0.0, 1.0], [1.0, 0.0]]))  # SPEC: [[0,1],[1,0]] -> swap, U = I
    assert list(ipiv) == [1, 1] and not zp
    np.testing.assert_array_equal(np.triu(W), np.eye(2))
    W, ipiv, zp = O.getrf(np.array([[1.0, 2.0], [2.0, 4.0]]))
    assert zp  # singular tile: exact zero pivot flagged (ledger 7)
    # tie-break: first maximum (ledger 6)
    W, ipiv, zp = O.getrf(np.array([[1.0, 0.0, 0.0], [-3.0, 1.0, 0.0], [3.0, 0.0, 1.0]]))
    assert ipiv[0] == 1


@pytest.mark.parametrize("b", [1, 3, 32, 100])
def test_inv_norm_matches_dense_inverse(b):
    T = RNG.standard_normal((b, b))
    W, _, _ = O.getrf(T)
    assert O.inv_norm1_from_lu(W) == pytest.approx(np.linalg.norm(np.linalg.inv(T), 1), rel=1e-11)
    W, _, _ = O.getrf(np.diag([2.0, 0.5]))
    assert O.inv_norm1_from_lu(W) == 2.0


@pytest.mark.parametrize("b", [2, 3, 17, 64, 128, 256])
def test_inv_norm_estimate_matches_lapack_dgecon(b):
    """NEXT f3: the oracle's Hager/Higham iteration is LAPACK's: dgecon on the same LU
    factors returns rcond = 1 / (||A||_1 * est), and est is a lower bound of the exact norm."""
    from scipy.linalg import lapack, lu_factor
    rng = np.random.default_rng(100 + b)
    for trial in range(6):
        T = rng.standard_normal((b, b)) if trial % 2 else rng.uniform(-0.5, 0.5, (b, b))
        W, _, _ = O.getrf(T)
        lu, _ = lu_factor(T)
        anorm = float(np.abs(T).sum(axis=0).max())
        rcond, info = lapack.dgecon(lu, anorm, norm="1")
        assert info == 0
        est = O.inv_norm1_estimate(W)
        assert est == pytest.approx(1.0 / (rcond * anorm), rel=1e-11)
        assert est <= O.inv_norm1_from_lu(W) * (1 + 1e-12)


def test_inv_norm_estimate_special_cases():
    W, _, _ = O.getrf(np.array([[4.0]]))
    assert O.inv_norm1_estimate(W) == 0.25                      # n = 1: |A^-1 x|
    W, _, _ = O.getrf(np.diag([2.0, 0.5, 8.0, 1.0]))
    assert O.inv_norm1_estimate(W) == 2.0                       # diagonal: exact (= max 1/|d|)
    from scipy.linalg import lapack, lu_factor
    T = np.triu(np.ones((6, 6)))          # ||T^-1||_1 = 2; the estimator stops at 17/9 (< 2)
    W, _, _ = O.getrf(T)
    rcond, _ = lapack.dgecon(lu_factor(T)[0], 6.0, norm="1")
    assert O.inv_norm1_estimate(W) == pytest.approx(1.0 / (6.0 * rcond), rel=1e-14)
    assert O.inv_norm1_estimate(W) == pytest.approx(17.0 / 9.0, rel=1e-14)
    assert O.inv_norm1_from_lu(W) == 2.0


@pytest.mark.parametrize("b,ib", [(8, 4), (32, 32), (64, 16), (50, 16), (128, 32)])
def test_geqrt_matches_lapack_dgeqrt(b, ib):
    T0 = RNG.standard_normal((b, b))
    tile = T0.copy()
    Tf = O.geqrt(tile, ib)
    a, t, info = lapack.dgeqrt(ib, T0.copy())
    assert info == 0
    assert rel(tile, a) < 1e-12  # V below the diagonal and R on/above it
    assert rel(Tf, t) < 1e-12
    # R equals numpy's QR R up to row signs
    R = np.linalg.qr(T0, mode="r")
    assert rel(np.abs(np.triu(tile)), np.abs(R)) < 1e-12


def test_unmqr_matches_dgemqrt_and_is_orthogonal():
    b, ib, nc = 64, 16, 40
    T0 = RNG.standard_normal((b, b))
    tile = T0.copy()
    Tf = O.geqrt(tile, ib)
    C = RNG.standard_normal((b, nc))
    C1 = C.copy()
    O.unmqr(tile, Tf, ib, C1)
    V = np.tril(tile, -1) + np.eye(b)
    ref, info = lapack.dgemqrt(V, Tf, C.copy(), side="L", trans="T")
    assert rel(C1, ref) < 1e-12
    # Q^T from applying to the identity: orthogonal and Q^T T0 = R
    Qt = np.eye(b)
    O.unmqr(tile, Tf, ib, Qt)
    assert np.linalg.norm(Qt @ Qt.T - np.eye(b)) < 10 * b * 2.2e-16
    assert rel(Qt @ T0, np.triu(tile)) < 1e-13


@pytest.mark.parametrize("tt", [False, True])
@pytest.mark.parametrize("b,ib", [(16, 4), (64, 32), (48, 16)])
def test_tsqrt_tsmqr_match_lapack_dtpqrt(tt, b, ib):
    R0 = np.triu(RNG.standard_normal((b, b)))
    A2 = RNG.standard_normal((b, b))
    if tt:
        low = np.tril(RNG.standard_normal((b, b)), -1)  # junk below: must be ignored and preserved
        A2 = np.triu(A2) + low
    R = R0.copy()
    B = A2.copy()
    T = O.tsqrt(R, B, ib, tt=tt)
    l = b if tt else 0
    a_ref, b_ref, t_ref, info = lapack.dtpqrt(l, ib, R0.copy(), (np.triu(A2) if tt else A2).copy())
    assert info == 0
    assert rel(np.triu(R), np.triu(a_ref)) < 1e-12
    Bv = np.triu(B) if tt else B
    assert rel(Bv, (np.triu(b_ref) if tt else b_ref)) < 1e-12
    assert rel(T, t_ref) < 1e-12
    if tt:
        np.testing.assert_array_equal(np.tril(B, -1), low)
    # TSMQR / TTMQR against dtpmqrt
    nc = 24
    C1 = RNG.standard_normal((b, nc))
    C2 = RNG.standard_normal((b, nc))
    c1, c2 = C1.copy(), C2.copy()
    O.tsmqr(B, T, ib, c1, c2, tt=tt)
    r1, r2, info = lapack.dtpmqrt(l, Bv, T, C1.copy(), C2.copy(), side="L", trans="T")
    assert rel(c1, r1) < 1e-12 and rel(c2, r2) < 1e-12
    # applying the transform to its own input annihilates the bottom tile
    c1, c2 = R0.copy(), (np.triu(A2) if tt else A2).copy()
    O.tsmqr(B, T, ib, c1, c2, tt=tt)
    assert np.linalg.norm(c2) < 1e-12 * np.linalg.norm(A2)
    assert rel(c1, np.triu(R)) < 1e-12


def test_larfg_matches_lapack():
    x = RNG.standard_normal(9)
    beta, tau, v = O.larfg(x[0], x[1:].copy())
    b2, xv, t2 = lapack.dlarfg(9, x[0], x[1:].copy())
    assert beta == pytest.approx(b2, rel=1e-14) and tau == pytest.approx(t2, rel=1e-14)
    np.testing.assert_allclose(v, xv, rtol=1e-13)
    beta, tau, v = O.larfg(3.0, np.zeros(4))
    assert tau == 0.0 and beta == 3.0


# ---------------------------------------------------------------- criteria hand values (SPEC)
def _one_step_decision(A, crit, alpha, reading=0):
    f = O.hybrid_factor(np.asfortranarray(A), 1, crit, alpha, mumps_reading=reading)
    return f.dec[0]


def test_criteria_hand_values():
    # Max, nb=1: A_kk=2, below {1}, alpha=1 -> 2 >= 1 -> LU
    A = np.array([[2.0, 0.3], [1.0, 1.7]])
    assert _one_step_decision(A, O.CRIT_MAX, 1.0) == O.LU
    # Sum stricter: A_kk=2, below {1,1,1}: Max LU, Sum 2 < 3 -> QR
    A = np.eye(4) * 2.0
    A[1:, 0] = 1.0
    assert _one_step_decision(A, O.CRIT_MAX, 1.0) == O.LU
    assert _one_step_decision(A, O.CRIT_SUM, 1.0) == O.QR
    # MUMPS nb=1: pivot 4, away 3, alpha 2.1 -> 8.4 >= 3 LU;  pivot 1, away 3 -> 2.1 < 3 QR
    for reading in (0, 1):
        A = np.array([[4.0, 0.0, 0.0], [1.0, 1.0, 0.0], [3.0, 0.0, 1.0]])
        assert _one_step_decision(A, O.CRIT_MUMPS, 2.1, reading) == O.LU
        A = np.array([[1.0, 0.0], [3.0, 1.0]])
        assert _one_step_decision(A, O.CRIT_MUMPS, 2.1, reading) == O.QR
    # alpha specials (ledger 4): alpha = 0 -> QR everywhere, alpha = inf -> LU everywhere
    A = I.uniform_matrix(7, 64)
    assert set(O.hybrid_factor(A, 16, O.CRIT_MAX, 0.0).dec) == {O.QR}
    assert set(O.hybrid_factor(A, 16, O.CRIT_MAX, math.inf).dec) == {O.LU}


def test_mumps_m1_equals_dense_formula():
    """M1 (ledger 1) algebra: with nonzero pivots, estimate(j) = away_max(j) * pivot(j)/local_max(j),
    so alpha*pivot(j) >= estimate(j)  <=>  alpha*local_max(j) >= away_max(j)."""
    for trial in range(40):
        b = 8
        T = RNG.standard_normal((b, b))
        below = RNG.standard_normal((3 * b, b)) * RNG.uniform(0.2, 3.0)
        W, _, _ = O.getrf(T)
        lm = np.max(np.abs(T), axis=0)
        am = np.max(np.abs(below), axis=0)
        alpha = RNG.uniform(0.5, 4.0)
        lu, margin = O.criterion_mumps(alpha, W, lm, am, 0)
        dense = bool(np.all(alpha * lm >= am))
        ratio = np.min(alpha * lm / am)
        if abs(ratio - 1.0) > 1e-12:
            assert lu == dense


def test_sum_implies_max_and_alpha_monotone():
    A = I.uniform_matrix(11, 96)
    for alpha in (1e3, 1e4, 3e4):
        fs = O.hybrid_factor(A, 16, O.CRIT_SUM, alpha)
        stats = fs.stats[0]
        inv = stats["inv_norm"]
        lu_sum, _ = O.criterion_max_sum(O.CRIT_SUM, alpha, inv, stats["s"])
        lu_max, _ = O.criterion_max_sum(O.CRIT_MAX, alpha, inv, stats["s"])
        assert (not lu_sum) or lu_max
        lu_big, _ = O.criterion_max_sum(O.CRIT_MAX, alpha * 2, inv, stats["s"])
        assert (not lu_max) or lu_big


# ---------------------------------------------------------------- P5: growth bounds, worst case
def _golden_rows(name):
    rows = []
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(line.split())
    return rows


@pytest.mark.parametrize("row", _golden_rows("worst_case_max.txt"))
def test_worst_case_matrix_attains_max_bound(row):
    alpha, n, nb, growth, decs = float(row[0]), int(row[1]), int(row[2]), float(row[3]), row[4]
    A = I.kron_lift(I.worst_case_max(n, alpha), nb) if nb > 1 else np.asfortranarray(
        I.worst_case_max(n, alpha))
    f = O.hybrid_factor(A, nb, O.CRIT_MAX, alpha)
    assert "".join("LQ"[d] for d in f.dec) == decs
    assert f.growth == growth  # exact: (1+alpha)^(n-1)
    assert growth == (1 + alpha) ** (n - 1)
    assert all(abs(m) < 1e-10 for m in f.margin[:-1])  # exact ties; last step vacuous


def test_block_diagonally_dominant_all_lu_and_sum_bound():
    """BDD (by columns, 1-norm) => Max and Sum with alpha >= 1 pass at every step;
    Sum with alpha = 1 bounds the growth by n."""
    n, nb = 6, 8
    N = n * nb
    A = RNG.standard_normal((N, N))
    for j in range(n):
        cj = slice(j * nb, (j + 1) * nb)
        off = sum(O.norm1(A[i * nb:(i + 1) * nb, cj]) for i in range(n) if i != j)
        A[cj, cj] = np.eye(nb) * (off + 1.0)
    A = np.asfortranarray(A)
    for crit in (O.CRIT_MAX, O.CRIT_SUM):
        f = O.hybrid_factor(A, nb, crit, 1.0)
        assert set(f.dec) == {O.LU}
        assert f.growth <= n
    # scalar diagonally dominant: growth <= 2
    Ad = RNG.standard_normal((24, 24))
    Ad += np.diag(np.sum(np.abs(Ad), axis=0) + 1.0)
    f = O.hybrid_factor(np.asfortranarray(Ad), 1, O.CRIT_SUM, 1.0)
    assert set(f.dec) == {O.LU} and f.growth <= 2.0


def _tile_norms(A, N, nb, k):
    n = O.ntiles(N, nb)
    return np.array([[O.norm1(A[O.tsl(N, nb, i), O.tsl(N, nb, j)]) for j in range(n)]
                     for i in range(n)])


def test_per_step_growth_inequalities_on_mixed_run():
    """Max: ||A_ij^(k+1)|| <= (1+alpha) max_{i'>=k} ||A_i'j^(k)|| on LU steps;
    Sum (alpha=1): sum_{i>k} ||A_ij^(k+1)|| <= sum_{i>=k} ||A_ij^(k)||;
    QR steps preserve the 2-norms of the active columns."""
    N, nb = 192, 16
    A = I.uniform_matrix(21, N)
    checks = {"lu": 0, "qr": 0}

    for crit, alpha in ((O.CRIT_MAX, 1.1e4), (O.CRIT_MAX, 3e4), (O.CRIT_SUM, 1.0)):
        def hook(k, Ab, Aa, d):
            n = O.ntiles(N, nb)
            if k + 1 >= n:
                return
            tb, ta = _tile_norms(Ab, N, nb, k), _tile_norms(Aa, N, nb, k)
            k0 = k * nb
            if d == O.LU:
                checks["lu"] += 1
                for j in range(k + 1, n):
                    if crit == O.CRIT_MAX:
                        bound = (1 + alpha) * tb[k:, j].max()
                        assert ta[k + 1:, j].max() <= bound * (1 + 1e-12)
                    else:
                        assert ta[k + 1:, j].sum() <= tb[k:, j].sum() * (1 + 1e-12)
            else:
                checks["qr"] += 1
                k1 = k0 + nb  # trailing columns: whole active column; panel: only R (V is stored below)
                np.testing.assert_allclose(np.linalg.norm(Aa[k0:, k1:], axis=0),
                                           np.linalg.norm(Ab[k0:, k1:], axis=0), rtol=1e-12)
                np.testing.assert_allclose(np.linalg.norm(np.triu(Aa[k0:k1, k0:k1]), axis=0),
                                           np.linalg.norm(Ab[k0:, k0:k1], axis=0), rtol=1e-12)
        O.hybrid_factor(A, nb, crit, alpha, on_step=hook)
    assert checks["lu"] > 0 and checks["qr"] > 0


# ---------------------------------------------------------------- P2/P3: the two extreme paths
def _restricted_pivot_ge(A, nb):
    """Independent scalar Gaussian elimination (ledger 24): pivot search at column c over rows
    c .. end of c's diagonal block; swaps on columns >= that block's start; eliminate all rows below."""
    A = np.array(A, dtype=np.float64, copy=True)
    N = A.shape[0]
    piv = np.zeros(N, dtype=np.int64)
    for c in range(N):
        blk0 = (c // nb) * nb
        blk1 = min(blk0 + nb, N)
        p = c + int(np.argmax(np.abs(A[c:blk1, c])))
        piv[c] = p
        if p != c:
            A[[c, p], blk0:] = A[[p, c], blk0:]
        A[c + 1:, c] /= A[c, c]
        A[c + 1:, c + 1:] -= np.outer(A[c + 1:, c], A[c, c + 1:])
    return A, piv


@pytest.mark.parametrize("N,nb", [(96, 32), (100, 32), (128, 16)])
def test_all_lu_path_is_restricted_pivot_gaussian_elimination(N, nb):
    A = I.uniform_matrix(3, N)
    f = O.hybrid_factor(A, nb, O.CRIT_MAX, math.inf)
    G, piv = _restricted_pivot_ge(A, nb)
    for k, ip in f.ipiv.items():
        np.testing.assert_array_equal(ip + k * nb, piv[k * nb:k * nb + len(ip)])
    assert rel(f.A, G) < 1e-11


@pytest.mark.parametrize("tree", ["greedy", "flat", "hqr2", "hqr4", "hqr16"])
@pytest.mark.parametrize("N,nb,D", [(128, 32, 1), (160, 32, 2), (150, 32, 3), (224, 16, 1)])
def test_all_qr_path_reproduces_householder_R(N, nb, D, tree):
    A, b = I.normal_system(9, N)
    f = O.hybrid_factor(A, nb, O.CRIT_MAX, 0.0, D=D, tree=tree)
    R = np.linalg.qr(A, mode="r")
    assert rel(np.abs(np.triu(f.A)), np.abs(R)) < 1e-12
    x = O.solve(f, b)
    assert rel(x, np.linalg.solve(A, b)) < 1e-10


@pytest.mark.parametrize("crit,alpha", [(O.CRIT_MAX, 1.0), (O.CRIT_MAX, 1e4), (O.CRIT_SUM, 4.0),
                                        (O.CRIT_MUMPS, 1.5), (O.CRIT_MUMPS, 4.0)])
def test_solve_matches_numpy_and_hpl3(crit, alpha):
    N, nb = 256, 32
    A, b = I.normal_system(2, N)
    f = O.hybrid_factor(A, nb, crit, alpha)
    x = O.solve(f, b)
    assert rel(x, np.linalg.solve(A, b)) < 1e-9
    assert O.hpl3(A, x, b) < 16


def test_hpl3_hand_value():
    A = 2.0 * np.eye(2)
    x = np.array([1.0, 1.0])
    d = 2.0 ** -40
    b = np.array([2.0, 2.0 + d])
    assert O.hpl3(A, x, b) == pytest.approx(d / (2.0 * 1.0 * 2.0 ** -53 * 2))


# ---------------------------------------------------------------- P4: brute force on tiny tiled matrices
def _dense_criterion(Ab, N, nb, k, crit, alpha):
    n = O.ntiles(N, nb)
    rk = O.tsl(N, nb, k)
    Akk = Ab[rk, rk]
    lhs = alpha / np.linalg.norm(np.linalg.inv(Akk), 1)
    norms = [np.linalg.norm(Ab[O.tsl(N, nb, i), rk], 1) for i in range(k + 1, n)]
    rhs = (max(norms) if crit == O.CRIT_MAX else sum(norms)) if norms else 0.0
    return lhs, rhs


@pytest.mark.parametrize("n", [2, 3])
@pytest.mark.parametrize("nb", [1, 2, 4])
def test_brute_force_all_decision_vectors(n, nb):
    N = n * nb
    A = np.asfortranarray(RNG.standard_normal((N, N)))
    b = RNG.standard_normal(N)
    xs = np.linalg.solve(A, b)
    for vec in itertools.product([0, 1], repeat=n):
        f = O.hybrid_factor(A, nb, forced=np.array(vec, dtype=np.uint8))
        # (M_n ... M_1) A = U : replay every step on A's columns
        U = O.apply_transforms(f, A)
        assert np.linalg.norm(np.tril(U, -1)) < 10 * N * 2.2e-16 * np.linalg.norm(A) * 1e3
        assert rel(np.triu(U), np.triu(f.A)) < 1e-10
        assert rel(O.solve(f, b), xs) < 1e-8
    # the criterion's decision vector is self-consistent with dense recomputation at every step
    for crit, alpha in ((O.CRIT_MAX, 1.0), (O.CRIT_MAX, 3.0), (O.CRIT_SUM, 2.0)):
        def hook(k, Ab, Aa, d):
            lhs, rhs = _dense_criterion(Ab, N, nb, k, crit, alpha)
            if abs(lhs - rhs) > 1e-9 * max(lhs, rhs):
                assert d == (O.LU if lhs >= rhs else O.QR)
        O.hybrid_factor(A, nb, crit, alpha, on_step=hook)


# ---------------------------------------------------------------- P9 ragged == padded; P8 flops
@pytest.mark.parametrize("crit,alpha", [(O.CRIT_MAX, 1.0), (O.CRIT_MAX, math.inf),
                                        (O.CRIT_MUMPS, 2.0)])
def test_ragged_equals_padded(crit, alpha):
    N, nb = 200, 64
    A = I.uniform_matrix(5, N)
    npad = O.ntiles(N, nb) * nb
    P = np.eye(npad)
    P[:N, :N] = A
    fr = O.hybrid_factor(A, nb, crit, alpha)
    fp = O.hybrid_factor(np.asfortranarray(P), nb, crit, alpha)
    np.testing.assert_array_equal(fr.dec[:-1], fp.dec[:-1])
    assert rel(fr.A[:N, :N], fp.A[:N, :N]) < 1e-12


def test_greedy_plan_structure():
    """Every row i > k is eliminated exactly once, pairs in a level are disjoint, the eliminator is
    still live, and only row k survives (SPEC trees invariants); depth = ceil(log2(m+1)) for D=1."""
    for n, k, D in ((9, 0, 1), (16, 3, 1), (17, 0, 2), (30, 5, 4), (5, 4, 1)):
        rows, ts, levels = O.qr_plan(k, n, D, "greedy")
        assert rows == list(range(k, n)) and ts == []
        live = set(range(k, n))
        for lvl in levels:
            used = [r for p in lvl for r in p]
            assert len(used) == len(set(used))
            for e, i in lvl:
                assert e in live and i in live and e < i
            for e, i in lvl:
                live.discard(i)
        assert live == {k}
        if D == 1:
            assert len(levels) == math.ceil(math.log2(n - k)) if n - k > 1 else len(levels) == 0


@pytest.mark.parametrize("a", [1, 2, 3, 4, 7, 40])
def test_hqr_plan_structure(a):
    """HQR tree with TS groups of a tiles (DESIGN reading 34): every row
    i > k is eliminated exactly once; a TS elimination has a live group head as eliminator that is
    a GEQRT row, the eliminated rows of a group follow their head in ascending order; TT levels run
    over GEQRT rows only, pairs disjoint, and only row k survives.  a = 1 is the greedy tree."""
    for n, k, D in ((9, 0, 1), (16, 3, 1), (17, 0, 2), (30, 5, 4), (5, 4, 1), (40, 0, 1)):
        rows, ts, levels = O.qr_plan(k, n, D, f"hqr{a}")
        if a == 1:
            assert (rows, ts, levels) == O.qr_plan(k, n, D, "greedy")
        live = set(range(k, n))
        for e, i in ts:
            assert e in rows and i not in rows and e < i and e % D == i % D
            assert e in live and i in live
            live.discard(i)
        assert set(rows) == live  # every non-head was killed by TS, every head is GEQRT'd
        for lvl in levels:
            used = [r for p in lvl for r in p]
            assert len(used) == len(set(used))
            for e, i in lvl:
                assert e in live and i in live and e < i
            for e, i in lvl:
                live.discard(i)
        assert live == {k}
        # group size: at most a - 1 TS eliminations per head
        from collections import Counter
        assert max(Counter(e for e, _ in ts).values(), default=0) <= a - 1


def test_table_i_sums_and_table_ii_arithmetic():
    for N, nb in ((1024, 128), (16384, 256), (32768, 256)):
        n = N // nb
        assert O.true_flops(N, nb, [0] * n) == pytest.approx(O.fake_flops(N), rel=1e-12)
        assert O.true_flops(N, nb, [1] * n) == pytest.approx(2 * O.fake_flops(N), rel=1e-12)
    for row in _golden_rows("table2.txt"):
        t, pct, fake, true = float(row[2]), float(row[3]), float(row[4]), float(row[5])
        assert O.fake_flops(20000) / t / 1e9 == pytest.approx(fake, rel=5e-3)
        if row[0].startswith("LUQR") or row[0] == "HQR":
            assert O.paper_true_flops(20000, pct / 100) / t / 1e9 == pytest.approx(true, rel=5e-3)


# ---------------------------------------------------------------- generator
def _splitmix_ref(seed, idx):
    M = (1 << 64) - 1
    g = 0x9E3779B97F4A7C15

    def mix(z):
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)
    kk = mix((seed + g) & M)
    u = mix((kk + (idx + 1) * g) & M)
    return (u >> 11) * 2.0 ** -53 - 0.5


def test_counter_generator_matches_plain_int_reference():
    idx = np.array([0, 1, 2, 12345, 2 ** 34 + 7, 131072 ** 2 + 5], dtype=np.uint64)
    got = I.uniform_counter(2, idx)
    for v, i in zip(got, idx):
        assert v == _splitmix_ref(2, int(i))
    A = I.uniform_matrix(0, 8)
    assert A[3, 5] == _splitmix_ref(0, 5 * 8 + 3)
    assert A.flags["F_CONTIGUOUS"]
    u = I.uniform_matrix(0, 256).ravel()
    assert -0.5 <= u.min() and u.max() < 0.5 and abs(u.mean()) < 0.01


# ---------------------------------------------------------------------------------------------
# NEXT f4: LU step variant A2
# ---------------------------------------------------------------------------------------------
def _a2_reconstruct(f):
    """A from the A2 all-LU factors by block elimination algebra: with A_kk = Q_k R_k,
    L~_ik = (stored L_ik) Q_k^T, U~_kk = Q_k R_k, U~_kj = Q_k (stored A_kj), A = sum_k L~_:k U~_k:."""
    N, nb, ib = f.N, f.nb, f.ib
    F = f.A
    A = np.zeros((N, N))
    for k in range(f.n):
        rk = O.tsl(N, nb, k)
        k0, k1 = rk.start, rk.stop
        Qt = np.eye(k1 - k0)
        O.unmqr(F[rk, rk], f.qr[k].T_geqrt[k], ib, Qt)  # Q_k^T, independent of the step code
        Q = Qt.T
        Lt = np.vstack([np.eye(k1 - k0), F[k1:N, k0:k1] @ Qt])
        Ut = np.hstack([Q @ np.triu(F[rk, rk]), Q @ F[k0:k1, k1:N]])
        A[k0:N, k0:N] += Lt @ Ut
    return A


@pytest.mark.parametrize("N,nb", [(384, 64), (300, 64)])
def test_a2_all_lu_is_block_elimination(N, nb):
    """alpha = inf under A2: the packed factors reassemble A (block LU with QR-factored pivots).
    Block elimination has no pivoting across tiles, so the input is made diagonally dominant
    (stable: the reassembly error is then at rounding level)."""
    A = I.uniform_matrix(0, N) + (N / 2.0) * np.eye(N)
    f = O.hybrid_factor(A, nb, O.CRIT_MAX, math.inf, lu_variant="A2")
    assert np.all(f.dec == O.LU)
    Ar = _a2_reconstruct(f)
    assert np.linalg.norm(Ar - A) / np.linalg.norm(A) < 1e-13
    b = I.uniform_rhs(0, N)
    x = O.solve(f, b)
    assert np.allclose(x, np.linalg.solve(A, b), rtol=0, atol=1e-9 * np.abs(x).max())


def test_a2_schur_complement_equals_a1():
    """The Schur complement A22 - A21 A11^-1 A12 does not depend on how A11 is factored: after an LU
    step, the A1 (GETRF) and A2 (GEQRT) trailing matrices agree to rounding."""
    A = I.normal_system(1, 512)[0]
    trail = {}

    def hook(tag):
        def on_step(k, before, after, d):
            if k == 0:
                trail[tag] = after[128:, 128:].copy()
        return on_step
    O.hybrid_factor(A, 128, O.CRIT_MAX, math.inf, on_step=hook("A1"))
    O.hybrid_factor(A, 128, O.CRIT_MAX, math.inf, lu_variant="A2", on_step=hook("A2"))
    d = np.linalg.norm(trail["A1"] - trail["A2"]) / np.linalg.norm(trail["A1"])
    assert d < 1e-12, d


@pytest.mark.parametrize("dist", ["uniform", "normal"])
def test_a2_criterion_inverse_norm_is_exact(dist):
    """||R^-1 Q^T||_1 from the in-place GEQRT factors equals ||A_kk^-1||_1 of the dense inverse."""
    A = I.uniform_matrix(5, 256) if dist == "uniform" else I.normal_system(5, 256)[0]
    W = np.array(A, order="F", copy=True)
    T, R, zp = O.a2_factor(W, 256, 128, 0, 32)
    v = O.a2_inv_norm1(W, 256, 128, 0, T, 32)
    ref = np.linalg.norm(np.linalg.inv(A[:128, :128]), 1)
    assert not zp
    assert abs(v - ref) <= 1e-11 * ref
    # MUMPS pivots |U_jj| = |R_jj| are the absolute diagonal of Householder R (numpy, up to signs)
    Rn = np.linalg.qr(A[:128, :128], mode="r")
    assert np.allclose(np.abs(np.diag(R)), np.abs(np.diag(Rn)), rtol=1e-12, atol=0)


def test_a2_qr_steps_reuse_the_diagonal_factorization():
    """A QR decision continues from the A2 GEQRT: with Max alpha = 1 (QR at every step
    but the last) the A2 factors equal A1's bit for bit except the last diagonal tile, which A2
    QR-factors (|R| = numpy's) where A1 LU-factors it."""
    N, nb = 512, 64
    A = I.uniform_matrix(0, N)
    f1 = O.hybrid_factor(A, nb, O.CRIT_MAX, 1.0)
    f2 = O.hybrid_factor(A, nb, O.CRIT_MAX, 1.0, lu_variant="A2")
    assert np.array_equal(f1.dec, f2.dec) and f1.dec[-1] == O.LU and np.all(f1.dec[:-1] == O.QR)
    last = slice(N - nb, N)
    F1, F2 = f1.A.copy(), f2.A.copy()
    F1[last, last] = 0.0
    F2[last, last] = 0.0
    assert np.array_equal(F1, F2)
    # the last tile before its factorization is the same in both runs: A1 holds its LU, A2 its QR
    Lw = np.tril(f1.A[last, last], -1) + np.eye(nb)
    S = Lw @ np.triu(f1.A[last, last])
    S = S[np.argsort(_perm_of(f1.ipiv[f1.n - 1]))]
    assert np.allclose(np.abs(np.diag(np.triu(f2.A[last, last]))),
                       np.abs(np.diag(np.linalg.qr(S, mode="r"))), rtol=1e-10, atol=0)


def _perm_of(ipiv):
    p = np.arange(len(ipiv))
    for c, r in enumerate(ipiv):
        p[[c, r]] = p[[r, c]]
    return p


# ---------------------------------------------------------------------------------------------
# NEXT f1: diagonal-domain pivoting
# ---------------------------------------------------------------------------------------------
def test_domain_pivoting_d1_is_lapack_lupp():
    """D = 1: the diagonal domain is the whole panel, every step is LU (no tile off the domain), and
    the factorization is right-looking LU with partial pivoting: pivots identical to LAPACK dgetrf
    (scipy lu_factor) and U equal to LAPACK's."""
    N, nb = 512, 64
    A = I.uniform_matrix(3, N)
    f = O.hybrid_factor(A, nb, O.CRIT_MAX, 1.0, D=1, pivot_scope="domain")
    assert np.all(f.dec == O.LU)
    lu, piv = sl.lu_factor(A)
    gpiv = np.concatenate([k * nb + f.ipiv[k] for k in range(f.n)])
    assert np.array_equal(gpiv, piv)
    U = np.triu(f.A)
    assert np.linalg.norm(U - np.triu(lu)) / np.linalg.norm(np.triu(lu)) < 1e-13
    b = I.uniform_rhs(3, N)
    assert np.allclose(O.solve(f, b), sl.lu_solve((lu, piv), b), rtol=0, atol=1e-10)


@pytest.mark.parametrize("crit,alpha", [(O.CRIT_MAX, 1.0), (O.CRIT_MAX, 1e4),
                                        (O.CRIT_SUM, 1e5), (O.CRIT_MUMPS, 2.1)])
def test_domain_pivoting_with_singleton_domains_is_tile_pivoting(crit, alpha):
    """D >= n: every domain is one tile, so diagonal-domain pivoting is tile-local pivoting."""
    N, nb = 768, 128
    A = I.normal_system(2, N)[0]
    f1 = O.hybrid_factor(A, nb, crit, alpha, D=6, pivot_scope="tile")
    f2 = O.hybrid_factor(A, nb, crit, alpha, D=6, pivot_scope="domain")
    assert np.array_equal(f1.dec, f2.dec)
    assert np.allclose(f1.margin, f2.margin, rtol=1e-13, atol=0, equal_nan=True)
    assert O.factor_diff(f2.A, f1.A) < 1e-14
    for k in f1.ipiv:
        assert np.array_equal(f1.ipiv[k], f2.ipiv[k])


def test_domain_statistics_and_pivoted_tile_by_hand():
    """3 x 3 tiles, D = 2, step 0: the domain is tiles {0, 2}; s = [||A_10||_1] (off the domain),
    local_max over tiles 0 and 2, away_max over tile 1, and the criterion's ||A_kk^-1|| is that of
    the diagonal tile after the domain's row interchanges."""
    nb, N = 8, 24
    A = I.normal_system(4, N)[0]
    s, lm, am = O.panel_stats_domain(A, N, nb, 0, 2)
    assert np.array_equal(s, [np.max(np.sum(np.abs(A[8:16, :8]), axis=0))])
    assert np.array_equal(lm, np.maximum(np.abs(A[:8, :8]).max(0), np.abs(A[16:24, :8]).max(0)))
    assert np.array_equal(am, np.abs(A[8:16, :8]).max(0))
    rows = np.r_[0:8, 16:24]
    assert np.array_equal(O.domain_rows(N, nb, 0, 2), rows)
    Wst, ipiv, zp = O.getrf_stack(A[rows, :8])
    P = np.arange(16)
    for c, p in enumerate(ipiv):
        P[[c, p]] = P[[p, c]]
    top = A[rows[P[:8]], :8]  # the diagonal tile after pivoting among the domain's tiles
    assert abs(O.inv_norm1_from_lu(Wst[:8]) - np.linalg.norm(np.linalg.inv(top), 1)) \
        <= 1e-12 * np.linalg.norm(np.linalg.inv(top), 1)
    # the stack LU is LAPACK's partial pivoting of the stacked domain
    lu, piv = sl.lu_factor(A[rows, :8])
    assert np.array_equal(ipiv, piv)


def test_domain_pivoting_mixed_run_solves_and_raises_lu_likelihood():
    """pivoting over the domain 'increases the likelihood of an LU step'.  Normal input,
    N = 1024, nb = 128, D = 2, Max alpha in the mixing range: at least as many LU steps as tile
    pivoting, and the solve is accurate."""
    N, nb = 1024, 128
    A, b = I.normal_system(1, N)
    for alpha in (3e3, 1e4, 3e4):
        ft = O.hybrid_factor(A, nb, O.CRIT_MAX, alpha, D=2, pivot_scope="tile")
        fd = O.hybrid_factor(A, nb, O.CRIT_MAX, alpha, D=2, pivot_scope="domain")
        assert np.sum(fd.dec == O.LU) >= np.sum(ft.dec == O.LU)
        assert O.hpl3(A, O.solve(fd, b), b) <= 16.0


def test_margin_hand_values():
    """ledger 21: margin = (lhs - rhs) / max(lhs, rhs).  Hand cases at nb = 1 (no rounding in the
    tile LU): lhs / rhs = 3 / 2 -> +1/3 (a /min or /(lhs+rhs) denominator would give 1/2 or 1/5),
    2 / 3 -> -1/3; MUMPS pivot 4, away 3, alpha 2.1 -> (8.4 - 3) / 8.4."""
    f = O.hybrid_factor(np.asfortranarray([[3.0, 0.0], [2.0, 1.0]]), 1, O.CRIT_MAX, 1.0)
    assert f.dec[0] == O.LU and f.margin[0] == pytest.approx(1.0 / 3.0, abs=1e-15)
    f = O.hybrid_factor(np.asfortranarray([[2.0, 0.0], [3.0, 1.0]]), 1, O.CRIT_MAX, 1.0)
    assert f.dec[0] == O.QR and f.margin[0] == pytest.approx(-1.0 / 3.0, abs=1e-15)
    # Sum: below {2, 2} against 3 -> rhs 4: (3 - 4) / 4
    A = np.asfortranarray([[3.0, 0.0, 0.0], [2.0, 1.0, 0.0], [2.0, 0.0, 1.0]])
    f = O.hybrid_factor(A, 1, O.CRIT_SUM, 1.0)
    assert f.dec[0] == O.QR and f.margin[0] == pytest.approx(-0.25, abs=1e-15)
    A = np.asfortranarray([[4.0, 0.0, 0.0], [1.0, 1.0, 0.0], [3.0, 0.0, 1.0]])
    f = O.hybrid_factor(A, 1, O.CRIT_MUMPS, 2.1)
    assert f.dec[0] == O.LU and f.margin[0] == pytest.approx((8.4 - 3.0) / 8.4, abs=1e-15)


def test_mumps_m1_m2_hand_case_nb2():
    """MUMPS readings on a 2 x 2 diagonal tile (worked by hand).  A_kk = [[2, 1], [1, 3]]: no swap,
    U = [[2, 1], [0, 2.5]], pivots (2, 2.5); local_max = (2, 3); growth_factor = (1, 2.5/3).
    Below: [[1, 4], [0.5, 1]] -> away_max = (1, 4).  alpha = 1.5 -> alpha*pivot = (3, 3.75).
    M1: estimate = away * own growth = (1, 4*2.5/3 = 10/3): 3 >= 1, 3.75 >= 10/3 -> LU,
        margin = min(2/3, (3.75 - 10/3)/3.75 = 1/9).
    M2: estimate(j) = away(j) * prod_{i<j} growth(i) = (1, 4*1 = 4): 3.75 < 4 -> QR,
        margin = min(2/3, (3.75 - 4)/4 = -1/16)."""
    A = np.zeros((4, 4))
    A[0:2, 0:2] = [[2.0, 1.0], [1.0, 3.0]]
    A[2:4, 0:2] = [[1.0, 4.0], [0.5, 1.0]]
    A[2:4, 2:4] = np.eye(2)
    A = np.asfortranarray(A)
    f1 = O.hybrid_factor(A, 2, O.CRIT_MUMPS, 1.5, mumps_reading=0)
    assert f1.dec[0] == O.LU and f1.margin[0] == pytest.approx(1.0 / 9.0, abs=1e-14)
    f2 = O.hybrid_factor(A, 2, O.CRIT_MUMPS, 1.5, mumps_reading=1)
    assert f2.dec[0] == O.QR and f2.margin[0] == pytest.approx(-1.0 / 16.0, abs=1e-14)


def test_noise_floor_variant_same_mathematics():
    """variant = 1 (reversed K-chunk Schur sums, the delta_floor run) computes the same
    factorization up to rounding: decisions and pivots identical, factors within a few ulps of
    growth-scaled noise, and not bit-identical (the summation order really differs)."""
    A = I.uniform_matrix(3, 512)
    forced = np.zeros(8, dtype=np.uint8)
    f0 = O.hybrid_factor(A, 64, forced=forced)
    f1 = O.hybrid_factor(A, 64, forced=forced, variant=1)
    for k in f0.ipiv:
        np.testing.assert_array_equal(f0.ipiv[k], f1.ipiv[k])
    d = O.factor_diff(f1.A, f0.A)
    assert 0.0 < d < 1e-9
    for scope, lu in (("domain", "A1"), ("tile", "A2")):
        g0 = O.hybrid_factor(A + 2 * np.eye(512), 64, forced=forced, D=2, pivot_scope=scope,
                             lu_variant=lu)
        g1 = O.hybrid_factor(A + 2 * np.eye(512), 64, forced=forced, D=2, pivot_scope=scope,
                             lu_variant=lu, variant=1)
        assert 0.0 < O.factor_diff(g1.A, g0.A) < 1e-11


def test_random_criterion():
    """Random criterion (P:817, P:953 alpha = 50; reading 35): the draws are the input recipe's
    counter generator (pinned to hlq_inputs' numpy implementation), LU iff 100 u_k < alpha, the
    LU share follows alpha, alpha = 0 / >= 100 give all QR / all LU, zero pivots still force QR."""
    us = np.array([O._splitmix_unit(O.RANDOM_SEED, k) for k in range(400)])
    np.testing.assert_array_equal(us, I.unit_counter(O.RANDOM_SEED, np.arange(400)))
    A = I.uniform_matrix(4, 512)
    f = O.hybrid_factor(A, 16, O.CRIT_RANDOM, 50.0)
    np.testing.assert_array_equal(f.dec == O.LU, us[:32] * 100.0 < 50.0)
    assert np.all(np.isnan(f.margin)) and not f.near_tie.any()
    assert set(O.hybrid_factor(A, 16, O.CRIT_RANDOM, 0.0).dec) == {O.QR}
    assert set(O.hybrid_factor(A, 16, O.CRIT_RANDOM, 100.0).dec) == {O.LU}
    share = np.mean(np.array([O._splitmix_unit(O.RANDOM_SEED, k) for k in range(4000)]) < 0.3)
    assert abs(share - 0.3) < 0.03
    Z = np.asfortranarray(np.eye(32))
    Z[0, 0] = 0.0  # exact zero pivot in the first tile (ledger 7): QR whatever the draw
    Z[1, 0] = 0.0
    assert O.hybrid_factor(Z, 16, O.CRIT_RANDOM, 100.0).dec[0] == O.QR


def test_larfg_small_alpha_log_is_diagnostics_only():
    """The oracle's reflector log (LARFG_LOG: |alpha| < ratio * ||(alpha, x)||, a Householder sign
    decision near its discontinuity, DESIGN reading 14) records the constructed near-zero alpha and
    changes no arithmetic."""
    rng = np.random.default_rng(5)
    N, nb = 96, 32
    A = rng.standard_normal((N, N))
    A[0, 0] = 1e-9  # the first reflector of step 0 eliminates against alpha = 1e-9
    f0 = O.hybrid_factor(A, nb, O.CRIT_MAX, 0.0)  # alpha = 0: every step QR
    O.LARFG_LOG = []
    try:
        f1 = O.hybrid_factor(A, nb, O.CRIT_MAX, 0.0)
        log = list(O.LARFG_LOG)
    finally:
        O.LARFG_LOG = None
    assert np.array_equal(f0.A, f1.A)
    assert any(k == 0 and al == 1e-9 and abs(al) < 1e-6 * nr for k, al, nr in log)


def test_noise_floor_variant2_same_mathematics():
    """variant = 2 (variant 1 plus the reflector norms of the QR panel kernels summed in reverse
    order) is the same all-QR factorization up to rounding for both trees: R and V within rounding
    noise of variant 0, not bit-identical to it nor to variant 1 (the panel rounding really
    differs), and the solve from its factors solves the system."""
    A = I.normal_system(2, 512)[0]
    b = I.uniform_rhs(7, 512)
    forced = np.ones(8, dtype=np.uint8)
    for tree in ("greedy", "hqr3"):
        f0 = O.hybrid_factor(A, 64, forced=forced, tree=tree)
        f1 = O.hybrid_factor(A, 64, forced=forced, tree=tree, variant=1)
        f2 = O.hybrid_factor(A, 64, forced=forced, tree=tree, variant=2)
        assert 0.0 < O.factor_diff(f2.A, f0.A) < 1e-11
        assert O.factor_diff(f2.A, f1.A) > 0.0
        x = O.solve(f2, b)
        assert np.linalg.norm(A @ x - b) / (np.linalg.norm(A) * np.linalg.norm(x)) < 1e-13
