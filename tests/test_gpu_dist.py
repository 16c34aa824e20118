"""GPU parity of the 2D block-cyclic path (row e): hlq_factor_dist on an EMULATED P x Q grid (all
ranks in this process on one B200; the collectives become device copies, the kernels are the
multi-GPU ones) vs the CPU oracle with the same QR-tree domains D (reading 16).

Bar as in test_gpu_parity.py: identical decision vectors (near ties take the oracle's decision),
normwise factor difference <= 1e-10, growth within 1e-10 relative, HPL3 <= 16; and the distributed
factors equal the single-GPU factors with the same D to rounding.
"""
import math

import numpy as np
import pytest

import hlq_inputs as I
from oracle import hlq_oracle as O
from test_gpu_parity import check_decision_record, hint_kwargs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def H():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1401_5522_b200 as H
    return H


def run_dist(H, A, b, nb, P, Q, crit=O.CRIT_MAX, alpha=1.0, D=None, forced=None, fo=None,
             pivot_scope="tile"):
    N = A.shape[0]
    D = P if D is None else D
    if fo is None:
        pre = {}

        def hook(k, Ab, Aa, d):
            sl = O.tsl(N, nb, k)
            pre[k] = Ab[sl, sl].copy()
        fo = O.hybrid_factor(A, nb, crit, alpha, D=D, forced=forced, on_step=hook,
                             pivot_scope=pivot_scope)
        fo.pre_tiles = pre
    grid = H.grid_local(P, Q)
    locs = []
    for (p, q) in grid.ranks():
        L = H.scatter_block_cyclic(A, nb, P, Q, p, q)
        locs.append(H.to_colmajor(L) if L.size else torch.zeros(0, dtype=torch.float64,
                                                                 device="cuda"))
    kw = dict(tree_domains=D)
    if pivot_scope == "domain":
        kw["pivot_scope"] = H.PIVOT_DOMAIN
    if forced is not None:
        f = H.hlq_factor_dist(grid, locs, N, nb, crit, alpha, forced=forced, **kw)
        fo.hinted_run, fo.forced_run = False, True
    else:
        hk = hint_kwargs(fo)  # the oracle's decisions only where it has a near tie
        f = H.hlq_factor_dist(grid, locs, N, nb, crit, alpha, **hk, **kw)
        fo.hinted_run, fo.forced_run = bool(hk), False
    db = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    x = f.solve(db).cpu().numpy()
    F = H.gather_block_cyclic(
        {pq: (H.from_colmajor(t) if t.numel() else np.zeros((0, 0)))
         for pq, t in zip(grid.ranks(), locs)}, N, nb, P, Q)
    return fo, f, F, x


def check(fo, f, F, x, A, b, tol=1e-10):
    np.testing.assert_array_equal(f.decisions(), fo.dec)
    diff = O.factor_diff(F, fo.A)
    check_decision_record(fo, f, getattr(fo, "hinted_run", False),
                          forced=getattr(fo, "forced_run", False), diff=diff)
    assert diff <= tol, f"factor diff {diff:.3e}"
    assert f.growth() == pytest.approx(fo.growth, rel=1e-10)
    h3 = O.hpl3(A, x, b)
    assert h3 <= 16.0, h3
    xo = O.solve(fo, b)
    assert np.linalg.norm(x - xo) <= 1e-8 * max(1.0, np.linalg.norm(xo))
    return diff


@pytest.mark.parametrize("P,Q", [(1, 2), (2, 1), (2, 2), (2, 3)])
@pytest.mark.parametrize("alpha", [1.0, math.inf, 1.2e4])
def test_grid_max_criterion(H, P, Q, alpha):
    N, nb = 1000, 64                       # 16 tiles, ragged last tile of 40
    A = I.uniform_matrix(0, N)
    b = I.uniform_rhs(0, N)
    fo, f, F, x = run_dist(H, A, b, nb, P, Q, alpha=alpha)
    check(fo, f, F, x, A, b)


@pytest.mark.parametrize("P,Q,D", [(1, 1, 2), (1, 2, 2), (2, 2, 4), (2, 1, 2)])
def test_grid_domains_match_single_gpu(H, P, Q, D):
    """C5 fixes D = 2 on every grid so that all grids compute the same factorization."""
    N, nb = 768, 64
    A = I.uniform_matrix(2, N)
    b = I.uniform_rhs(2, N)
    fo, f, F, x = run_dist(H, A, b, nb, P, Q, alpha=1.0, D=D)
    check(fo, f, F, x, A, b)
    dA = H.to_colmajor(A)
    fs = H.hlq_factor_ex(dA, N, nb, O.CRIT_MAX, 1.0, tree_domains=D, **hint_kwargs(fo))
    np.testing.assert_array_equal(fs.decisions(), f.decisions())
    assert O.factor_diff(F, H.from_colmajor(dA)) <= 1e-13


@pytest.mark.parametrize("P,Q,D,crit,alpha", [
    (2, 1, 2, O.CRIT_MAX, 300.0), (2, 2, 2, O.CRIT_MAX, 300.0), (1, 2, 2, O.CRIT_MAX, 300.0),
    (2, 3, 4, O.CRIT_MAX, 300.0), (2, 2, 2, O.CRIT_MUMPS, 2.1), (2, 1, 2, O.CRIT_MAX, math.inf),
    (1, 1, 1, O.CRIT_MAX, math.inf)])
def test_grid_domain_pivoting(H, P, Q, D, crit, alpha):
    """NEXT f1 on the 2D grid (reading 33): the diagonal domain (tiles i = k mod D, P | D)
    lives on one process row, so the stacked partial-pivoting LU, the domain statistics and the
    domain's row interchanges are rank-local; the pivots travel in the panel package.  Against the
    oracle's domain-pivoting run and the single-GPU domain-pivoting path (same kernels)."""
    N, nb = 1000, 64                       # 16 tiles, ragged last tile of 40
    A = I.uniform_matrix(2, N)
    b = I.uniform_rhs(2, N)
    fo, f, F, x = run_dist(H, A, b, nb, P, Q, crit=crit, alpha=alpha, D=D, pivot_scope="domain")
    check(fo, f, F, x, A, b)
    if P == 1 and Q == 1 and D == 1:      # D = 1: LU with partial pivoting over the whole panel
        assert (fo.dec == 0).all()
    dA = H.to_colmajor(A)
    fs = H.hlq_factor_ex(dA, N, nb, crit, alpha, tree_domains=D, pivot_scope=H.PIVOT_DOMAIN,
                         **hint_kwargs(fo))
    np.testing.assert_array_equal(fs.decisions(), f.decisions())
    assert O.factor_diff(F, H.from_colmajor(dA)) <= 1e-13


@pytest.mark.parametrize("f_qr", [0.0, 0.5, 1.0])
def test_grid_forced_patterns(H, f_qr):
    N, nb = 1024, 128
    A = I.uniform_matrix(3, N)
    b = I.uniform_rhs(3, N)
    forced = I.bernoulli_pattern(30, N // nb, f_qr)
    fo, f, F, x = run_dist(H, A, b, nb, 2, 2, forced=forced)
    check(fo, f, F, x, A, b)


@pytest.mark.parametrize("crit,alpha", [(O.CRIT_SUM, 1e6), (O.CRIT_MUMPS, 4.0), (O.CRIT_MUMPS, 1.0)])
def test_grid_other_criteria(H, crit, alpha):
    N, nb = 768, 64
    A, b = I.normal_system(1, N)
    fo, f, F, x = run_dist(H, A, b, nb, 2, 2, crit=crit, alpha=alpha)
    check(fo, f, F, x, A, b)


@pytest.mark.parametrize("N,nb,P,Q", [(100, 128, 2, 2), (300, 64, 2, 3), (129, 64, 2, 2),
                                      (1000, 320, 2, 2), (1000, 320, 1, 2)])
def test_grid_degenerate_sizes(H, N, nb, P, Q):
    """n = 1 (ranks with empty local arrays), fewer tile rows than process rows, ragged 1-row tile."""
    A = I.uniform_matrix(0, N)
    b = I.uniform_rhs(0, N)
    fo, f, F, x = run_dist(H, A, b, nb, P, Q, alpha=1.2e4)
    check(fo, f, F, x, A, b)


def test_grid_kronecker_worst_case(H):
    """P:525-532 lifted to A_alpha (x) I_nb: every decision an exact tie (LU), growth 128."""
    nb, n = 64, 8
    A = np.ascontiguousarray(I.kron_lift(I.worst_case_max(n, 1.0), nb))
    N = A.shape[0]
    b = I.uniform_rhs(0, N)
    fo, f, F, x = run_dist(H, A, b, nb, 2, 2, alpha=1.0, D=2)
    assert f.growth() == 128.0
    np.testing.assert_array_equal(f.decisions(), np.zeros(n, dtype=np.uint8))
    assert O.factor_diff(F, fo.A) == 0.0


def test_cyclic_generator_bit_identical(H):
    """Each rank generates only its own tiles of the seeded global matrix (C5 recipe)."""
    N, nb, P, Q = 1000, 64, 2, 3
    grid = H.grid_local(P, Q)
    locs = []
    for (p, q) in grid.ranks():
        m, n = H.local_shape(N, nb, P, Q, p, q)
        locs.append(torch.empty(m * n, dtype=torch.float64, device="cuda"))
    H.hlq_generate_uniform_cyclic(grid, locs, N, nb, 2)
    torch.cuda.synchronize()
    got = H.gather_block_cyclic(
        {pq: t.cpu().numpy().reshape(H.local_shape(N, nb, P, Q, *pq)[1], -1).T
         for pq, t in zip(grid.ranks(), locs)}, N, nb, P, Q)
    np.testing.assert_array_equal(got, I.uniform_matrix(2, N))


def test_distributed_residual_matches_host(H):
    N, nb, P, Q = 700, 64, 2, 2
    A = I.uniform_matrix(4, N)
    b = I.uniform_rhs(4, N)
    x = np.linalg.solve(A, b)
    grid = H.grid_local(P, Q)
    locs = [H.to_colmajor(H.scatter_block_cyclic(A, nb, P, Q, p, q)) for (p, q) in grid.ranks()]
    dx = torch.from_numpy(x).cuda()
    db = torch.from_numpy(b).cuda()
    r = H.hlq_residual_dist(grid, locs, N, nb, dx, db)
    assert r["A_inf"] == pytest.approx(np.abs(A).sum(axis=1).max(), rel=1e-14)
    assert r["x_inf"] == np.abs(x).max()
    assert r["resid_inf"] == pytest.approx(np.abs(A @ x - b).max(), rel=0.5, abs=1e-15)
    assert r["hpl3"] == pytest.approx(O.hpl3(A, x, b), rel=0.5, abs=1e-3)


def test_nccl_grid_single_rank(H):
    """The NCCL plumbing (unique id, CommInitRank, row/column CommSplit, AllGather, Broadcast,
    AllReduce) on a real 1 x 1 communicator gives the emulated grid's factorization."""
    N, nb = 768, 64
    A = I.uniform_matrix(0, N)
    b = I.uniform_rhs(0, N)
    fo = O.hybrid_factor(A, nb, O.CRIT_MAX, 1.2e4, D=2)
    uid = H.nccl_unique_id()
    grid = H.grid_nccl(uid, 1, 0, 1, 1)
    dA = H.to_colmajor(A)
    f = H.hlq_factor_dist(grid, [dA], N, nb, O.CRIT_MAX, 1.2e4, tree_domains=2,
                          **hint_kwargs(fo))
    db = torch.from_numpy(b).cuda()
    x = f.solve(db).cpu().numpy()
    check(fo, f, H.from_colmajor(dA), x, A, b)
    f.free()
    grid.free()
