"""Seeded synthetic inputs for the hybrid LU-QR hot path (shared by the oracle and the GPU tests).

This module holds NONE of the method's arithmetic: it only draws numbers and assembles the
BASELINE.json input matrices (configs C1-C5).  Both the oracle
(`oracle/`) and the product path consume these arrays; neither side imports the other.

Counter-based uniform generator G_u (SURVEY §8d "Generators"): a SplitMix64 finalizer of
(key(seed) + (idx+1)*GAMMA) mod 2^64, mapped to [-0.5, 0.5) as (u >> 11) * 2^-53 - 0.5.
It is integer-only, so the CUDA library implements the same function bit-identically
(`hlq_generate_uniform` in include/hlq.h) for matrices too large to build on the host (C5).
Indexing: A(i, j) -> idx = j*N + i (0-based, column-major); b(i) -> idx = N*N + i.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_S30, _S27, _S31, _S11 = np.uint64(30), np.uint64(27), np.uint64(31), np.uint64(11)
TWO_M53 = 2.0 ** -53


def _mix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finalizer on uint64 arrays (wrap-around arithmetic)."""
    z = (z ^ (z >> _S30)) * _M1
    z = (z ^ (z >> _S27)) * _M2
    return z ^ (z >> _S31)


def key(seed: int) -> np.uint64:
    with np.errstate(over="ignore"):
        return _mix64(np.array([np.uint64(seed) + GAMMA], dtype=np.uint64))[0]


def uniform_counter(seed: int, idx: np.ndarray) -> np.ndarray:
    """G_u(seed, idx) in [-0.5, 0.5): bit-identical to the device generator."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = key(seed) + (idx + np.uint64(1)) * GAMMA
        u = _mix64(z)
    return (u >> _S11).astype(np.float64) * TWO_M53 - 0.5


def unit_counter(seed: int, idx: np.ndarray) -> np.ndarray:
    """Same stream mapped to [0, 1) (used for the seeded Bernoulli decision pattern, C3)."""
    return uniform_counter(seed, idx) + 0.5


def uniform_matrix(seed: int, N: int) -> np.ndarray:
    """A(i,j) = G_u(seed, j*N+i) as a Fortran-ordered (column-major) float64 array."""
    j, i = np.meshgrid(np.arange(N, dtype=np.uint64), np.arange(N, dtype=np.uint64))
    return np.asfortranarray(uniform_counter(seed, j * np.uint64(N) + i))


def uniform_rhs(seed: int, N: int) -> np.ndarray:
    return uniform_counter(seed, np.uint64(N) * np.uint64(N) + np.arange(N, dtype=np.uint64))


def normal_system(seed: int, N: int):
    """G_n(seed): numpy default_rng(seed); A = standard_normal((N,N)) (C order draw), then b."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((N, N))
    b = rng.standard_normal(N)
    return np.asfortranarray(A), b


def wilkinson_type(N: int) -> np.ndarray:
    """C4(a): 1 on the diagonal, -1 strictly below, 1 in the last column."""
    A = np.tril(-np.ones((N, N)), -1) + np.eye(N)
    A[:, -1] = 1.0
    return np.asfortranarray(A)


def worst_case_max(n: int, alpha: float) -> np.ndarray:
    """The n x n generalisation of PAPER.md:525-532 (Max-criterion worst case):
    alpha^-1 on the diagonal, -1 strictly below, 1 in the last column (last diagonal entry 1)."""
    A = np.tril(-np.ones((n, n)), -1) + np.eye(n) / alpha
    A[:, -1] = 1.0
    return A


def kron_lift(A: np.ndarray, nb: int) -> np.ndarray:
    """A (x) I_nb: every scalar becomes an nb x nb scaled identity tile."""
    return np.asfortranarray(np.kron(A, np.eye(nb)))


def bernoulli_pattern(seed: int, n: int, f: float) -> np.ndarray:
    """C3 forced decisions: d_k = QR (1) iff U(seed, k) < f, U from the counter stream in [0,1)."""
    if f <= 0.0:
        return np.zeros(n, dtype=np.uint8)
    if f >= 1.0:
        return np.ones(n, dtype=np.uint8)
    u = unit_counter(seed, np.arange(n, dtype=np.uint64))
    return (u < f).astype(np.uint8)


# Special matrices of the paper's stability study (Table III) -- ONLY those the paper
# itself defines by a formula (the rest of Higham's toolbox is not reproduced).  1-based i, j as in
# the paper; random ingredients drawn from numpy default_rng(seed).  NEXT f3.
SPECIAL_BY_FORMULA = ("house", "parter", "ris", "hankel", "compan", "lehmer", "demmel", "hilb",
                      "lotkin", "orthogo")


def special_matrix(name: str, n: int, seed: int = 7) -> np.ndarray:
    i = np.arange(1, n + 1, dtype=np.float64)[:, None]
    j = np.arange(1, n + 1, dtype=np.float64)[None, :]
    rng = np.random.default_rng(seed)
    if name == "house":      # A = eye(n) - beta*v*v'; v ~ randn, beta = 2/(v'v) (reading 31)
        v = rng.standard_normal(n)
        A = np.eye(n) - (2.0 / float(v @ v)) * np.outer(v, v)
    elif name == "parter":   # A(i,j) = 1/(i - j + 0.5)
        A = 1.0 / (i - j + 0.5)
    elif name == "ris":      # A(i,j) = 0.5/(n - i - j + 1.5)
        A = 0.5 / (n - i - j + 1.5)
    elif name == "hankel":   # hankel(c, r), c, r = randn(n,1), c(n) = r(1)
        c = rng.standard_normal(n)
        r = rng.standard_normal(n)
        c[-1] = r[0]
        s_ = (i + j - 1).astype(np.int64)   # A(i,j) = c(i+j-1) if i+j-1 <= n else r(i+j-n)
        A = np.where(s_ <= n, c[np.minimum(s_, n) - 1], r[np.clip(s_ - n, 1, n) - 1])
    elif name == "compan":   # compan(randn(n+1,1)): first row -p(2:)/p(1), ones below the diagonal
        p = rng.standard_normal(n + 1)
        A = np.diag(np.ones(n - 1), -1)
        A[0, :] = -p[1:] / p[0]
    elif name == "lehmer":   # A(i,j) = i/j for j >= i, symmetric
        A = np.minimum(i, j) / np.maximum(i, j)
    elif name == "demmel":   # D*(eye(n) + 1e-7*rand(n)), D = diag(10^(14*(0:n-1)/n)) (ledger 29)
        D = 10.0 ** (14.0 * np.arange(n) / n)
        A = D[:, None] * (np.eye(n) + 1e-7 * rng.random((n, n)))
    elif name == "hilb":     # 1/(i + j - 1)
        A = 1.0 / (i + j - 1)
    elif name == "lotkin":   # the Hilbert matrix with its first row all ones
        A = 1.0 / (i + j - 1)
        A[0, :] = 1.0
    elif name == "orthogo":  # sqrt(2/(n+1)) sin(i j pi/(n+1))
        A = np.sqrt(2.0 / (n + 1)) * np.sin(i * j * np.pi / (n + 1))
    else:
        raise ValueError(f"special matrix {name!r} is not defined by a formula in the paper")
    return np.asfortranarray(A)


def config_system(name: str, N: int | None = None):
    """Return (A, b, meta) for a named BASELINE config at its size (or an override N).

    C1: N=1024, U[-.5,.5] from seed 0;  C2: N=16384 normal seed 1;  C3: N=32768 uniform seed 3;
    C4a/b/c: N=4096 Wilkinson-type / +1e-6 noise (seed 4) / normal seed 5 with i>j tiles x1e3;
    C5: N=131072 uniform seed 2 (built on the device by the product path; host build only for small N).
    """
    name = name.upper()
    if name == "C1":
        N = N or 1024
        return uniform_matrix(0, N), uniform_rhs(0, N), {"nb": 128}
    if name == "C2":
        N = N or 16384
        A, b = normal_system(1, N)
        return A, b, {"nb": 256}
    if name == "C3":
        N = N or 32768
        return uniform_matrix(3, N), uniform_rhs(3, N), {"nb": 256}
    if name == "C4A":
        N = N or 4096
        return wilkinson_type(N), uniform_rhs(6, N), {"nb": 128}
    if name == "C4B":
        N = N or 4096
        A = wilkinson_type(N) + 1e-6 * 2.0 * uniform_matrix(4, N)
        return np.asfortranarray(A), uniform_rhs(6, N), {"nb": 128}
    if name == "C4C":
        N = N or 4096
        nb = 128
        A, b = normal_system(5, N)
        for i in range(0, N, nb):
            for j in range(0, i, nb):
                A[i:i + nb, j:j + nb] *= 1e3
        return A, b, {"nb": nb}
    if name == "C5":
        N = N or 131072
        return uniform_matrix(2, N), uniform_rhs(2, N), {"nb": 320}
    raise ValueError(f"unknown config {name}")
