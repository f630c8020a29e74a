"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no factorizations, no Sturm
counts, no eigen-anything): it only builds the tridiagonal inputs (d, e) of the
BASELINE.json configs and of the small test families. Both `oracle/` and the
product path consume its outputs; neither is imported from here.

BASELINE.json configs (BJ:7-11; concrete recipes in SURVEY.md 8(d) table and
DESIGN.md "Input recipe"):
  1  1-2-1 Toeplitz, n=1000, d=2, e=1, fp64, range A
  2  random, n=4000, d,e ~ U[-1,1] (PCG64 seed), fp64, range A
  3  glued Wilkinson W21 x 200 with glue 2^-26, n=4200, fp64, range A
  4  random, n=20000, fp32, d~N(0,1), e~|N(0,1)|, range I il=1..iu=2000
  5  Legendre-type, n=50000, d=0, e_k=k/sqrt(4k^2-1), fp64, range A
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GLUE = 2.0 ** -26  # sqrt(eps_fp64) exactly (BJ:9 "sqrt(eps_fp64)=1.49e-8")


@dataclass
class Problem:
    name: str
    d: np.ndarray          # diagonal, float64 or float32
    e: np.ndarray          # off-diagonal (n-1), same dtype
    range: str = "A"       # 'A' all, 'I' index range, 'V' value range
    il: int = 1
    iu: int = 0
    vl: float = 0.0
    vu: float = 0.0

    @property
    def n(self) -> int:
        return int(self.d.shape[0])

    @property
    def io(self) -> str:
        return "f32" if self.d.dtype == np.float32 else "f64"

    def index_range(self):
        """1-based inclusive index range requested (for 'A' and 'I')."""
        if self.range == "A":
            return 1, self.n
        if self.range == "I":
            return self.il, self.iu
        raise ValueError("index_range undefined for range 'V'")


def one_two_one(n: int) -> Problem:
    """Config 1 (BJ:7): d_i = 2, e_i = 1."""
    return Problem("1-2-1", np.full(n, 2.0), np.ones(max(n - 1, 0)))


def random_uniform(n: int, seed: int = 0) -> Problem:
    """Config 2 (BJ:8): d then e drawn U[-1,1] from numpy PCG64(seed)."""
    rng = np.random.default_rng(seed)
    d = rng.uniform(-1.0, 1.0, n)
    e = rng.uniform(-1.0, 1.0, max(n - 1, 0))
    return Problem(f"random-u{seed}", d, e)


def wilkinson_block(m: int = 21) -> tuple[np.ndarray, np.ndarray]:
    """W_m^+ : d_k = |(m-1)/2 - k|, k = 0..m-1, unit off-diagonal."""
    h = (m - 1) // 2
    d = np.abs(h - np.arange(m)).astype(np.float64)
    return d, np.ones(m - 1)


def glued_wilkinson(copies: int = 200, m: int = 21, glue: float = GLUE) -> Problem:
    """Config 3 (BJ:9): `copies` W21 blocks, glued by `glue` at e[m*k-1], k=1..copies-1."""
    db, eb = wilkinson_block(m)
    n = copies * m
    d = np.tile(db, copies)
    e = np.empty(n - 1)
    for k in range(copies):
        e[k * m:k * m + m - 1] = eb
        if k + 1 < copies:
            e[k * m + m - 1] = glue
    return Problem(f"glued-W{m}x{copies}", d, e)


def random_normal_f32(n: int = 20000, seed: int = 0, il: int = 1, iu: int = 2000) -> Problem:
    """Config 4 (BJ:10): d = f32(N(0,1)), then e = f32(|N(0,1)|), PCG64(seed); range I."""
    rng = np.random.default_rng(seed)
    d = rng.standard_normal(n).astype(np.float32)
    e = np.abs(rng.standard_normal(max(n - 1, 0))).astype(np.float32)
    return Problem(f"random-n{seed}-f32", d, e, range="I", il=il, iu=min(iu, n))


def legendre(n: int = 50000) -> Problem:
    """Config 5 (BJ:11): d = 0, e_k = k/sqrt(4k^2-1), k = 1..n-1, rounded to fp64."""
    k = np.arange(1, n, dtype=np.float64)
    return Problem("legendre", np.zeros(n), k / np.sqrt(4.0 * k * k - 1.0))


def clement(n: int) -> Problem:
    """Clement/Kac matrix: d = 0, e_k = sqrt(k(n-k)); spectrum +-(n-1), +-(n-3), ..."""
    k = np.arange(1, n, dtype=np.float64)
    return Problem("clement", np.zeros(n), np.sqrt(k * (n - k)))


def random_small(n: int, seed: int, kind: str = "uniform") -> Problem:
    """Small seeded matrices for brute-force and parity tests."""
    rng = np.random.default_rng(1000 + seed)
    if kind == "uniform":
        d = rng.uniform(-1.0, 1.0, n)
        e = rng.uniform(-1.0, 1.0, max(n - 1, 0))
    elif kind == "graded":  # entries spanning many orders of magnitude
        d = rng.uniform(-1.0, 1.0, n) * 10.0 ** rng.uniform(-6, 0, n)
        e = rng.uniform(0.1, 1.0, max(n - 1, 0)) * 10.0 ** rng.uniform(-6, 0, max(n - 1, 0))
    elif kind == "integer":
        d = rng.integers(-4, 5, n).astype(np.float64)
        e = rng.integers(1, 4, max(n - 1, 0)).astype(np.float64)
    else:
        raise ValueError(kind)
    return Problem(f"small-{kind}-{seed}", d, e)


def split_matrix(n: int, seed: int, split_at=(None,)) -> Problem:
    """Random matrix with some exact zero off-diagonals (preprocessing split path)."""
    p = random_small(n, seed)
    e = p.e.copy()
    for s in split_at:
        if s is None:
            s = n // 2
        if 0 <= s < n - 1:
            e[s] = 0.0
    return Problem(f"split-{seed}", p.d, e)


CONFIGS = {
    1: lambda: one_two_one(1000),
    2: lambda: random_uniform(4000, 0),
    3: lambda: glued_wilkinson(200, 21),
    4: lambda: random_normal_f32(20000, 0, 1, 2000),
    5: lambda: legendre(50000),
}


def config(k: int) -> Problem:
    return CONFIGS[k]()


@dataclass
class DenseProblem:
    """Dense symmetric input A = Q T Q^T of the paper's dense experiments (PAPER.md L1529-L1531:
    "applying random orthogonal similarity transformations to the tridiagonal matrices of the
    previous experiments"); t is the tridiagonal source, kept for reference only."""
    name: str
    A: np.ndarray          # n x n float64, exactly symmetric, column-major (Fortran order)
    t: Problem

    @property
    def n(self) -> int:
        return int(self.A.shape[0])


def random_orthogonal(n: int, seed: int) -> np.ndarray:
    """Haar-random orthogonal matrix: Q of the QR factorization of a Gaussian matrix with the
    signs of diag(R) folded in (input generation only)."""
    rng = np.random.default_rng(7000 + seed)
    G = rng.standard_normal((n, n))
    Q, R = np.linalg.qr(G)
    return Q * np.sign(np.diag(R))[None, :]


def dense_from(t: Problem, seed: int = 0) -> DenseProblem:
    """A = Q T Q^T, symmetrised exactly ((A + A^T) / 2), float64, column-major."""
    n = t.n
    Q = random_orthogonal(n, seed)
    T = np.diag(t.d.astype(np.float64))
    if n > 1:
        T += np.diag(t.e.astype(np.float64), 1) + np.diag(t.e.astype(np.float64), -1)
    A = Q @ T @ Q.T
    A = 0.5 * (A + A.T)
    return DenseProblem(f"dense-{t.name}", np.asfortranarray(A), t)


def dense_config(n: int = 4096, seed: int = 0) -> DenseProblem:
    """NEXT-4 bench workload: A = Q T Q^T with T the config-2 recipe (random uniform) of size n."""
    return dense_from(random_uniform(n, seed), seed)
