"""Seeded synthetic inputs shaped like the paper's workloads (DESIGN.md §5 "input recipe").

This module is shared by the oracle-side tests and the CUDA-side tests / bench; it holds none
of the method's arithmetic (no sketching, no A, no solve) -- only data generation.

The paper's datasets (California Housing, Boston, RCV1, YearPredictionMSD) are not
available here; BASELINE.json's configs c1..c5 stand in for them (c3 is RCV1-shaped: sparse
primal, ~0.1% density).
"""

from dataclasses import dataclass, field

import numpy as np
import torch


@dataclass
class Config:
    name: str
    kind: str            # "dense" or "csr"
    n: int
    d: int
    lam: float
    sketch: str
    tau: int
    beta: float = 0.5
    gamma: float = 1.0
    tol: float = 1e-4
    max_iter: int = 100000
    subcount_k: int = 0
    col_decay: bool = False   # X = G diag(j^-1/2), j 1-based (BASELINE.json c2, c5)
    noise: float = 0.01
    nnz_per_row: int = 0
    zipf_a: float = 0.0
    extra: dict = field(default_factory=dict)


# BASELINE.json "configs", in order.
CONFIGS = {
    "c1": Config("c1", "dense", 1000, 50, 1e-2, "subsample", 10, beta=0.0, tol=0.0, max_iter=300,
                 noise=0.1),
    "c2": Config("c2", "dense", 100_000, 2000, 1e-4 * 100_000, "subsample", 200, col_decay=True),
    "c3": Config("c3", "csr", 500_000, 50_000, 1e-3, "count", 500, nnz_per_row=50),
    "c4": Config("c4", "csr", 20_000, 1_000_000, 1e-3, "subcount", 256, subcount_k=4,
                 nnz_per_row=500, zipf_a=1.1),
    "c5": Config("c5", "dense", 2_000_000, 4096, 1e-4 * 2_000_000, "subsample", 1024,
                 col_decay=True),
    # Kernel ridge stand-in (not a BASELINE.json config): California-Housing-shaped
    # (n = 20640, d = 8), Gaussian kernel with the median-distance bandwidth
    # sigma^2 = E||x - x'||^2 / 2 = d, subsample tau = m / 20.
    "k1": Config("k1", "kernel", 20_640, 8, 1e-3, "subsample", 1032, noise=0.1,
                 extra={"sigma": 8 ** 0.5}),
}


def dense_problem(n, d, seed=0, col_decay=False, noise=0.01, device="cpu"):
    """X (n x d, float64, row-major), y = X w* + noise * N(0,1), w* ~ N(0,1).

    Entries of X are N(0,1), times j^{-1/2} for column j (1-based) when col_decay.
    Generated with torch's seeded generator on `device` (CPU or CUDA)."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    X = torch.randn(n, d, generator=g, dtype=torch.float64, device=device)
    if col_decay:
        scale = 1.0 / torch.sqrt(torch.arange(1, d + 1, dtype=torch.float64, device=device))
        X.mul_(scale)
    w_star = torch.randn(d, generator=g, dtype=torch.float64, device=device)
    y = X @ w_star + noise * torch.randn(n, generator=g, dtype=torch.float64, device=device)
    return X, y


def csr_uniform(n, d, nnz_per_row, seed=0, unit_rows=True):
    """CSR with ~nnz_per_row uniform distinct column positions per row (sorted), values N(0,1),
    each row normalised to unit l2 norm; y ~ N(0,1).  (BASELINE.json c3.)

    Returns (rowptr int64[n+1], colidx int32[nnz], vals float64[nnz], y float64[n])."""
    rng = np.random.default_rng(seed)
    k = min(nnz_per_row, d)
    cols = np.sort(rng.integers(0, d, size=(n, k), dtype=np.int64), axis=1)
    keep = np.ones_like(cols, dtype=bool)
    keep[:, 1:] = cols[:, 1:] != cols[:, :-1]
    counts = keep.sum(axis=1)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    colidx = cols[keep].astype(np.int32)
    vals = rng.standard_normal(colidx.shape[0])
    if unit_rows:
        sq = np.add.reduceat(vals * vals, rowptr[:-1]) if n > 0 else np.zeros(0)
        sq[counts == 0] = 1.0
        vals /= np.repeat(np.sqrt(sq), counts)
    y = rng.standard_normal(n)
    return rowptr, colidx, vals, y


def csr_zipf(n, d, nnz_per_row, a=1.1, seed=0):
    """CSR whose column popularity is Zipf(a): per row, column ranks are drawn from Zipf(a)
    truncated to [1, d] until nnz_per_row distinct ranks are found; rank -> column through a
    seeded permutation; values N(0,1); y ~ N(0,1).  (BASELINE.json c4.)"""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(d).astype(np.int64)
    k = min(nnz_per_row, d)
    rows = []
    batch = max(2 * k, 64)
    for _ in range(n):
        got = np.empty(0, dtype=np.int64)
        while got.shape[0] < k:
            z = rng.zipf(a, size=batch)
            z = z[z <= d]
            cand = np.concatenate([got, z])
            _, first = np.unique(cand, return_index=True)
            got = cand[np.sort(first)]
        rows.append(np.sort(perm[got[:k] - 1]))
    counts = np.array([r.shape[0] for r in rows], dtype=np.int64)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    colidx = np.concatenate(rows).astype(np.int32) if n else np.zeros(0, np.int32)
    vals = rng.standard_normal(colidx.shape[0])
    y = rng.standard_normal(n)
    return rowptr, colidx, vals, y


def csr_to_scipy(rowptr, colidx, vals, n, d):
    import scipy.sparse as sp
    return sp.csr_matrix((vals, colidx, rowptr), shape=(n, d))


def kernel_problem(n, d, seed=0, noise=0.1):
    """Inputs for the kernel ridge route: X ~ N(0,1) (n x d), y = sin(X w*) + noise N(0,1),
    w* ~ N(0, 1/d) (a smooth nonlinear target the Gaussian kernel can fit)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    w = rng.standard_normal(d) / np.sqrt(d)
    y = np.sin(X @ w) + noise * rng.standard_normal(n)
    return X, y
