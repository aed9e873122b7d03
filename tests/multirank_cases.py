"""Problem cases of the multi-rank tests (tests/test_gpu_multirank.py, tests/multirank_worker.py):
small enough for the oracle, with several GEMM tiles / CSR rows per rank and ragged shards."""
import numpy as np

import rsinputs


def csr_column_block(rowptr, colidx, vals, c0, clen):
    """Columns [c0, c0 + clen) of a CSR matrix, with local column indices (dual feature shard)."""
    keep = (colidx >= c0) & (colidx < c0 + clen)
    ck = np.concatenate([[0], np.cumsum(keep, dtype=np.int64)])
    return ck[rowptr].astype(np.int64), (colidx[keep] - c0).astype(np.int32), vals[keep]


def _csr_primal():
    return rsinputs.csr_uniform(3001, 400, 14, seed=4)


def _csr_dual():
    return rsinputs.csr_zipf(300, 5000, 40, a=1.1, seed=6)


CASES = {
    # dense primal, row shards: the per-iteration allreduce of u (GRAM), of A S (IMPLICIT), the
    # group Grams (GRAM sketch-ahead), b and A (EXPLICIT setup)
    "dense_gram": dict(data="dense", n=4001, d=301, lam=0.4, mode="gram", kind="subsample", tau=37,
                       iters=14, seed=3, sseed=5, check_every=5),
    "dense_implicit": dict(data="dense", n=4001, d=301, lam=0.4, mode="implicit", kind="count", tau=40,
                           iters=12, seed=3, sseed=6),
    "dense_explicit": dict(data="dense", n=4001, d=301, lam=0.4, mode="explicit", kind="subcount",
                           tau=30, k=3, iters=12, seed=3, sseed=7),
    "dense_explicit_big": dict(data="dense", n=4001, d=601, lam=0.4, mode="explicit", kind="subsample",
                               tau=260, iters=10, seed=3, sseed=8),
    # dense dual (n < d) through R = X^T: feature shards of X are row shards of R
    "dense_dual_gram": dict(data="dense", n=300, d=1201, lam=0.5, mode="gram", kind="subsample", tau=40,
                            iters=12, seed=5, sseed=3, dual=True),
    "dense_dual_implicit": dict(data="dense", n=300, d=1201, lam=0.5, mode="implicit", kind="count",
                                tau=30, iters=12, seed=5, sseed=4, dual=True),
    # CSR primal, nnz-balanced row shards
    "csr_primal_gram": dict(data="csr", make=_csr_primal, n=3001, d=400, lam=1e-2, mode="gram",
                            kind="count", tau=40, iters=12, sseed=2),
    "csr_primal_implicit": dict(data="csr", make=_csr_primal, n=3001, d=400, lam=1e-2, mode="implicit",
                                kind="subsample", tau=33, iters=12, sseed=3),
    # CSR dual (n < d), nnz-balanced feature shards (Zipf column popularity)
    "csr_dual_gram": dict(data="csr", make=_csr_dual, n=300, d=5000, lam=1e-3, mode="gram",
                          kind="subcount", tau=16, k=4, iters=12, sseed=4),
    "csr_dual_implicit": dict(data="csr", make=_csr_dual, n=300, d=5000, lam=1e-3, mode="implicit",
                              kind="subsample", tau=25, iters=12, sseed=5),
}
