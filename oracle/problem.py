"""The ridge linear system A w = b (Section "Linear system formulation").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* Ridge objective 1/2 ||X w - y||^2 + lambda/2 ||w||^2, lambda > 0 (Eq. ridge).
* Primal (Eq. linear): (X^T X + lambda I) w = X^T y.
* Dual (Eq. duallinear): (X X^T + lambda I) alpha = y, w = X^T alpha.
* Route: primal when d <= n, dual when n < d.
* Unified form (Eq. Axb): A = B + lambda I, b = X^T y (primal) or y (dual), m = d or n.
* Direct solve: Cholesky of the SPD A (the paper's baseline uses LAPACK gesv,
  P:L1029; A is SPD so a Cholesky solve computes the same solution).
"""

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

PRIMAL, DUAL = "primal", "dual"


def route(n, d):
    """primal form preferred when d <= n, dual when n < d (tie -> primal)."""
    return PRIMAL if d <= n else DUAL


def _dense(M):
    return M.toarray() if sp.issparse(M) else np.asarray(M, dtype=np.float64)


def build(X, y, lam, which=None):
    """Return dict(route, m, A (dense m x m), b) for Eq. Axb."""
    if not lam > 0:
        raise ValueError("lambda must be > 0 (P:L36)")
    n, d = X.shape
    which = which or route(n, d)
    y = np.asarray(y, dtype=np.float64)
    if which == PRIMAL:
        B = _dense(X.T @ X)
        b = np.asarray(X.T @ y, dtype=np.float64).ravel()
        m = d
    else:
        B = _dense(X @ X.T)
        b = y.copy()
        m = n
    A = B + lam * np.eye(m)
    return dict(route=which, m=m, A=A, b=b, lam=lam)


def recover_weights(X, alpha):
    """Dual recovery w = X^T alpha ("a multiplication by X^T is required")."""
    return np.asarray(X.T @ alpha, dtype=np.float64).ravel()


def direct_solve(A, b):
    """Direct SPD solve via Cholesky: A = L L^T, then two triangular solves."""
    c = sla.cho_factor(A, lower=True)
    return sla.cho_solve(c, b)


def rbf_kernel(X, sigma):
    """Gaussian (RBF) kernel matrix K_ij = exp(-||x_i - x_j||^2 / (2 sigma^2)) (P:L175-180,
    Eq. Gausskernel), from the explicit differences x_i - x_j (one row of K at a time)."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    K = np.empty((n, n))
    for i in range(n):
        diff = X - X[i]
        K[i] = np.exp(-np.einsum("jk,jk->j", diff, diff) / (2.0 * sigma * sigma))
    return K


def build_kernel(X, y, lam, sigma):
    """Kernel ridge system: K (K + lambda I) alpha = K y (Eq. kernelridge), i.e.
    A = K^T (K + lambda I), b = K^T y, m = n; the predictor is K alpha."""
    if not lam > 0:
        raise ValueError("lambda must be > 0 (P:L36)")
    K = rbf_kernel(X, sigma)
    y = np.asarray(y, dtype=np.float64)
    n = K.shape[0]
    A = K.T @ (K + lam * np.eye(n))
    b = K.T @ y
    return dict(route="kernel", m=n, A=A, b=b, K=K, lam=lam)
