"""Sketch-and-project with momentum, literally as printed (Alg. 2), and the plain
method (Alg. 1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Alg. 2, constant gamma_k = gamma and beta_k = beta:

    w^{-1} = w^0 = 0,  r^{-1} = r^0 = A w^0 - b = -b
    while ||r^k|| / ||r^0|| > eps  (printed "<=": typo, R1)
        S_k ~ D
        r_S = S_k^T r^k
        delta_k = least_norm_solution(S_k^T A S_k, r_S)
        w^{k+1} = (1 + beta) w^k - beta w^{k-1} - gamma S_k delta_k
        r^{k+1} = (1 + beta) r^k - beta r^{k-1} - gamma A S_k delta_k       (Eq. res_update_mom)

AS is formed either implicitly, X^T (X S) + lambda S (primal) / X (X^T S) + lambda S (dual), or
from the explicit A (R10); both equal A S in exact arithmetic.

least_norm_solution: with lambda > 0 and S of full column rank (disjoint
supports) G = S^T A S is SPD and G^+ g = G^{-1} g, computed by Cholesky reading only G's lower
triangle (R3, R12).  A count-sketch bucket with no coordinate is an all-zero column
of S: its row/column of G and its entry of g are zero, and the exact least-norm solution has
delta_b = 0; this is realised by setting G_bb = 1 (R3).
"""

import numpy as np
import scipy.linalg as sla

from . import problem as P
from . import sketch as SK


class Operator:
    """The map S -> A S for the system of Eq. Axb."""

    def __init__(self, X, y, lam, which=None, explicit=False):
        n, d = X.shape
        self.X, self.lam = X, lam
        self.route = which or P.route(n, d)
        self.m = d if self.route == P.PRIMAL else n
        self.b = (np.asarray(X.T @ y, dtype=np.float64).ravel() if self.route == P.PRIMAL
                  else np.asarray(y, dtype=np.float64).copy())
        self.A = P.build(X, y, lam, self.route)["A"] if explicit else None

    @classmethod
    def from_system(cls, A, b):
        """An explicit system A w = b (e.g. kernel ridge)."""
        op = cls.__new__(cls)
        op.X, op.lam, op.route = None, 0.0, "explicit"
        op.m = A.shape[0]
        op.A = np.asarray(A, dtype=np.float64)
        op.b = np.asarray(b, dtype=np.float64).ravel()
        return op

    def AS(self, S):
        """A S as a dense m x tau array (S: scipy sparse m x tau)."""
        if self.A is not None:
            return np.asarray(self.A @ S.toarray())
        X = self.X
        if self.route == P.PRIMAL:
            XS = np.asarray(X @ S.toarray())               # n x tau
            out = np.asarray(X.T @ XS)                     # d x tau
        else:
            XtS = np.asarray(X.T @ S.toarray())            # d x tau
            out = np.asarray(X @ XtS)                      # n x tau
        return out + self.lam * S.toarray()

    def apply(self, w):
        """A w (used only by tests to check the residual invariant)."""
        if self.A is not None:
            return self.A @ w
        X = self.X
        if self.route == P.PRIMAL:
            return np.asarray(X.T @ (X @ w)).ravel() + self.lam * w
        return np.asarray(X @ (X.T @ w)).ravel() + self.lam * w


def sketched_solve(G, g, empty):
    """delta = least_norm_solution(G, g) for SPD G (+ empty-bucket rule), Cholesky, lower."""
    G = np.array(G, dtype=np.float64, copy=True)
    g = np.array(g, dtype=np.float64, copy=True)
    for bkt in empty:
        G[bkt, :] = 0.0
        G[:, bkt] = 0.0
        G[bkt, bkt] = 1.0
        g[bkt] = 0.0
    c = sla.cho_factor(G, lower=True, check_finite=True)
    return sla.cho_solve(c, g)


def solve_momentum(op, kind, tau, gamma=1.0, beta=0.0, tol=0.0, max_iter=100, seed=0,
                   subcount_k=0, record=False, trace=False, schedule=None):
    """Alg. 2 with constant (gamma, beta), or with gamma_k, beta_k = schedule(k) (an
    oracle.momentum schedule).  Returns dict(w, r, iterations, converged, trace, [records]).
    `w` is the system iterate (alpha in the dual route)."""
    m = op.m
    b = op.b
    w_prev = np.zeros(m)
    w = np.zeros(m)
    r_prev = -b.copy()
    r = -b.copy()
    nb = np.linalg.norm(b)
    out = dict(trace=[], records=[])
    k = 0
    if nb == 0.0:   # b = 0: w^0 = 0 is the solution, 0 iterations
        return dict(w=w, r=r, iterations=0, converged=True, **out)
    while k < max_iter and np.linalg.norm(r) > tol * nb:
        if schedule is not None:
            gamma, beta = schedule(k)  # gamma_k, beta_k
        sk = SK.draw(kind, m, tau, k, seed, subcount_k)
        S = SK.materialize(sk)
        AS = op.AS(S)
        G = S.T @ AS                   # S^T A S, tau x tau
        g = S.T @ r                    # r_S = S^T r^k
        delta = sketched_solve(np.asarray(G), np.asarray(g).ravel(), SK.empty_buckets(sk))
        Sd = np.asarray(S @ delta).ravel()
        ASd = AS @ delta
        w_next = (1.0 + beta) * w - beta * w_prev - gamma * Sd
        r_next = (1.0 + beta) * r - beta * r_prev - gamma * ASd
        w_prev, w, r_prev, r = w, w_next, r, r_next
        if record:
            out["records"].append(dict(sketch=sk, delta=delta, G=np.asarray(G), g=np.asarray(g).ravel()))
        k += 1
        if trace:
            out["trace"].append(np.linalg.norm(r) / nb)
    converged = bool(np.linalg.norm(r) <= tol * nb)
    return dict(w=w, r=r, iterations=k, converged=converged, **out)


def solve_sketch_project(op, kind, tau, tol=0.0, max_iter=100, seed=0, subcount_k=0):
    """Alg. 1, literal: least_norm_solution by a least-squares solver (SVD-based,
    minimum norm), w <- w - S delta, r <- r - A S delta."""
    m = op.m
    b = op.b
    w = np.zeros(m)
    r = -b.copy()
    nb = np.linalg.norm(b)
    k = 0
    while k < max_iter and np.linalg.norm(r) > tol * nb:
        sk = SK.draw(kind, m, tau, k, seed, subcount_k)
        S = SK.materialize(sk)
        AS = op.AS(S)
        rS = S.T @ r
        delta = np.linalg.lstsq(np.asarray(S.T @ AS), np.asarray(rS).ravel(), rcond=None)[0]
        w = w - np.asarray(S @ delta).ravel()
        r = r - AS @ delta
        k += 1
    return dict(w=w, r=r, iterations=k)


def solve(X, y, lam, kind, tau, gamma=1.0, beta=0.0, tol=0.0, max_iter=100, seed=0,
          subcount_k=0, explicit=False, which=None, record=False, trace=False,
          momentum="constant", eta=0.995):
    """Whole ridge solve: build the system, run Alg. 2, recover w (dual: X^T alpha).
    momentum: "constant" (gamma, beta) or an oracle.momentum schedule ("heuristic", "theory",
    "cor1") with parameter eta."""
    from . import momentum as MOM
    op = Operator(X, y, lam, which, explicit)
    sched = None if momentum == "constant" else MOM.make(momentum, gamma, beta, eta)
    res = solve_momentum(op, kind, tau, gamma, beta, tol, max_iter, seed, subcount_k, record, trace,
                         schedule=sched)
    res["route"] = op.route
    res["weights"] = res["w"] if op.route == P.PRIMAL else P.recover_weights(X, res["w"])
    return res


def solve_kernel(X, y, lam, sigma, kind, tau, gamma=1.0, beta=0.0, tol=0.0, max_iter=100, seed=0,
                 subcount_k=0, momentum="constant", eta=0.995):
    """Kernel ridge regression: Alg. 2 on K (K + lambda I) alpha = K y."""
    from . import momentum as MOM
    sysk = P.build_kernel(X, y, lam, sigma)
    op = Operator.from_system(sysk["A"], sysk["b"])
    sched = None if momentum == "constant" else MOM.make(momentum, gamma, beta, eta)
    res = solve_momentum(op, kind, tau, gamma, beta, tol, max_iter, seed, subcount_k,
                         schedule=sched)
    res["route"] = "kernel"
    res["weights"] = res["w"]
    res["K"] = sysk["K"]
    return res


# ------------------------------------------------------------------ extended precision (x87, 64-bit)
def cholesky_solve_ld(G, g):
    """G^{-1} g for SPD G in np.longdouble: the textbook Cholesky G = L L^T (column by column,
    L_jj = sqrt(G_jj - sum_k L_jk^2), L_ij = (G_ij - sum_k L_ik L_jk) / L_jj, lower triangle read),
    then L y = g and L^T x = y by substitution (P:L217 least-norm solution = G^{-1} g, DESIGN R3)."""
    G = np.array(G, dtype=np.longdouble)
    n = G.shape[0]
    L = np.zeros((n, n), dtype=np.longdouble)
    for j in range(n):
        d = G[j, j] - np.dot(L[j, :j], L[j, :j])
        if not d > 0:
            raise np.linalg.LinAlgError("not SPD")
        L[j, j] = np.sqrt(d)
        L[j + 1:, j] = (G[j + 1:, j] - L[j + 1:, :j] @ L[j, :j]) / L[j, j]
    y = np.zeros(n, dtype=np.longdouble)
    for i in range(n):
        y[i] = (g[i] - np.dot(L[i, :i], y[:i])) / L[i, i]
    x = np.zeros(n, dtype=np.longdouble)
    for i in range(n - 1, -1, -1):
        x[i] = (y[i] - np.dot(L[i + 1:, i], x[i + 1:])) / L[i, i]
    return x


def solve_system_ld(A, b, kind, tau, gamma=1.0, beta=0.0, iters=10, seed=0, subcount_k=0):
    """Alg. 2 on an explicit system A w = b carried out in np.longdouble (64-bit
    significand, eps = 2^-63): the reference that an ill-conditioned fp64 run is compared against.
    Same sketch stream, same recurrences as solve_momentum; A and b are converted exactly."""
    A = np.asarray(A, dtype=np.longdouble)
    b = np.asarray(b, dtype=np.longdouble)
    m = A.shape[0]
    w_prev = np.zeros(m, dtype=np.longdouble)
    w = np.zeros(m, dtype=np.longdouble)
    r_prev, r = -b.copy(), -b.copy()
    g_, b_ = np.longdouble(gamma), np.longdouble(beta)
    for k in range(iters):
        sk = SK.draw(kind, m, tau, k, seed, subcount_k)
        S = np.zeros((m, tau), dtype=np.longdouble)
        S[sk["coord"], sk["bucket"]] = sk["sign"]
        AS = A @ S
        G = S.T @ AS
        g = S.T @ r
        for bkt in SK.empty_buckets(sk):
            G[bkt, :] = 0
            G[:, bkt] = 0
            G[bkt, bkt] = 1
            g[bkt] = 0
        delta = cholesky_solve_ld(G, g)
        w_next = (1 + b_) * w - b_ * w_prev - g_ * (S @ delta)
        r_next = (1 + b_) * r - b_ * r_prev - g_ * (AS @ delta)
        w_prev, w, r_prev, r = w, w_next, r, r_next
    return dict(w=w, r=r, iterations=iters)
