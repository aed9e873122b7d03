"""Pins for oracle/problem.py and oracle/solver.py against what the paper and the mathematics fix:
textbook normal equations, the dual-equivalence Lemma, S = I solving in one step
(P:L243), tau = 1 coordinate descent with momentum in closed form (Eq. CDmom), beta = 0
reducing to Alg. 1 with its projection constraint, the residual invariant
r = A w - b, the empty-bucket least-norm rule, and
convergence to the direct solve (BASELINE.json)."""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import problem as P
from oracle import sketch as SK
from oracle import solver as SV
import rsinputs


def _small(n=60, d=12, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((n, d))
    y = rng.standard_normal(n)
    return X, y


# ----------------------------------------------------------------------------- problem build

def test_build_identity_examples():
    X = np.eye(2)
    y = np.array([1.0, 2.0])
    pr = P.build(X, y, 1.0)
    assert pr["route"] == "primal"
    assert np.array_equal(pr["A"], 2 * np.eye(2)) and np.array_equal(pr["b"], y)


def test_build_entrywise_textbook():
    X, y = _small(9, 4, 1)
    lam = 0.3
    pr = P.build(X, y, lam)
    n, d = X.shape
    for i in range(d):
        assert abs(pr["b"][i] - sum(X[k, i] * y[k] for k in range(n))) < 1e-12
        for j in range(d):
            ref = sum(X[k, i] * X[k, j] for k in range(n)) + (lam if i == j else 0.0)
            assert abs(pr["A"][i, j] - ref) < 1e-12
    du = P.build(X.T.copy(), np.arange(4.0), lam)
    assert du["route"] == "dual" and du["m"] == 4
    assert np.allclose(du["A"], X.T @ X + lam * np.eye(4)) and np.array_equal(du["b"], np.arange(4.0))


def test_route_rule():
    assert P.route(10, 10) == "primal" and P.route(10, 3) == "primal" and P.route(3, 10) == "dual"
    with pytest.raises(ValueError):
        P.build(np.eye(2), np.ones(2), 0.0)


def test_dual_lemma():
    """X^T (X X^T + lam I)^{-1} y = (X^T X + lam I)^{-1} X^T y."""
    rng = np.random.default_rng(2)
    X = rng.standard_normal((8, 20))
    y = rng.standard_normal(8)
    lam = 0.5
    pr = P.build(X, y, lam, "primal")
    du = P.build(X, y, lam, "dual")
    w_p = P.direct_solve(pr["A"], pr["b"])
    w_d = P.recover_weights(X, P.direct_solve(du["A"], du["b"]))
    assert np.linalg.norm(w_p - w_d) <= 1e-10 * np.linalg.norm(w_p)


def test_direct_solve_vs_gesv():
    X, y = _small(100, 30, 3)
    pr = P.build(X, y, 0.1)
    w = P.direct_solve(pr["A"], pr["b"])
    w2 = np.linalg.solve(pr["A"], pr["b"])   # LAPACK gesv, the paper's direct baseline
    assert np.linalg.norm(w - w2) <= 1e-12 * np.linalg.norm(w2)
    assert np.linalg.norm(pr["A"] @ w - pr["b"]) <= 1e-12 * np.linalg.norm(pr["b"])


# ----------------------------------------------------------------------------- solver pins

@pytest.mark.parametrize("which", ["primal", "dual"])
def test_S_identity_one_step(which):
    """tau = m subsample (S = I, up to column order), gamma=1, beta=0: w^1 = A^{-1} b."""
    X, y = _small(40, 15, 4)
    if which == "dual":
        X = X.T.copy()
        y = y[:15]
    op = SV.Operator(X, y, 0.7)
    res = SV.solve_momentum(op, "subsample", op.m, 1.0, 0.0, 0.0, 1, seed=3)
    A = P.build(X, y, 0.7)["A"]
    w_star = np.linalg.solve(A, op.b)
    assert res["iterations"] == 1
    assert np.linalg.norm(res["w"] - w_star) <= 1e-10 * np.linalg.norm(w_star)
    assert np.linalg.norm(res["r"]) <= 1e-10 * np.linalg.norm(op.b)


def test_tau1_is_coordinate_descent_with_momentum():
    """P:L816 Eq. CDmom: w^{k+1} = w^k - gamma (A_i: w^k - b_i)/A_ii e_i + beta (w^k - w^{k-1})."""
    X, y = _small(50, 10, 5)
    lam, gamma, beta, K, seed = 0.2, 0.8, 0.3, 40, 17
    op = SV.Operator(X, y, lam)
    res = SV.solve_momentum(op, "subsample", 1, gamma, beta, 0.0, K, seed=seed)
    A = P.build(X, y, lam)["A"]
    b = op.b
    w_prev = np.zeros(10)
    w = np.zeros(10)
    for k in range(K):
        i = int(SK.draw("subsample", 10, 1, k, seed)["coord"][0])
        e = np.zeros(10)
        e[i] = 1.0
        w_next = w - gamma * (A[i] @ w - b[i]) / A[i, i] * e + beta * (w - w_prev)
        w_prev, w = w, w_next
    assert np.linalg.norm(res["w"] - w) <= 1e-12 * np.linalg.norm(w)


@pytest.mark.parametrize("kind", ["subsample", "count", "subcount"])
def test_beta0_equals_alg1_and_projection(kind):
    """beta=0, gamma=1 is Alg. 1: same iterates as the literal least-squares version,
    and every step satisfies the sketched constraint S_k^T A w^{k+1} = S_k^T b, and the
    A-norm error is non-increasing (projection)."""
    X, y = _small(80, 20, 6)
    lam = 0.05
    op = SV.Operator(X, y, lam)
    K = 25
    r2 = SV.solve_momentum(op, kind, 5, 1.0, 0.0, 0.0, K, seed=8, subcount_k=2, record=True)
    r1 = SV.solve_sketch_project(op, kind, 5, 0.0, K, seed=8, subcount_k=2)
    assert np.linalg.norm(r2["w"] - r1["w"]) <= 1e-11 * np.linalg.norm(r1["w"])
    A = P.build(X, y, lam)["A"]
    w_star = np.linalg.solve(A, op.b)
    opk = SV.Operator(X, y, lam)
    w = np.zeros(20)
    prev_err = np.sqrt((w - w_star) @ A @ (w - w_star))
    for k in range(K):
        res = SV.solve_momentum(opk, kind, 5, 1.0, 0.0, 0.0, k + 1, seed=8, subcount_k=2)
        sk = SK.draw(kind, 20, 5, k, 8, 2)
        S = SK.materialize(sk)
        cons = S.T @ (A @ res["w"] - op.b)
        assert np.linalg.norm(cons) <= 1e-10 * np.linalg.norm(op.b)
        err = np.sqrt((res["w"] - w_star) @ A @ (res["w"] - w_star))
        assert err <= prev_err * (1 + 1e-12) + 1e-12
        prev_err = err


@pytest.mark.parametrize("which,kind,explicit,beta", [
    ("primal", "subsample", False, 0.0), ("primal", "subsample", False, 0.5),
    ("primal", "count", True, 0.5), ("primal", "subcount", False, 0.5),
    ("dual", "subcount", False, 0.5), ("dual", "count", False, 0.0),
    ("dual", "subsample", True, 0.5)])
def test_residual_invariant(which, kind, explicit, beta):
    """Maintained r^k equals A w^k - b (Eq. res_update_mom)."""
    X, y = _small(120, 30, 9)
    if which == "dual":
        X = X.T.copy()
        y = y[:30]
    op = SV.Operator(X, y, 0.1, explicit=explicit)
    res = SV.solve_momentum(op, kind, 6, 1.0, beta, 0.0, 300, seed=1, subcount_k=2)
    fresh = op.apply(res["w"]) - op.b
    assert np.linalg.norm(res["r"] - fresh) <= 1e-10 * np.linalg.norm(op.b)


def test_implicit_equals_explicit_AS():
    X, y = _small(70, 14, 10)
    lam = 0.3
    opi = SV.Operator(X, y, lam)
    ope = SV.Operator(X, y, lam, explicit=True)
    S = SK.materialize(SK.draw("count", 14, 4, 0, 1))
    assert np.allclose(opi.AS(S), ope.AS(S), rtol=0, atol=1e-11 * np.abs(ope.A).max())
    Xs = sp.csr_matrix(X)
    ops = SV.Operator(Xs, y, lam)
    assert np.allclose(ops.AS(S), ope.AS(S), rtol=0, atol=1e-11 * np.abs(ope.A).max())


@pytest.mark.parametrize("beta,iters", [(0.0, 300), (0.5, 1000)])
def test_config1_converges_to_direct_solve(beta, iters):
    """BASELINE.json c1: 1000x50, lambda 1e-2, subsample tau=10 -> the direct Cholesky solution
    within 1e-6 relative.  beta=0 reaches it in the config's 300 iterations; constant beta=0.5
    heavy ball contracts more slowly on this well-conditioned system (7.7e-5 at 300 iterations,
    4e-9 at 600), so it is checked at 1000 iterations (reading R19)."""
    cfg = rsinputs.CONFIGS["c1"]
    X, y = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, noise=cfg.noise)
    X, y = X.numpy(), y.numpy()
    res = SV.solve(X, y, cfg.lam, "subsample", cfg.tau, 1.0, beta, 0.0, iters, seed=0)
    pr = P.build(X, y, cfg.lam)
    w_star = np.linalg.solve(pr["A"], pr["b"])
    assert res["iterations"] == iters
    assert np.linalg.norm(res["weights"] - w_star) <= 1e-6 * np.linalg.norm(w_star)


def test_empty_bucket_least_norm():
    """P:L217 least_norm_solution: with an empty count bucket, the Cholesky + G_bb=1 rule gives the
    pseudo-inverse (least-norm) solution."""
    X, y = _small(90, 50, 11)
    op = SV.Operator(X, y, 0.2)
    rng = np.random.default_rng(0)
    r = rng.standard_normal(50)
    hits = 0
    for it in range(300):
        sk = SK.draw("count", 50, 10, it, 0)
        e = SK.empty_buckets(sk)
        if e.size == 0:
            continue
        S = SK.materialize(sk)
        AS = op.AS(S)
        G = np.asarray(S.T @ AS)
        g = np.asarray(S.T @ r).ravel()
        d1 = SV.sketched_solve(G, g, e)
        d2 = np.linalg.pinv(G, rcond=1e-12, hermitian=True) @ g
        assert np.linalg.norm(d1 - d2) <= 1e-10 * np.linalg.norm(d2)
        assert np.all(d1[e] == 0.0)
        hits += 1
    assert hits >= 3


def test_zero_rhs_zero_iterations():
    X, _ = _small(30, 5, 12)
    res = SV.solve(X, np.zeros(30), 0.1, "subsample", 2, max_iter=50, tol=1e-4)
    assert res["iterations"] == 0 and np.all(res["weights"] == 0)


def test_dual_solve_recovers_primal_solution():
    rng = np.random.default_rng(13)
    X = rng.standard_normal((20, 60))
    y = rng.standard_normal(20)
    res = SV.solve(X, y, 1.0, "subsample", 20, 1.0, 0.0, 0.0, 1, seed=0)   # tau = m: exact
    assert res["route"] == "dual"
    pr = P.build(X, y, 1.0, "primal")
    w_star = np.linalg.solve(pr["A"], pr["b"])
    assert np.linalg.norm(res["weights"] - w_star) <= 1e-10 * np.linalg.norm(w_star)


def test_tolerance_stop_rule():
    """Stop as soon as ||r^k|| <= tol ||r^0|| (printed '<=' in the while is a typo)."""
    X, y = _small(200, 20, 14)
    res = SV.solve(X, y, 0.5, "subsample", 5, 1.0, 0.5, 1e-6, 10000, seed=2, trace=True)
    assert res["converged"]
    tr = res["trace"]
    assert tr[-1] <= 1e-6 and all(t > 1e-6 for t in tr[:-1])


def test_extended_precision_oracle_matches_fp64_on_well_conditioned():
    """solve_system_ld (np.longdouble Alg. 2, hand-written Cholesky) agrees with the fp64 oracle to
    ~1e-14 on a well-conditioned explicit system, and its Cholesky solve reproduces
    numpy.linalg.solve on a random SPD matrix: pins the extended-precision reference that the
    ill-conditioned kernel-ridge GPU case is compared against."""
    import numpy as np
    from oracle import problem as P
    from oracle import solver as OV
    rng = np.random.default_rng(3)
    M = rng.standard_normal((30, 30))
    G = M @ M.T + 30 * np.eye(30)
    g = rng.standard_normal(30)
    x = OV.cholesky_solve_ld(G, g)
    assert np.allclose(np.asarray(x, dtype=np.float64), np.linalg.solve(G, g), rtol=1e-13, atol=0)
    X = rng.standard_normal((200, 12))
    y = rng.standard_normal(200)
    pr = P.build(X, y, 0.7)
    ref = OV.solve_momentum(OV.Operator.from_system(pr["A"], pr["b"]), "count", 5, 1.0, 0.5, 0.0, 25, seed=2)
    ld = OV.solve_system_ld(pr["A"], pr["b"], "count", 5, 1.0, 0.5, 25, seed=2)
    w = np.asarray(ld["w"], dtype=np.float64)
    assert np.linalg.norm(w - ref["w"]) <= 1e-13 * np.linalg.norm(ref["w"])
