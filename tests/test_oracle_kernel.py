"""Pins of the oracle's kernel ridge route (oracle/problem.py rbf_kernel, build_kernel; SURVEY
NEXT-4) against what the paper fixes."""
import numpy as np
import pytest

from oracle import problem as OP
from oracle import solver as OV


def test_rbf_two_points_closed_form():
    X = np.array([[0.0, 0.0], [3.0, 4.0]])          # ||x1 - x2||^2 = 25
    K = OP.rbf_kernel(X, sigma=2.0)
    e = np.exp(-25.0 / 8.0)                          # Eq. Gausskernel
    assert np.allclose(K, [[1.0, e], [e, 1.0]], rtol=0, atol=1e-16)


def test_rbf_structure():
    rng = np.random.default_rng(0)
    X = rng.standard_normal((40, 3))
    K = OP.rbf_kernel(X, 1.3)
    assert np.array_equal(K, K.T) and np.all(np.diag(K) == 1.0)
    assert np.all((K > 0) & (K <= 1))
    assert np.linalg.eigvalsh(K).min() > -1e-12      # a Gram matrix <phi(x_i), phi(x_j)>
    # brute force entry
    i, j = 7, 31
    assert K[i, j] == pytest.approx(np.exp(-np.sum((X[i] - X[j]) ** 2) / (2 * 1.3 ** 2)), rel=1e-15)


def test_kernel_system_is_dual_objective_stationarity():
    """A alpha - b = grad of 1/2 ||K alpha - y||^2 + lambda/2 alpha^T K alpha."""
    rng = np.random.default_rng(1)
    X = rng.standard_normal((30, 4))
    y = rng.standard_normal(30)
    lam = 0.3
    s = OP.build_kernel(X, y, lam, 1.1)
    K = s["K"]
    alpha = rng.standard_normal(30)
    obj = lambda a: 0.5 * np.sum((K @ a - y) ** 2) + 0.5 * lam * a @ K @ a
    h = 1e-6
    grad_fd = np.array([(obj(alpha + h * e) - obj(alpha - h * e)) / (2 * h) for e in np.eye(30)])
    assert np.allclose(s["A"] @ alpha - s["b"], grad_fd, rtol=1e-6, atol=1e-6)


def test_kernel_identity_limit():
    """Far-apart points: K = I, so A = (1 + lambda) I, b = y and alpha = y / (1 + lambda)."""
    X = np.arange(6, dtype=np.float64)[:, None] * 100.0
    y = np.array([1.0, -2.0, 3.0, 0.5, 0.0, 4.0])
    s = OP.build_kernel(X, y, 0.25, 1.0)
    assert np.array_equal(s["K"], np.eye(6))
    res = OV.solve_kernel(X, y, 0.25, 1.0, "subsample", 6, max_iter=1)   # S = I: one step
    assert np.allclose(res["w"], y / 1.25, rtol=1e-14, atol=1e-15)


def test_kernel_solve_converges_to_direct():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((40, 3))
    y = np.sin(X @ np.array([1.0, -0.5, 0.25])) + 0.01 * rng.standard_normal(40)
    s = OP.build_kernel(X, y, 1.0, 0.8)
    a_star = OP.direct_solve(s["A"], s["b"])
    res = OV.solve_kernel(X, y, 1.0, 0.8, "subsample", 20, tol=1e-10, max_iter=20000, seed=3)
    assert res["converged"]
    cond = np.linalg.cond(s["A"])
    assert np.linalg.norm(res["w"] - a_star) <= 10 * cond * 1e-10 * np.linalg.norm(a_star)
