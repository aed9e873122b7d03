"""Pins of the oracle's momentum schedules (oracle/momentum.py) against what the
paper fixes: Prop. 1 (heavy ball == iterate averaging), Cor. 1's closed form as a
special case of Thm. 1's zeta recursion, the printed starting values
beta_0 = 0 and the shape P:L926 describes for the theoretical rule."""
import numpy as np
import pytest

import rsinputs
from oracle import momentum as M
from oracle import problem as OP
from oracle import sketch as OS
from oracle import solver as OV


def test_cor1_is_thm1_recursion_with_constant_eta():
    for eta in (0.3, 0.5, 0.9, 0.995):
        etas = [eta] * 60
        z = M.zeta_from_etas(etas)
        assert np.allclose(z, [k * (1 - eta) for k in range(60)], rtol=1e-14, atol=1e-14)
        gb = M.map_to_heavy_ball(etas, z)
        c = M.corollary1(eta)
        for k in range(59):
            assert gb[k] == pytest.approx(c(k), rel=1e-13, abs=1e-15)


def test_starting_values_and_ranges():
    for name in ("heuristic", "theory", "cor1"):
        f = M.make(name, eta=0.5 if name == "cor1" else 0.995)
        g0, b0 = f(0)
        assert b0 == 0.0                       # beta_0 = 0 (zeta_0 = 0)
        for k in (0, 1, 10, 100, 1000, 10**5):
            g, b = f(k)
            assert 0 < g <= 1 and 0 <= b < 1   # the ranges Alg. 2 admits
    assert M.heuristic()(12345)[0] == 1.0


def test_theory_rule_shape():
    """beta increases from 0 to 0.5 while the step size decreases from 1 to 0.5."""
    f = M.theory(0.995)
    g = np.array([f(k)[0] for k in range(400)])
    b = np.array([f(k)[1] for k in range(400)])
    ks = int(np.argmax(b >= 0.5))
    assert 150 < ks < 260
    assert np.all(np.diff(b[:ks + 1]) > 0) and np.all(np.diff(g[:ks]) < 0)
    assert abs(b[ks + 5] - 0.5) < 0.01 and abs(g[ks + 5] - 0.5) < 0.01
    assert np.all(b[ks + 2:] == b[ks + 2]) and np.all(g[ks + 2:] == g[ks + 2])
    assert g[0] == pytest.approx(0.995 / (1 + 0.005), rel=1e-15)


def test_prop1_heavy_ball_equals_iterate_averaging():
    """Prop. 1: z^k = z^{k-1} - eta_k grad(w^k), w^{k+1} = (1 - 1/(zeta_{k+1}+1)) w^k
    + z^k/(zeta_{k+1}+1) gives the heavy-ball iterates with the mapped (gamma_k, beta_k); the
    gradient is the sketch-and-project step S_k delta_k."""
    X, y = rsinputs.dense_problem(200, 12, seed=3)
    X, y = X.numpy(), y.numpy()
    op = OV.Operator(X, y, 0.5)
    m, b = op.m, op.b
    etas = [0.7 + 0.2 * np.sin(k) for k in range(41)]   # any sequence in (0, 1)
    z = M.zeta_from_etas(etas)
    gb = M.map_to_heavy_ball(etas, z)
    # iterate averaging
    w = np.zeros(m)
    zz = w.copy()          # z^{-1} = w^0
    ws_ia = [w.copy()]
    for k in range(40):
        sk = OS.draw("subsample", m, 4, k, 9)
        S = OS.materialize(sk)
        AS = op.AS(S)
        r = op.apply(w) - b
        delta = np.linalg.solve(np.asarray(S.T @ AS), np.asarray(S.T @ r).ravel())
        grad = np.asarray(S @ delta).ravel()
        zz = zz - etas[k] * grad
        w = (1 - 1 / (z[k + 1] + 1)) * w + zz / (z[k + 1] + 1)
        ws_ia.append(w.copy())
    # heavy ball through the oracle's Alg. 2 with the mapped schedule
    res = OV.solve_momentum(op, "subsample", 4, max_iter=40, seed=9, schedule=lambda k: gb[k])
    assert np.linalg.norm(res["w"] - ws_ia[40]) <= 1e-10 * np.linalg.norm(ws_ia[40])


@pytest.mark.parametrize("name", ["heuristic", "theory", "cor1"])
def test_schedules_keep_residual_invariant_and_converge(name):
    X, y = rsinputs.dense_problem(300, 20, seed=1)
    X, y = X.numpy(), y.numpy()
    res = OV.solve(X, y, 1e-1, "subsample", 5, tol=0.0, max_iter=400, seed=2, momentum=name,
                   eta=0.5 if name == "cor1" else 0.995)
    pr = OP.build(X, y, 1e-1)
    r_true = pr["A"] @ res["w"] - pr["b"]
    assert np.linalg.norm(res["r"] - r_true) <= 1e-10 * np.linalg.norm(pr["b"])
    assert np.linalg.norm(res["r"]) < 0.5 * np.linalg.norm(pr["b"])
