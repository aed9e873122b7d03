"""Momentum parameter schedules (gamma_k, beta_k) of the paper.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Sources (P = /root/reference/PAPER.md):
  * iterate-averaging parametrisation and its map to heavy ball (Eq.
    etalambdatogammbetagen):   gamma_k = eta_k / (zeta_{k+1} + 1),   beta_k = zeta_k / (zeta_{k+1} + 1)
  * Thm. 1 restriction on zeta (Eq. zeta_kaptheo):
        zeta_0 = 0,   zeta_k = (1 / eta_k) sum_{t=0}^{k-1} eta_t (1 - eta_t)   (k >= 1)
  * Cor. 1, constant eta < 1 (Eq. cst_eta_lambda_to_gamma_beta_formula):
        gamma_k = eta / ((k+1)(1-eta) + 1),   beta_k = 1 - (2 - eta) / ((k+1)(1-eta) + 1)
  * "theoretical" switch rule (Eq. parameterswitchtheory):
        eta_k = 0.995 if beta_k < 0.5, 1 if beta_k >= 0.5
    Circular as printed (beta_k depends on eta_k); reading DESIGN.md R24: the switch is decided
    on the previous step, eta_k = eta if beta_{k-1} < 0.5 (beta_{-1} = 0) else 1, and once
    switched eta stays 1.  With eta = 1, eta(1 - eta) = 0, so zeta freezes and (gamma, beta)
    become constant (gamma ~ 0.5, beta ~ 0.5 as P:L926 describes).
  * "heuristic" rule (Eq. parametersheurististic): gamma_k = 1 and beta_k of Cor. 1.
    The figure captions use eta = 0.5 and the equations eta = 0.995 (R17); eta is a
    parameter here, default 0.995.

Each schedule is a function k -> (gamma_k, beta_k).  The theoretical rule is computed from the
general Thm. 1 recursion (the eta sequence, the partial sums, the map), not from a closed form.
"""

import numpy as np


def constant(gamma, beta):
    return lambda k: (float(gamma), float(beta))


def zeta_from_etas(etas):
    """zeta_k for k = 0 .. len(etas)-1 from Eq. zeta_kaptheo (plain loop)."""
    z = []
    acc = 0.0
    for k, e in enumerate(etas):
        z.append(0.0 if k == 0 else acc / e)
        acc += e * (1.0 - e)
    return z


def map_to_heavy_ball(etas, zetas):
    """(gamma_k, beta_k) for k = 0 .. len(etas)-2 from Eq. etalambdatogammbetagen."""
    return [(etas[k] / (zetas[k + 1] + 1.0), zetas[k] / (zetas[k + 1] + 1.0))
            for k in range(len(etas) - 1)]


def corollary1(eta):
    """Cor. 1 closed form (constant eta < 1)."""
    assert 0.0 < eta < 1.0

    def f(k):
        den = (k + 1) * (1.0 - eta) + 1.0
        return eta / den, 1.0 - (2.0 - eta) / den
    return f


def heuristic(eta=0.995):
    """Eq. parametersheurististic: gamma_k = 1, beta_k of Cor. 1."""
    c = corollary1(eta)
    return lambda k: (1.0, c(k)[1])


def theory(eta=0.995, kmax=1_000_000):
    """Eq. parameterswitchtheory through the Thm. 1 recursion, reading R24: eta_0 = eta and
    eta_{k+1} = 1 once beta_k >= 0.5 (beta_k evaluated with eta_{k+1} = eta; re-evaluated with
    eta_{k+1} = 1 it only grows, so the rule is self-consistent), else eta."""
    table = []
    S = 0.0            # sum_{t<k} eta_t (1 - eta_t)
    e_k = eta          # eta_k
    zeta = 0.0         # zeta_k (zeta_0 = 0)
    switched = False
    for _ in range(kmax):
        S1 = S + e_k * (1.0 - e_k)
        e1 = 1.0 if switched else eta
        z1 = S1 / e1                                   # zeta_{k+1}
        g, b = e_k / (z1 + 1.0), zeta / (z1 + 1.0)
        if not switched and b >= 0.5:
            switched = True
            e1 = 1.0
            z1 = S1 / e1
            g, b = e_k / (z1 + 1.0), zeta / (z1 + 1.0)
        table.append((g, b))
        if e_k == 1.0:     # eta(1 - eta) = 0 from here on: zeta frozen, (gamma, beta) constant
            break
        S, e_k, zeta = S1, e1, z1
    last = table[-1]
    return lambda k: table[k] if k < len(table) else last


SCHEDULES = {"constant": None, "heuristic": heuristic, "theory": theory, "cor1": corollary1}


def make(name, gamma=1.0, beta=0.0, eta=0.995):
    if name == "constant":
        return constant(gamma, beta)
    return SCHEDULES[name](eta)
