"""Pins for oracle/sketch.py: brute-force selection, exact structure of the count and
SubCount sketches, uniformity (chi-square), the printed (s, k) rule, and materialisation."""

import itertools
import math
import os

import numpy as np
import pytest
from scipy import stats

from oracle import sketch as SK
from oracle.philox import philox4x32_10, seed_key

HERE = os.path.dirname(os.path.abspath(__file__))


def _py_philox(c, k):
    """Scalar pure-Python Philox4x32-10 (brute-force cross-check of the vectorised oracle)."""
    c = list(c)
    k0, k1 = k
    for rnd in range(10):
        p0 = 0xD2511F53 * c[0]
        p1 = 0xCD9E8D57 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & 0xFFFFFFFF, p1 & 0xFFFFFFFF,
             ((p0 >> 32) ^ c[3] ^ k1) & 0xFFFFFFFF, p0 & 0xFFFFFFFF]
        if rnd < 9:
            k0 = (k0 + 0x9E3779B9) & 0xFFFFFFFF
            k1 = (k1 + 0xBB67AE85) & 0xFFFFFFFF
    return c


@pytest.mark.parametrize("m,tau,it,seed", [(1, 1, 0, 0), (7, 3, 2, 1), (64, 10, 5, 2**40 + 3),
                                           (33, 33, 0, 9)])
def test_subsample_brute_force(m, tau, it, seed):
    key = seed_key(seed)
    keys = []
    for i in range(m):
        x, y, _, _ = _py_philox([i, it, 0, 0], key)
        keys.append(((x << 32) | y, i))
    expect = [i for _, i in sorted(keys)[:tau]]
    sk = SK.draw("subsample", m, tau, it, seed)
    assert sk["coord"].tolist() == expect
    assert len(set(expect)) == tau and all(0 <= i < m for i in expect)
    assert sk["bucket"].tolist() == list(range(tau)) and np.all(sk["sign"] == 1)


def test_subsample_tau_equals_m_is_permutation():
    sk = SK.draw("subsample", 50, 50, 3, 11)
    assert sorted(sk["coord"].tolist()) == list(range(50))


def test_subsample_uniform_over_subsets_chi2():
    """Eq. subsample: every 3-subset of [8] has probability 1/C(8,3)."""
    m, tau, draws, seed = 8, 3, 60000, 123
    k0, k1 = seed_key(seed)
    i = np.repeat(np.arange(m, dtype=np.uint64)[None, :], draws, axis=0)
    it = np.repeat(np.arange(draws, dtype=np.uint64)[:, None], m, axis=1)
    x, y, _, _ = philox4x32_10(i, it, 0, 0, k0, k1)
    key64 = (x << np.uint64(32)) | y
    sel = np.sort(np.argsort(key64, axis=1, kind="stable")[:, :tau], axis=1)
    for t in (0, 1, 2, 999):   # the vectorised selection equals draw()
        assert sorted(SK.draw("subsample", m, tau, t, seed)["coord"].tolist()) == sel[t].tolist()
    codes = (sel[:, 0] * 64 + sel[:, 1] * 8 + sel[:, 2])
    subsets = {a * 64 + b * 8 + c: 0 for a, b, c in itertools.combinations(range(m), tau)}
    for cval, cnt in zip(*np.unique(codes, return_counts=True)):
        subsets[int(cval)] = cnt
    obs = np.array(list(subsets.values()))
    assert obs.shape[0] == math.comb(8, 3)
    p = stats.chisquare(obs).pvalue
    assert p > 1e-4


@pytest.mark.parametrize("m,tau", [(6, 2), (50, 10), (1000, 37)])
def test_count_exact_structure(m, tau):
    """Each coordinate in exactly one bucket with one +-1 (BASELINE north_star)."""
    for it in range(3):
        sk = SK.draw("count", m, tau, it, 5)
        S = SK.materialize(sk).toarray()
        assert S.shape == (m, tau)
        nz_per_row = (S != 0).sum(axis=1)
        assert np.all(nz_per_row == 1)
        assert set(np.unique(S[S != 0]).tolist()) <= {-1.0, 1.0}
        assert np.all((sk["bucket"] >= 0) & (sk["bucket"] < tau))
        assert sk["coord"].tolist() == list(range(m))


def test_count_bucket_uniform_and_sign_balance():
    m, tau = 200000, 50
    sk = SK.draw("count", m, tau, 0, 77)
    counts = np.bincount(sk["bucket"], minlength=tau)
    assert stats.chisquare(counts).pvalue > 1e-4
    npos = int((sk["sign"] > 0).sum())
    assert stats.binomtest(npos, m, 0.5).pvalue > 1e-4


def test_count_bucket_brute_force():
    m, tau, it, seed = 40, 7, 3, 1234
    sk = SK.draw("count", m, tau, it, seed)
    key = seed_key(seed)
    for i in range(m):
        x, y, _, _ = _py_philox([i, it, 1, 0], key)
        assert sk["bucket"][i] == (x * tau) >> 32
        assert sk["sign"][i] == (1 - 2 * (y & 1))


def _golden_subcount():
    rows = []
    with open(os.path.join(HERE, "golden", "subcount_params.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                rows.append([int(t) for t in line.split()])
    return rows


@pytest.mark.parametrize("row", _golden_subcount())
def test_subcount_params_paper_rule(row):
    tau, m, s, k = row
    assert SK.subcount_params(tau, m) == (s, k)


def test_subcount_params_override_and_errors():
    assert SK.subcount_params(256, 20000, 4) == (1024, 4)
    with pytest.raises(ValueError):
        SK.subcount_params(0, 10)
    with pytest.raises(ValueError):
        SK.subcount_params(11, 10)
    with pytest.raises(ValueError):
        SK.subcount_params(5, 10, 3)


@pytest.mark.parametrize("m,tau,k", [(6, 2, 2), (100, 5, 0), (20000, 256, 4), (30, 30, 0)])
def test_subcount_exact_structure(m, tau, k):
    """S^T = Sigma D I_C: s distinct coordinates, every bucket exactly k of them,
    signs +-1; positions j go to bucket j // k in selection order (Eq. Sigmacount)."""
    s, kk = SK.subcount_params(tau, m, k)
    sk = SK.draw("subcount", m, tau, 4, 99, k)
    S = SK.materialize(sk).toarray()
    assert len(set(sk["coord"].tolist())) == s
    assert np.all((S != 0).sum(axis=0) == kk)          # each row of S^T: exactly k non-zeros
    assert np.all((S != 0).sum(axis=1) <= 1)
    assert set(np.unique(S[S != 0]).tolist()) <= {-1.0, 1.0}
    sel = SK.select_smallest_keys(m, s, 4, 99)
    assert sk["coord"].tolist() == sel.tolist()
    assert sk["bucket"].tolist() == [j // kk for j in range(s)]
    key = seed_key(99)
    for j in range(min(s, 20)):
        x, _, _, _ = _py_philox([int(sk["coord"][j]), 4, 2, 0], key)
        assert sk["sign"][j] == 1 - 2 * (x & 1)


@pytest.mark.parametrize("kind", ["subsample", "count", "subcount"])
def test_materialize_matches_entrywise_application(kind):
    """S^T A, S^T A S, S^T r by explicit entry loops equal the materialised products (m <= 16)."""
    rng = np.random.default_rng(3)
    m, tau = 16, 4
    M = rng.standard_normal((m, m))
    A = M @ M.T + np.eye(m)
    r = rng.standard_normal(m)
    sk = SK.draw(kind, m, tau, 1, 42, 2 if kind == "subcount" else 0)
    SA = np.zeros((tau, m))
    Sr = np.zeros(tau)
    for c, b, s in zip(sk["coord"], sk["bucket"], sk["sign"]):
        SA[b] += s * A[c]
        Sr[b] += s * r[c]
    SAS = np.zeros((tau, tau))
    for c, b, s in zip(sk["coord"], sk["bucket"], sk["sign"]):
        SAS[:, b] += s * SA[:, c]
    S = SK.materialize(sk)
    assert np.allclose(S.T @ A, SA, rtol=0, atol=1e-12)
    assert np.allclose(S.T @ A @ S, SAS, rtol=0, atol=1e-12)
    assert np.allclose(S.T @ r, Sr, rtol=0, atol=1e-12)


def test_empty_buckets_detected():
    found = False
    for it in range(200):
        sk = SK.draw("count", 50, 10, it, 0)
        e = SK.empty_buckets(sk)
        S = SK.materialize(sk).toarray()
        assert np.array_equal(e, np.flatnonzero((S != 0).sum(axis=0) == 0))
        found |= e.size > 0
    assert found   # m=50, tau=10: ~5% of draws have an empty bucket (R4)
