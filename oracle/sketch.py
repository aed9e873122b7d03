"""Sketching matrices S in R^{m x tau} (Definition "sketching matrix").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Three kinds are on the hot path:

* Subsample (Eq. subsample): S = I_C, C a uniformly random tau-subset of [m].
* Count: every coordinate i is sent to a uniformly random bucket h(i) in [tau]
  with a random sign sigma(i) (reading R4: hashed, no subsampling).
* SubCount (Eq. Sigmacount): S^T = Sigma D I_C with |C| = s = k*tau; the s selected
  coordinates, in selection (key) order, are summed k at a time (bucket = position // k) with
  random signs (reading R5).

The randomness follows the sketch-stream contract of DESIGN.md §3, written here from its
statement (integer arithmetic only):

* key = (seed mod 2**32, seed >> 32); counter = (coordinate i, iteration it, stream, 0).
* stream 0, selection: key64_i = (x << 32) | y; the selected set is the tau (or s) indices
  with the smallest (key64_i, i), listed in that ascending order.
* stream 1, count: h(i) = floor(x * tau / 2**32), sigma(i) = 1 - 2*(y & 1).
* stream 2, subcount sign of the selected coordinate c: sigma = 1 - 2*(x & 1) from counter
  (c, it, 2, 0).

A sketch is returned as the list of its non-zero entries (coord, bucket, sign): S has
S[coord_e, bucket_e] = sign_e and no other non-zeros.  ``materialize`` builds S explicitly.
"""

import numpy as np
import scipy.sparse as sp

from .philox import philox4x32_10, seed_key

SUBSAMPLE, COUNT, SUBCOUNT = "subsample", "count", "subcount"
STREAM_SELECT, STREAM_COUNT, STREAM_SUBCOUNT_SIGN = 0, 1, 2


def subcount_params(tau, m, k=0):
    """(s, k) of the SubCount sketch: if 10*tau <= m then k = 10, else k = floor(m/tau);
    s = k*tau.  A caller-given k > 0 overrides the rule (reading R6, config c4)."""
    if not 1 <= tau <= m:
        raise ValueError("tau must be in [1, m]")
    if k <= 0:
        k = 10 if 10 * tau <= m else m // tau
    s = k * tau
    if s > m:
        raise ValueError("subcount s = k*tau exceeds m")
    return s, k


def _stream(m_idx, it, stream, seed):
    k0, k1 = seed_key(seed)
    i = np.asarray(m_idx, dtype=np.uint64)
    return philox4x32_10(i, np.uint64(it), np.uint64(stream), np.uint64(0), k0, k1)


def select_smallest_keys(m, count, it, seed):
    """The `count` indices of [0, m) with the smallest (key64_i, i), in ascending order."""
    i = np.arange(m, dtype=np.uint64)
    x, y, _, _ = _stream(i, it, STREAM_SELECT, seed)
    key64 = (x << np.uint64(32)) | y
    order = np.lexsort((i, key64))          # primary key64, ties broken by i
    return order[:count].astype(np.int64)


def draw(kind, m, tau, it, seed, subcount_k=0):
    """Draw S_it (Alg. 2 line "Sample an independent copy S_k ~ D").

    Returns dict(kind, m, tau, coord, bucket, sign) with int64 coord/bucket and float64 sign.
    """
    if not 1 <= tau <= m:
        raise ValueError("tau must be in [1, m]")
    if kind == SUBSAMPLE:
        coord = select_smallest_keys(m, tau, it, seed)
        bucket = np.arange(tau, dtype=np.int64)
        sign = np.ones(tau)
    elif kind == COUNT:
        coord = np.arange(m, dtype=np.int64)
        x, y, _, _ = _stream(coord, it, STREAM_COUNT, seed)
        bucket = ((x * np.uint64(tau)) >> np.uint64(32)).astype(np.int64)
        sign = 1.0 - 2.0 * (y & np.uint64(1)).astype(np.float64)
    elif kind == SUBCOUNT:
        s, k = subcount_params(tau, m, subcount_k)
        coord = select_smallest_keys(m, s, it, seed)
        bucket = np.arange(s, dtype=np.int64) // k
        x, _, _, _ = _stream(coord, it, STREAM_SUBCOUNT_SIGN, seed)
        sign = 1.0 - 2.0 * (x & np.uint64(1)).astype(np.float64)
    else:
        raise ValueError(f"unknown sketch kind {kind!r}")
    return dict(kind=kind, m=m, tau=tau, coord=coord, bucket=bucket, sign=sign)


def materialize(sk):
    """Explicit S (m x tau, scipy CSC) with S[coord_e, bucket_e] = sign_e."""
    return sp.csc_matrix((sk["sign"], (sk["coord"], sk["bucket"])), shape=(sk["m"], sk["tau"]))


def empty_buckets(sk):
    """Buckets (columns of S) with no non-zero: possible for the count sketch only."""
    used = np.zeros(sk["tau"], dtype=bool)
    used[sk["bucket"]] = True
    return np.flatnonzero(~used)
