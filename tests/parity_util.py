"""Comparison helpers of the GPU parity tests (reading R27).

`assert_close(got, ref, tol)` checks BOTH
  * normwise:    ||got - ref||_2 / ||ref||_2 <= tol                         (BASELINE.json, R18)
  * elementwise: |got_i - ref_i| <= tol * max(|ref_i|, rms(ref))  for every i   (R27)
The elementwise bound catches a few wrong coordinates that a norm ratio hides; its floor rms(ref)
= ||ref||_2 / sqrt(len) keeps coordinates that are zero up to rounding from failing on relative
noise.  It is stricter than the normwise bound by up to sqrt(len)."""

import numpy as np


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def elementwise(a, b):
    """max_i |a_i - b_i| / max(|b_i|, rms(b))."""
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    if b.size == 0:
        return 0.0
    rms = np.linalg.norm(b) / np.sqrt(b.size)
    floor = np.maximum(np.abs(b), rms if rms > 0 else 1.0)
    return float(np.max(np.abs(a - b) / floor))


def assert_close(got, ref, tol, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    assert np.all(np.isfinite(got)), (what, "non-finite entries")
    nr, ew = rel(got, ref), elementwise(got, ref)
    assert nr <= tol and ew <= tol, f"{what}: normwise {nr:.3e}, elementwise {ew:.3e} > {tol:.1e}"
