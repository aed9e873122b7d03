"""Pins for oracle/philox.py: published known-answer vectors and the CUDA toolkit's
curand_Philox4x32_10 compiled for the host (an independent library implementation)."""

import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle.philox import philox4x32_10, seed_key

HERE = os.path.dirname(os.path.abspath(__file__))


def _kat_rows():
    rows = []
    with open(os.path.join(HERE, "golden", "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                rows.append([int(t, 16) for t in line.split()])
    return rows


def test_known_answer_vectors():
    rows = _kat_rows()
    assert len(rows) == 3
    for r in rows:
        out = philox4x32_10(*r[:6])
        assert [int(v) for v in out] == r[6:]


@pytest.fixture(scope="module")
def curand_host(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = str(tmp_path_factory.mktemp("curand") / "curand_philox_host")
    subprocess.run([nvcc, "-O2", "-Wno-deprecated-gpu-targets", "-o", exe,
                    os.path.join(HERE, "tools", "curand_philox_host.cu")], check=True,
                   capture_output=True)
    return exe


def test_matches_curand_host_grid(curand_host):
    rng = np.random.default_rng(7)
    n = 4000
    a = rng.integers(0, 2**32, size=(n, 6), dtype=np.uint64)
    a[:100, 1:4] = 0                      # sketch-stream shaped counters (i, k, stream, 0)
    a[:100, 0] = np.arange(100)
    a[:100, 2] = 2
    text = "\n".join(" ".join(str(int(v)) for v in row) for row in a) + "\n"
    res = subprocess.run([curand_host], input=text, capture_output=True, text=True, check=True)
    ref = np.array([[int(t) for t in line.split()] for line in res.stdout.strip().splitlines()],
                   dtype=np.uint64)
    out = np.stack(philox4x32_10(a[:, 0], a[:, 1], a[:, 2], a[:, 3], a[:, 4], a[:, 5]), axis=1)
    assert out.shape == ref.shape
    assert np.array_equal(out, ref)


def test_seed_key_split():
    assert seed_key(0) == (0, 0)
    assert seed_key((5 << 32) | 7) == (7, 5)
    assert seed_key(2**64 - 1) == (2**32 - 1, 2**32 - 1)
