"""C-ABI library: loads, exports every symbol include/ridgesketch.h declares, host-only helpers,
argument validation before any GPU work, and loud failure (RS_ECUDA) without a GPU."""

import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ridgesketch.h")


@pytest.fixture(scope="module")
def rs():
    from paper_2105_05565_b200 import build
    build()
    from paper_2105_05565_b200 import ridgesketch
    return ridgesketch


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rs_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_boundary():
    fns = _declared_functions()
    for f in ("rs_create_dense", "rs_create_csr", "rs_solve", "rs_destroy", "rs_status_string",
              "rs_last_error", "rs_sketch_draw", "rs_get_state"):
        assert f in fns


def test_library_exports_every_declared_symbol(rs):
    lib = C.CDLL(rs.LIB_PATH)
    missing = [f for f in _declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_abi_version_and_status_strings(rs):
    assert rs.rs_abi_version() == 5
    assert rs.rs_status_string(0) == "RS_OK"
    for s in range(1, 8):
        assert rs.rs_status_string(s).startswith("RS_E")


def test_shard_range(rs):
    for total in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            spans = [rs.rs_shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0
            assert sum(n for _, n in spans) == total
            for (b0, n0), (b1, _) in zip(spans, spans[1:]):
                assert b0 + n0 == b1
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1


def test_shard_rows_nnz(rs):
    rng = np.random.default_rng(0)
    counts = rng.integers(0, 100, size=1000)
    counts[:10] = 5000   # heavy head
    rowptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    for world in (1, 2, 4, 8):
        spans = [rs.rs_shard_rows_nnz(rowptr, r, world) for r in range(world)]
        assert spans[0][0] == 0 and sum(n for _, n in spans) == 1000
        for (b0, n0), (b1, _) in zip(spans, spans[1:]):
            assert b0 + n0 == b1
        loads = [rowptr[b + n] - rowptr[b] for b, n in spans]
        assert max(loads) <= rowptr[-1] / world + counts.max()


def test_validation_before_gpu(rs):
    X = np.zeros((3, 2))
    y = np.zeros(3)
    with pytest.raises(rs.RSError) as e:
        rs.rs_create_dense(X, y, 0.0)          # lambda must be > 0
    assert e.value.status == rs.RS_EINVAL
    with pytest.raises(rs.RSError) as e:
        rs.rs_create_dense(np.zeros((0, 2)), np.zeros(0), 1.0)
    assert e.value.status == rs.RS_EINVAL
    with pytest.raises(rs.RSError) as e:
        rs.rs_create_csr(3, 2, np.array([0, 1, 1, 1]), np.array([0], np.int32), np.ones(1),
                         y, -1.0, mode="explicit")
    assert e.value.status == rs.RS_EINVAL
    with pytest.raises(rs.RSError) as e:
        rs.rs_create_kernel(X, y, 1.0, 0.0)    # sigma must be > 0
    assert e.value.status == rs.RS_EINVAL
    with pytest.raises(rs.RSError) as e:
        rs.rs_sketch_draw("count", 10, 11, 0, 0)   # tau > m
    assert e.value.status == rs.RS_EINVAL


def test_no_cpu_fallback_without_gpu(rs):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(rs.RSError) as e:
        rs.rs_create_dense(np.ones((4, 2)), np.ones(4), 1.0)
    assert e.value.status == rs.RS_ECUDA
    with pytest.raises(rs.RSError) as e:
        rs.rs_sketch_draw("subsample", 10, 3, 0, 0)
    assert e.value.status == rs.RS_ECUDA


def test_host_coll_id(rs):
    """Group names of the host-staged collective (RS_COLL_HOST): distinct, NUL-terminated, a POSIX
    shared-memory name (leading '/', no other '/')."""
    a, b = rs.rs_host_coll_id(), rs.rs_host_coll_id()
    assert a != b and len(a) == 128
    name = a.split(b"\0")[0].decode()
    assert name.startswith("/") and "/" not in name[1:] and 1 < len(name) < 100
