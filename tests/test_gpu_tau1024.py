"""GPU parity at the production sketch size of BASELINE.json c5 (tau = 1024, m = d = 4096).

c5 itself is 2e6 x 4096 (65.5 GB); the oracle cannot iterate on it, so these cases keep c5's
m = 4096, tau = 1024, column decay j^(-1/2), lambda = 1e-4 n and beta = 0.5 and reduce n to 20000
(the per-iteration tau x tau system, the large-tau factorisation slots, the M = 1024 DMMA
contraction and the lower-tile Gram GEMM are exactly c5's; only the K extent of the X contractions
is shorter).  Every GPU mode (IMPLICIT, GRAM, EXPLICIT) runs 50 iterations of Alg. 2
and is compared with the oracle's iterates (one oracle run per sketch kind, explicit A: the
oracle's implicit and explicit AS agree to rounding, pin P13) normwise and elementwise at 1e-10
(tests/parity_util.py, R18/R27).  Count (tau = 1000) and SubCount (tau = 1000, k = 2)
cover the other sketch kinds at the same scale."""

import numpy as np
import pytest
import torch

import rsinputs
from oracle import solver as OV
from parity_util import assert_close

pytestmark = pytest.mark.gpu

N, D, ITERS = 20000, 4096, 50
LAM = 1e-4 * N
CASES = {"subsample": (1024, 0), "count": (1000, 0), "subcount": (1000, 2)}


@pytest.fixture(scope="module")
def rs():
    from paper_2105_05565_b200 import build
    build()
    from paper_2105_05565_b200 import ridgesketch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return ridgesketch


@pytest.fixture(scope="module")
def data():
    X, y = rsinputs.dense_problem(N, D, seed=11, col_decay=True, noise=0.01)
    return X.numpy(), y.numpy()


_ORACLE = {}


def oracle(data, kind):
    if kind not in _ORACLE:
        X, y = data
        tau, k = CASES[kind]
        _ORACLE[kind] = OV.solve(X, y, LAM, kind, tau, 1.0, 0.5, 0.0, ITERS, seed=3, subcount_k=k,
                                 explicit=True)
    return _ORACLE[kind]


@pytest.mark.parametrize("mode", ["explicit", "gram", "implicit"])
@pytest.mark.parametrize("kind", ["subsample", "count", "subcount"])
def test_c5_shape_tau1024_50_steps(rs, data, kind, mode):
    X, y = data
    tau, k = CASES[kind]
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    h = rs.rs_create_dense(Xd, yd, LAM, mode=mode, borrow=True)
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, ITERS, seed=3, subcount_k=k)
        _, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = oracle(data, kind)
    assert rep["iterations"] == ITERS
    assert_close(w, ref["w"], 1e-10, f"{mode}/{kind} w")
    assert_close(r, ref["r"], 1e-10, f"{mode}/{kind} r")
