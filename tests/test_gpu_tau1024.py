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


# ---------------------------------------------------------------- overlapped pipeline, many groups
OV_ITERS = 520   # > 2 groups of P = 2 (num_sms - 32) = 232 slots on a 148-SM B200

_OV_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import rsinputs
from paper_2105_05565_b200 import build
build()
from paper_2105_05565_b200 import ridgesketch as rs
X, y = rsinputs.dense_problem(int(sys.argv[3]), int(sys.argv[4]), seed=11, col_decay=True, noise=0.01)
h = rs.rs_create_dense(X.cuda(), y.cuda(), float(sys.argv[5]), mode="explicit", borrow=True)
w, rep = rs.rs_solve(h, "subsample", 1024, 1.0, 0.5, 0.0, int(sys.argv[6]), seed=3)
_, r = rs.rs_get_state(h)
rs.rs_destroy(h)
assert rep["overlap_sms"] > 0, rep
np.savez(sys.argv[2], w=w, r=r, nb=rep["inverse_blocks"])
"""


def _ov_oracle(data, kind):
    key = ("ov", kind)
    if key not in _ORACLE:
        X, y = data
        tau, k = CASES[kind]
        _ORACLE[key] = OV.solve(X, y, LAM, kind, tau, 1.0, 0.5, 0.0, OV_ITERS, seed=3, subcount_k=k,
                                explicit=True)
    return _ORACLE[key]


@pytest.mark.parametrize("kind", ["subsample", "count", "subcount"])
def test_c5_shape_overlapped_groups(rs, data, kind):
    """EXPLICIT at c5's tau with a subsample sketch runs the overlapped pipeline: the
    first set's first num_sms slots are factored up front and the rest beside the first group
    (per-slot ready flags), then every group's k_iterate on OV_SMS SMs runs beside the next group's
    two-per-SM factorisation, whose CTAs claim slots and step aside on SMs beyond the budget.  520
    iterations cross two group boundaries and every slot of both sets (count: the slots' rows of
    A S^T, also for the first set's tail); the iterates equal the oracle's (1e-9: 520 steps of
    rounding)."""
    X, y = data
    tau, k = CASES[kind]
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    h = rs.rs_create_dense(Xd, yd, LAM, mode="explicit", borrow=True)
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, OV_ITERS, seed=3, subcount_k=k)
        _, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    assert rep["iterations"] == OV_ITERS
    # c5's subsample sketch runs the overlapped pipeline (the SM split is the engine's model)
    assert kind != "subsample" or rep["overlap_sms"] > 0, rep["overlap_sms"]
    assert rep["inverse_blocks"] == 2, rep["inverse_blocks"]   # tau >= 512: two super-blocks
    ref = _ov_oracle(data, kind)
    assert_close(w, ref["w"], 1e-9, f"{kind} w")
    assert_close(r, ref["r"], 1e-9, f"{kind} r")


@pytest.mark.parametrize("env", [{"RS_OV_SPLIT": "0"}, {"RS_BF_DUAL": "0"}, {"RS_SB_NB": "1"},
                                 {"RS_SB_NB": "3"}, {"RS_SB_NB": "6", "RS_BF_DUAL": "0"}])
def test_c5_shape_overlapped_switches(tmp_path, data, env):
    """The process-wide A/B switches of the overlapped pipeline (read once per process, so in a
    child): the whole first set up front (RS_OV_SPLIT=0), the 8-warp one-slot-per-SM
    factorisation (RS_BF_DUAL=0) and the blocked inverse's super-block count (RS_SB_NB: 1 = the
    full W = L^{-1}; 3 = blocks of 384, 384, 256; 6 = five of 192 and one of 64)
    give the oracle's iterates too (the default is 2 blocks of 512)."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outp = tmp_path / "ov.npz"
    res = subprocess.run([sys.executable, "-c", _OV_CHILD, root, str(outp), str(N), str(D), repr(LAM),
                          str(OV_ITERS)], env=dict(os.environ, **env), capture_output=True, text=True,
                         timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    got = np.load(outp)
    assert int(got["nb"]) == int(env.get("RS_SB_NB", 2)), int(got["nb"])
    ref = _ov_oracle(data, "subsample")
    assert_close(got["w"], ref["w"], 1e-9, f"{env} w")
    assert_close(got["r"], ref["r"], 1e-9, f"{env} r")
