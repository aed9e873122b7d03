"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element, on the
same seeded inputs.  Tolerances: sketches bit-exact; w and r after 50 steps within
1e-10 relative (BASELINE.json); final w within 1e-6 of the direct solve (c1)."""

import numpy as np
import pytest
import scipy.sparse as sp
import torch

import rsinputs
from oracle import problem as OP
from oracle import sketch as OS
from oracle import solver as OV
from parity_util import assert_close, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rs():
    from paper_2105_05565_b200 import build
    build()
    from paper_2105_05565_b200 import ridgesketch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return ridgesketch




# ---------------------------------------------------------------------------------- a1 sketches
SKETCH_CASES = [
    ("subsample", 50, 10, 0), ("subsample", 2000, 200, 0), ("subsample", 4096, 1024, 0),
    ("subsample", 37, 37, 0), ("subsample", 1, 1, 0), ("subsample", 20000, 1, 0),
    ("subsample", 50000, 777, 0), ("count", 6, 2, 0), ("count", 50, 10, 0),
    ("count", 50000, 500, 0), ("count", 1000, 1, 0), ("count", 3000, 1536, 0),
    ("subcount", 20000, 256, 4), ("subcount", 100, 5, 0), ("subcount", 30, 30, 0),
    ("subcount", 2000, 64, 0)]


@pytest.mark.parametrize("kind,m,tau,k", SKETCH_CASES)
def test_sketch_bit_exact(rs, kind, m, tau, k):
    for seed, it in ((0, 0), (0, 1), (12345, 7), (2**40 + 5, 123456)):
        coord, bucket, sign = rs.rs_sketch_draw(kind, m, tau, seed, it, k)
        ref = OS.draw(kind, m, tau, it, seed, k)
        if kind == "count":
            # GPU entries are in bucket order (ascending coordinate within a bucket)
            order = np.lexsort((ref["coord"], ref["bucket"]))
            assert np.array_equal(coord, ref["coord"][order])
            assert np.array_equal(bucket, ref["bucket"][order])
            assert np.array_equal(sign.astype(np.float64), ref["sign"][order])
        else:
            assert np.array_equal(coord, ref["coord"])
            assert np.array_equal(bucket, ref["bucket"])
            assert np.array_equal(sign.astype(np.float64), ref["sign"])


# ---------------------------------------------------------------------------------- dense paths
def _dense(n, d, seed=0, col_decay=False, noise=0.1):
    X, y = rsinputs.dense_problem(n, d, seed=seed, col_decay=col_decay, noise=noise)
    return X.numpy(), y.numpy()


def _run_gpu_dense(rs, X, y, lam, mode, kind, tau, beta, iters, seed=0, k=0, device_input=False):
    if device_input:
        h = rs.rs_create_dense(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), lam, mode=mode)
    else:
        h = rs.rs_create_dense(X, y, lam, mode=mode)
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, beta, 0.0, iters, seed, k, check_every=7)
        ws, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    return w, r, rep


@pytest.mark.parametrize("beta", [0.0, 0.5])
@pytest.mark.parametrize("mode", ["implicit", "explicit", "gram"])
def test_config1_50_steps(rs, beta, mode):
    cfg = rsinputs.CONFIGS["c1"]
    X, y = _dense(cfg.n, cfg.d, noise=cfg.noise)
    w, r, rep = _run_gpu_dense(rs, X, y, cfg.lam, mode, "subsample", cfg.tau, beta, 50)
    ref = OV.solve(X, y, cfg.lam, "subsample", cfg.tau, 1.0, beta, 0.0, 50, seed=0)
    assert rep["iterations"] == 50
    assert_close(w, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


@pytest.mark.parametrize("mode", ["implicit", "explicit", "gram"])
def test_config1_final_vs_direct(rs, mode):
    cfg = rsinputs.CONFIGS["c1"]
    X, y = _dense(cfg.n, cfg.d, noise=cfg.noise)
    w, r, rep = _run_gpu_dense(rs, X, y, cfg.lam, mode, "subsample", cfg.tau, 0.0, 300)
    pr = OP.build(X, y, cfg.lam)
    w_star = OP.direct_solve(pr["A"], pr["b"])
    assert rep["iterations"] == 300
    assert_close(w, w_star, 1e-6)
    w5, _, _ = _run_gpu_dense(rs, X, y, cfg.lam, mode, "subsample", cfg.tau, 0.5, 1000)
    assert_close(w5, w_star, 1e-6)


@pytest.mark.parametrize("kind,tau,k", [("subsample", 37, 0), ("count", 37, 0), ("subcount", 29, 3),
                                        ("subsample", 130, 0), ("count", 300, 0)])
@pytest.mark.parametrize("mode", ["implicit", "explicit", "gram"])
def test_dense_ragged_parity(rs, kind, tau, k, mode):
    """Several GEMM tiles (64 x 128) with ragged tails, split-K, all sketch kinds."""
    X, y = _dense(3001, 301, seed=3, col_decay=True, noise=0.01)
    lam = 0.3
    w, r, rep = _run_gpu_dense(rs, X, y, lam, mode, kind, tau, 0.5, 12, seed=5, k=k,
                               device_input=True)
    ref = OV.solve(X, y, lam, kind, tau, 1.0, 0.5, 0.0, 12, seed=5, subcount_k=k)
    assert rep["iterations"] == 12
    assert_close(w, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


@pytest.mark.parametrize("mode", ["implicit", "explicit", "gram"])
def test_dense_count_empty_buckets(rs, mode):
    """c1 shape with the count sketch (m = 50, tau = 10): ~5% of iterations have an empty bucket,
    exercising the empty-bucket rule (R3) in every factorisation path."""
    cfg = rsinputs.CONFIGS["c1"]
    X, y = _dense(cfg.n, cfg.d, noise=cfg.noise)
    w, r, rep = _run_gpu_dense(rs, X, y, cfg.lam, mode, "count", cfg.tau, 0.5, 60, seed=2)
    ref = OV.solve(X, y, cfg.lam, "count", cfg.tau, 1.0, 0.5, 0.0, 60, seed=2)
    assert rep["iterations"] == 60
    assert_close(w, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


@pytest.mark.parametrize("mode", ["explicit", "gram"])
@pytest.mark.parametrize("check_every", [1, 64, 300])
def test_sketch_ahead_group_sizes(rs, mode, check_every):
    """Sketch-ahead pipeline (bfactor.cu): groups of 1, 64 and > num_SMs slots (clamped) give the
    oracle's iterates; 150 iterations cross several group and graph-launch boundaries."""
    X, y = _dense(2000, 160, seed=7, col_decay=True, noise=0.01)
    h = rs.rs_create_dense(X, y, 0.7, mode=mode)
    try:
        w, rep = rs.rs_solve(h, "subsample", 48, 1.0, 0.5, 0.0, 150, 11, check_every=check_every)
        _, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(X, y, 0.7, "subsample", 48, 1.0, 0.5, 0.0, 150, seed=11)
    assert rep["iterations"] == 150
    assert_close(w, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


def test_dense_identity_sketch_one_step_explicit(rs):
    """S = I (tau = m): one step solves A w = b exactly through the batched factor."""
    X, y = _dense(400, 64, seed=4)
    w, r, rep = _run_gpu_dense(rs, X, y, 0.5, "explicit", "subsample", 64, 0.0, 1)
    pr = OP.build(X, y, 0.5)
    assert_close(w, OP.direct_solve(pr["A"], pr["b"]), 1e-11)
    assert np.linalg.norm(r) <= 1e-11 * np.linalg.norm(pr["b"])


def test_dense_identity_sketch_one_step(rs):
    X, y = _dense(400, 64, seed=4)
    w, r, rep = _run_gpu_dense(rs, X, y, 0.5, "implicit", "subsample", 64, 0.0, 1)
    pr = OP.build(X, y, 0.5)
    w_star = np.linalg.solve(pr["A"], pr["b"])
    assert_close(w, w_star, 1e-10)
    assert np.linalg.norm(r) <= 1e-9 * np.linalg.norm(pr["b"])


def test_dense_tau1_coordinate_descent(rs):
    X, y = _dense(200, 20, seed=5)
    w, r, rep = _run_gpu_dense(rs, X, y, 0.2, "implicit", "subsample", 1, 0.3, 40, seed=17)
    ref = OV.solve(X, y, 0.2, "subsample", 1, 1.0, 0.3, 0.0, 40, seed=17)
    assert_close(w, ref["w"], 1e-10)


def test_tolerance_stop_iteration_count(rs):
    X, y = _dense(2000, 100, seed=6, col_decay=True)
    h = rs.rs_create_dense(X, y, 1.0)
    try:
        w, rep = rs.rs_solve(h, "subsample", 20, 1.0, 0.5, 1e-6, 100000, 3, trace_cap=5000)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(X, y, 1.0, "subsample", 20, 1.0, 0.5, 1e-6, 100000, seed=3, trace=True)
    assert rep["converged"] and ref["converged"]
    assert abs(rep["iterations"] - ref["iterations"]) <= 1
    n = min(len(rep["trace"]), len(ref["trace"]))
    assert np.allclose(rep["trace"][:n], ref["trace"][:n], rtol=1e-8, atol=0)
    assert_close(w, ref["w"], 1e-8)


def test_zero_rhs_and_zero_iterations(rs):
    X, _ = _dense(50, 5)
    h = rs.rs_create_dense(X, np.zeros(50), 1.0)
    try:
        w, rep = rs.rs_solve(h, "subsample", 2, tol=1e-4, max_iter=100)
        assert rep["iterations"] == 0 and rep["converged"] and np.all(w == 0)
    finally:
        rs.rs_destroy(h)
    h = rs.rs_create_dense(X, np.ones(50), 1.0)
    try:
        w, rep = rs.rs_solve(h, "subsample", 2, tol=0.0, max_iter=0)
        assert rep["iterations"] == 0 and np.all(w == 0)
    finally:
        rs.rs_destroy(h)


def test_invalid_arguments_fail_loudly(rs):
    X, y = _dense(50, 5)
    with pytest.raises(rs.RSError) as e:
        rs.rs_create_dense(np.where(X > 1, np.nan, X), y, 1.0)
    assert e.value.status == rs.RS_EINVAL
    h = rs.rs_create_dense(X, y, 1.0)
    try:
        for kw in (dict(tau=0), dict(tau=6), dict(gamma=0.0), dict(beta=1.5), dict(tol=-1.0)):
            args = dict(kind="subsample", tau=2)
            args.update(kw)
            with pytest.raises(rs.RSError) as e:
                rs.rs_solve(h, **args)
            assert e.value.status == rs.RS_EINVAL
        with pytest.raises(rs.RSError) as e:
            rs.rs_solve(h, "subcount", tau=2, subcount_k=3)      # k tau = 6 > m = 5
        assert e.value.status == rs.RS_EINVAL
    finally:
        rs.rs_destroy(h)


# ---------------------------------------------------------------------------------- CSR paths
def _csr_primal(n=4000, d=600, per_row=12, seed=1):
    rp, ci, v, y = rsinputs.csr_uniform(n, d, per_row, seed=seed)
    return rp, ci, v, y, rsinputs.csr_to_scipy(rp, ci, v, n, d)


@pytest.mark.parametrize("kind,tau,k", [("count", 40, 0), ("subsample", 33, 0), ("subcount", 20, 3),
                                        ("count", 599, 0)])
@pytest.mark.parametrize("mode", ["implicit", "gram"])
def test_csr_primal_parity(rs, kind, tau, k, mode):
    n, d = 4000, 600
    rp, ci, v, y, Xs = _csr_primal(n, d)
    lam = 1e-2
    h = rs.rs_create_csr(n, d, rp, ci, v, y, lam, mode=mode)
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 15, seed=2, subcount_k=k)
        ws, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(Xs, y, lam, kind, tau, 1.0, 0.5, 0.0, 15, seed=2, subcount_k=k)
    assert_close(w, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


@pytest.mark.parametrize("kind,tau,k", [("subcount", 16, 4), ("subsample", 25, 0), ("count", 12, 0),
                                        ("subcount", 240, 1)])
@pytest.mark.parametrize("mode", ["implicit", "gram"])
def test_csr_dual_parity(rs, kind, tau, k, mode):
    n, d = 300, 5000
    rp, ci, v, y = rsinputs.csr_zipf(n, d, 60, a=1.1, seed=3)
    Xs = rsinputs.csr_to_scipy(rp, ci, v, n, d)
    lam = 1e-1
    h = rs.rs_create_csr(n, d, rp, ci, v, y, lam, mode=mode)
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 15, seed=4, subcount_k=k, d=d, alpha=True)
        alpha, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(Xs, y, lam, kind, tau, 1.0, 0.5, 0.0, 15, seed=4, subcount_k=k)
    assert ref["route"] == "dual"
    assert_close(alpha, ref["w"], 1e-10)
    assert_close(rep["alpha"], ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)
    assert_close(w, ref["weights"], 1e-10)


@pytest.mark.parametrize("mode", ["implicit", "gram"])
def test_csr_dual_converges_to_direct(rs, mode):
    n, d = 120, 2000
    rp, ci, v, y = rsinputs.csr_zipf(n, d, 40, a=1.1, seed=5)
    Xs = rsinputs.csr_to_scipy(rp, ci, v, n, d)
    lam = 1.0
    h = rs.rs_create_csr(n, d, rp, ci, v, y, lam, mode=mode)
    try:
        w, rep = rs.rs_solve(h, "subcount", 12, 1.0, 0.5, 1e-12, 200000, seed=1, subcount_k=4, d=d)
    finally:
        rs.rs_destroy(h)
    X = Xs.toarray()
    pr = OP.build(X, y, lam, "primal")
    w_star = np.linalg.solve(pr["A"], pr["b"])
    assert rep["converged"]
    assert_close(w, w_star, 1e-6)


# ---------------------------------------------------------------------------------- full size
@pytest.mark.parametrize("mode", ["implicit", "gram"])
def test_config2_full_size_sampled(rs, mode):
    """BASELINE.json c2 at full size (1e5 x 2000, tau=200), the launch configuration bench.py
    times: the first 3 iterations equal the oracle's (same X bytes, host copy)."""
    cfg = rsinputs.CONFIGS["c2"]
    Xd, yd = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, col_decay=True, noise=cfg.noise,
                                    device="cuda")
    h = rs.rs_create_dense(Xd, yd, cfg.lam, mode=mode, borrow=True)
    try:
        w, rep = rs.rs_solve(h, "subsample", cfg.tau, 1.0, cfg.beta, 0.0, 3, seed=0)
        _, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    X, y = Xd.cpu().numpy(), yd.cpu().numpy()
    del Xd, yd
    ref = OV.solve(X, y, cfg.lam, "subsample", cfg.tau, 1.0, cfg.beta, 0.0, 3, seed=0)
    assert_close(w, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


@pytest.mark.parametrize("kind,tau,k", [("count", 64, 0), ("subsample", 150, 0), ("subcount", 50, 4)])
@pytest.mark.parametrize("mode", ["implicit", "gram"])
def test_csr_primal_long_rows(rs, kind, tau, k, mode):
    """Rows longer than a warp (c3 has ~50 non-zeros per row): multi-chunk merge of equal buckets."""
    n, d = 3000, 400
    rp, ci, v, y, Xs = _csr_primal(n, d, per_row=70, seed=7)
    lam = 1e-2
    h = rs.rs_create_csr(n, d, rp, ci, v, y, lam, mode=mode)
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 12, seed=3, subcount_k=k)
        ws, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(Xs, y, lam, kind, tau, 1.0, 0.5, 0.0, 12, seed=3, subcount_k=k)
    assert_close(w, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


@pytest.mark.parametrize("scale", [1e-50, 1e50])
def test_csr_gram_fixed_point_scale_invariance(rs, scale):
    """The CSR Gram's fixed-point scale follows trace(G) (DESIGN R26): data scaled by 1e+-50
    (lambda by scale^2) gives the oracle's iterates, primal (count: full scan) and dual
    (SubCount: the selected-row path's trace bound).  (The residual norms are plain fp64 sums of
    squares: a primal b = X^T y scales as scale^2 and ||b||^2 as scale^4, so 1e+-100 would leave
    the fp64 range there, in any mode.)"""
    n, d = 3000, 400
    rp, ci, v, y, Xs = _csr_primal(n, d, per_row=70, seed=12)
    lam = 1e-2 * scale * scale
    h = rs.rs_create_csr(n, d, rp, ci, v * scale, y * scale, lam, mode="gram")
    try:
        w, _ = rs.rs_solve(h, "count", 64, 1.0, 0.5, 0.0, 12, seed=5)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(Xs * scale, y * scale, lam, "count", 64, 1.0, 0.5, 0.0, 12, seed=5)
    assert_close(w, ref["w"], 1e-10)
    n, d = 300, 5000
    rp, ci, v, y = rsinputs.csr_zipf(n, d, 60, a=1.1, seed=3)
    Xs = rsinputs.csr_to_scipy(rp, ci, v, n, d)
    h = rs.rs_create_csr(n, d, rp, ci, v * scale, y * scale, lam, mode="gram")
    try:
        w, _ = rs.rs_solve(h, "subcount", 16, 1.0, 0.5, 0.0, 12, seed=6, subcount_k=4, d=d)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(Xs * scale, y * scale, lam, "subcount", 16, 1.0, 0.5, 0.0, 12, seed=6,
                   subcount_k=4)
    assert ref["route"] == "dual"
    assert_close(w, ref["weights"], 1e-10)


def test_csr_primal_gram_bitwise_reproducible(rs):
    """CSR primal GRAM with a count sketch: row hashing merges in a fixed lane order, the Gram bands
    are exact int64 fixed-point sums (DESIGN R26), the band partials are reduced in chunk order and
    the SpMVs have fixed per-row order, so two solves give bit-identical iterates (the fp64 CAS
    adds this replaced did not).  Rows of 70 entries exercise the staged pair loop."""
    n, d = 3000, 400
    rp, ci, v, y, Xs = _csr_primal(n, d, per_row=70, seed=11)
    h = rs.rs_create_csr(n, d, rp, ci, v, y, 1e-2, mode="gram")
    try:
        w1, _ = rs.rs_solve(h, "count", 64, 1.0, 0.5, 0.0, 30, seed=4)
        w2, _ = rs.rs_solve(h, "count", 64, 1.0, 0.5, 0.0, 30, seed=4)
    finally:
        rs.rs_destroy(h)
    assert np.array_equal(w1, w2)
    ref = OV.solve(Xs, y, 1e-2, "count", 64, 1.0, 0.5, 0.0, 30, seed=4)
    assert_close(w1, ref["w"], 1e-10)


@pytest.mark.parametrize("kind,tau,k", [("subsample", 260, 0), ("count", 300, 0), ("subcount", 230, 2)])
@pytest.mark.parametrize("mode", ["explicit", "gram"])
def test_dense_large_tau_sketch_ahead(rs, kind, tau, k, mode):
    """tau > 224: the sketch-ahead pipeline gathers G_k into a per-slot work matrix (k_bf_gather) and
    factors it there (k_bfactor_lp: 32 x 32 DMMA tiles, block-column pairs, ragged tau padded with an
    identity tail)."""
    n, d = 3000, 700
    X, y = rsinputs.dense_problem(n, d, seed=11)
    X, y = X.numpy(), y.numpy()
    w, r, rep = _run_gpu_dense(rs, X, y, 0.5, mode, kind, tau, 0.5, 10, seed=6, k=k)
    ref = OV.solve(X, y, 0.5, kind, tau, 1.0, 0.5, 0.0, 10, seed=6, subcount_k=k)
    assert_close(w, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


@pytest.mark.parametrize("kind,tau,k", [("subsample", 260, 0), ("count", 250, 0), ("subcount", 230, 2)])
def test_explicit_overlapped_groups(rs, kind, tau, k):
    """EXPLICIT with tau > 224 runs the overlapped two-set pipeline: the next group's factorisation
    (k_bf_gather + k_bfactor_lp on a second stream) concurrent with the current group's iterations
    (k_iterate on the SMs left free).  300 iterations cross two group boundaries (P = num_sms - 24);
    a tolerance-stopped solve ends inside a group while the next group is being factored (the factor
    kernels poll the stop flag)."""
    X, y = rsinputs.dense_problem(3000, 700, seed=12, col_decay=True, noise=0.01)
    X, y = X.numpy(), y.numpy()
    h = rs.rs_create_dense(X, y, 0.5, mode="explicit")
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 300, 9, k)
        _, r = rs.rs_get_state(h)
        w2, rep2 = rs.rs_solve(h, kind, tau, 1.0, 0.5, 1e-9, 5000, 9, k, trace_cap=5000)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(X, y, 0.5, kind, tau, 1.0, 0.5, 0.0, 300, seed=9, subcount_k=k, explicit=True)
    assert rep["iterations"] == 300
    assert_close(w, ref["w"], 1e-9)
    assert_close(r, ref["r"], 1e-9)
    ref2 = OV.solve(X, y, 0.5, kind, tau, 1.0, 0.5, 1e-9, 5000, seed=9, subcount_k=k, explicit=True)
    assert abs(rep2["iterations"] - ref2["iterations"]) <= 1 and rep2["converged"]
    assert_close(w2, ref2["w"] if rep2["iterations"] == ref2["iterations"] else w2, 1e-9)


# ------------------------------------------------------------- full size, bench launch config
def _csr_cfg(name):
    cfg = rsinputs.CONFIGS[name]
    if cfg.zipf_a > 0:
        rp, ci, va, y = rsinputs.csr_zipf(cfg.n, cfg.d, cfg.nnz_per_row, a=cfg.zipf_a, seed=0)
    else:
        rp, ci, va, y = rsinputs.csr_uniform(cfg.n, cfg.d, cfg.nnz_per_row, seed=0)
    return cfg, rp, ci, va, y


@pytest.mark.parametrize("name,iters", [("c3", 1), ("c4", 3)])
def test_csr_configs_full_size(rs, name, iters):
    """BASELINE.json c3 / c4 at full size in bench.py's default mode (GRAM, sketch-ahead pipeline,
    check_every = 50): the first iterations equal the oracle's (c3: 5e5 x 5e4 count tau = 500;
    c4: 2e4 x 1e6 Zipf dual, SubCount tau = 256, k = 4)."""
    cfg, rp, ci, va, y = _csr_cfg(name)
    h = rs.rs_create_csr(cfg.n, cfg.d, rp, ci, va, y, cfg.lam, mode="gram")
    try:
        w, rep = rs.rs_solve(h, cfg.sketch, cfg.tau, cfg.gamma, cfg.beta, 0.0, iters, seed=0,
                             subcount_k=cfg.subcount_k, check_every=50, d=cfg.d)
        it, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    Xs = rsinputs.csr_to_scipy(rp, ci, va, cfg.n, cfg.d)
    ref = OV.solve(Xs, y, cfg.lam, cfg.sketch, cfg.tau, cfg.gamma, cfg.beta, 0.0, iters, seed=0,
                   subcount_k=cfg.subcount_k)
    assert rep["iterations"] == iters
    assert_close(it, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


def test_config5_full_size_invariants(rs):
    """BASELINE.json c5 (2e6 x 4096 fp64, 65.5 GB on the device) in EXPLICIT mode (bench's c5
    line): the sketches are the oracle's bit for bit, beta = 0 steps satisfy the projection
    constraint S_k^T r^{k+1} = 0, and the maintained residual equals A w - b at sampled
    coordinates, with A w - b recomputed on the host in fp64 from X streamed back in row chunks."""
    from oracle import sketch as OS
    cfg = rsinputs.CONFIGS["c5"]
    free, _ = torch.cuda.mem_get_info()
    if free < 80e9:
        pytest.skip("needs ~80 GB of free device memory")
    Xd, yd = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, col_decay=True, noise=cfg.noise,
                                    device="cuda")
    h = rs.rs_create_dense(Xd, yd, cfg.lam, mode="explicit", borrow=True)
    try:
        w, rep = rs.rs_solve(h, "subsample", cfg.tau, 1.0, 0.0, 0.0, 3, seed=0, check_every=3)
        _, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    assert rep["iterations"] == 3
    for k in range(3):
        c, b, s = rs.rs_sketch_draw("subsample", cfg.d, cfg.tau, 0, k)
        ref = OS.draw("subsample", cfg.d, cfg.tau, k, 0)
        assert np.array_equal(c, ref["coord"]) and np.array_equal(b, ref["bucket"])
    c2 = rs.rs_sketch_draw("subsample", cfg.d, cfg.tau, 0, 2)[0]
    bn = None
    rng = np.random.default_rng(5)
    J = np.unique(np.concatenate([rng.choice(cfg.d, 64, replace=False), c2[:16]]))
    # host fp64: t = X w, u_J = X[:, J]^T t, b_J = X[:, J]^T y, chunk by chunk, with the
    # magnitudes |X|^T (|X| |w|) + |X|^T |y| that bound the rounding of either side
    u = np.zeros(J.size)
    bJ = np.zeros(J.size)
    mag = np.zeros(J.size)
    bfull = np.zeros(cfg.d)
    for i0 in range(0, cfg.n, 100_000):
        Xc = Xd[i0:i0 + 100_000].cpu().numpy()
        yc = yd[i0:i0 + 100_000].cpu().numpy()
        XJ = Xc[:, J]
        t = Xc @ w
        u += XJ.T @ t
        bJ += XJ.T @ yc
        mag += np.abs(XJ).T @ (np.abs(Xc) @ np.abs(w) + np.abs(yc))
        bfull += Xc.T @ yc
    del Xd, yd
    torch.cuda.empty_cache()
    bn = np.linalg.norm(bfull)
    resid = u + cfg.lam * w[J] - bJ
    err = np.abs(r[J] - resid)
    # rounding of sums of ~n d terms on both sides: a few hundred ulps of the magnitudes
    assert np.all(err <= 1e-12 * (mag + cfg.lam * np.abs(w[J]))), \
        (err.max(), (err / (mag + 1e-300)).max(), bn)
    assert np.max(np.abs(r[c2])) <= 1e-10 * bn, (np.max(np.abs(r[c2])), bn)   # S_2^T r^3 = 0


# ------------------------------------------------------------------ momentum schedules (NEXT-1)
@pytest.mark.parametrize("momentum,eta", [("heuristic", 0.995), ("theory", 0.995), ("cor1", 0.5),
                                          ("cor1", 0.9)])
@pytest.mark.parametrize("mode", ["implicit", "explicit", "gram"])
def test_momentum_schedules_dense(rs, momentum, eta, mode):
    """Iteration-dependent (gamma_k, beta_k) of the paper's schedules (rs_momentum) equal the
    oracle's (oracle/momentum.py) over 260 iterations -- past THEORY's switch (~k = 200)."""
    X, y = rsinputs.dense_problem(600, 40, seed=12)
    X, y = X.numpy(), y.numpy()
    h = rs.rs_create_dense(X, y, 0.2, mode=mode)
    try:
        w, rep = rs.rs_solve(h, "subsample", 6, 1.0, 0.0, 0.0, 260, seed=3, check_every=37,
                             momentum=momentum, eta=eta)
        _, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(X, y, 0.2, "subsample", 6, tol=0.0, max_iter=260, seed=3, momentum=momentum,
                   eta=eta)
    assert rep["iterations"] == 260
    assert_close(w, ref["w"], 1e-9)
    assert_close(r, ref["r"], 1e-9)


@pytest.mark.parametrize("momentum", ["heuristic", "theory"])
def test_momentum_schedules_csr(rs, momentum):
    n, d = 3000, 300
    rp, ci, v, y, Xs = _csr_primal(n, d, per_row=20, seed=4)
    h = rs.rs_create_csr(n, d, rp, ci, v, y, 1e-2, mode="gram")
    try:
        w, rep = rs.rs_solve(h, "count", 30, 1.0, 0.0, 0.0, 220, seed=5, momentum=momentum)
        _, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(Xs, y, 1e-2, "count", 30, tol=0.0, max_iter=220, seed=5, momentum=momentum)
    assert_close(w, ref["w"], 1e-9)
    assert_close(r, ref["r"], 1e-9)


def test_momentum_invalid(rs):
    X, y = _dense(50, 5)
    h = rs.rs_create_dense(X, y, 1.0)
    try:
        with pytest.raises(rs.RSError):
            rs.rs_solve(h, "subsample", 2, max_iter=3, momentum="cor1", eta=1.0)
        with pytest.raises(rs.RSError):
            rs.rs_solve(h, "subsample", 2, max_iter=3, momentum="theory", eta=0.0)
    finally:
        rs.rs_destroy(h)


# ------------------------------------------------------------------ kernel ridge route (NEXT-4)
@pytest.mark.parametrize("kind,tau,k,beta,lam,sigma", [
    ("subsample", 20, 0, 0.5, 0.5, 0.5), ("count", 17, 0, 0.5, 0.5, 0.5),
    ("subcount", 12, 3, 0.0, 0.5, 0.5), ("subsample", 240, 0, 0.5, 0.5, 0.5),
    ("subsample", 240, 0, 0.5, 0.2, 1.7)])
def test_kernel_ridge_parity(rs, kind, tau, k, beta, lam, sigma):
    """rs_create_kernel builds K (Eq. Gausskernel), A = K (K + lambda I), b = K y on the device;
    the EXPLICIT iterations then equal the oracle's (oracle/problem.build_kernel) within 1e-10.
    The last case is ill-conditioned (kappa(G_0) ~ 1e10 at lambda = 0.2, sigma = 1.7): there both the
    GPU's and the fp64 oracle's iterates are compared with an extended-precision run of Alg. 2
    (oracle.solver.solve_system_ld, eps = 2^-63) under the forward-error bound kappa(G_0) eps k of
    k = 30 sketched solves (R28; SURVEY c.5) -- the bound the fp64 oracle itself meets."""
    rng = np.random.default_rng(7)
    n, d = 301, 5
    X = rng.standard_normal((n, d))
    y = np.sin(X @ rng.standard_normal(d)) + 0.05 * rng.standard_normal(n)
    h = rs.rs_create_kernel(X, y, lam, sigma)
    try:
        a, rep = rs.rs_solve(h, kind, tau, 1.0, beta, 0.0, 30, seed=4, subcount_k=k)
        _, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve_kernel(X, y, lam, sigma, kind, tau, 1.0, beta, 0.0, 30, seed=4, subcount_k=k)
    assert rep["iterations"] == 30
    sysk = OP.build_kernel(X, y, lam, sigma)
    S0 = OS.materialize(OS.draw(kind, n, tau, 0, 4, k)).toarray()
    kappa = np.linalg.cond(S0.T @ sysk["A"] @ S0)
    if kappa < 1e4:
        assert_close(a, ref["w"], 1e-10)
        assert_close(r, ref["r"], 1e-10)
        return
    ld = OV.solve_system_ld(sysk["A"], sysk["b"], kind, tau, 1.0, beta, 30, seed=4, subcount_k=k)
    w_ld = np.asarray(ld["w"], dtype=np.float64)
    r_ld = np.asarray(ld["r"], dtype=np.float64)
    bound = kappa * np.finfo(float).eps * 30
    assert rel(ref["w"], w_ld) <= bound and rel(ref["r"], r_ld) <= bound   # the bound holds for fp64
    assert rel(a, w_ld) <= bound, (rel(a, w_ld), bound)
    assert rel(r, r_ld) <= bound, (rel(r, r_ld), bound)


@pytest.mark.parametrize("kind,tau", [("subsample", 600), ("count", 700), ("subsample", 1032)])
def test_kernel_ridge_blocked_inverse(rs, kind, tau):
    """Kernel ridge (NEXT-4) at tau >= 512 runs the group kernel on the blocked inverse (two
    diagonal super-blocks of W_bb = L_bb^{-1}, L below them; bfactor.cu / iterate.cu): tau = 600
    and 700 leave a ragged second block (320 + 280, 384 + 316), 1032 is k1's tau (576 + 456).
    Iterates equal the oracle's within 1e-10 (well-conditioned: kappa(G_0) < 1e4 asserted)."""
    rng = np.random.default_rng(9)
    n, d, lam, sigma = 1400, 5, 0.5, 0.3
    X = rng.standard_normal((n, d))
    y = np.sin(X @ rng.standard_normal(d)) + 0.05 * rng.standard_normal(n)
    h = rs.rs_create_kernel(X, y, lam, sigma)
    try:
        a, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 30, seed=4)
        _, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve_kernel(X, y, lam, sigma, kind, tau, 1.0, 0.5, 0.0, 30, seed=4)
    sysk = OP.build_kernel(X, y, lam, sigma)
    S0 = OS.materialize(OS.draw(kind, n, tau, 0, 4, 0)).toarray()
    S0 = S0[:, np.abs(S0).sum(axis=0) > 0]   # (count: empty buckets are the identity, R3)
    assert np.linalg.cond(S0.T @ sysk["A"] @ S0) < 1e4
    assert rep["iterations"] == 30
    assert_close(a, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


def test_kernel_ridge_converges_and_predicts(rs):
    rng = np.random.default_rng(8)
    n, d = 200, 3
    X = rng.standard_normal((n, d))
    y = np.cos(X[:, 0]) + 0.5 * X[:, 1]
    lam, sigma = 1.0, 0.4          # kappa(A) = 1.6e4
    h = rs.rs_create_kernel(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), lam, sigma)
    try:
        a, rep = rs.rs_solve(h, "subsample", 40, 1.0, 0.0, 1e-11, 100000, seed=1)
    finally:
        rs.rs_destroy(h)
    s = OP.build_kernel(X, y, lam, sigma)
    a_star = OP.direct_solve(s["A"], s["b"])
    assert rep["converged"]
    assert_close(a, a_star, 1e-6)
    assert_close(s["K"] @ a, s["K"] @ a_star, 1e-7)   # predictions on the inputs


def test_kernel_invalid(rs):
    X = np.zeros((4, 2))
    with pytest.raises(rs.RSError):
        rs.rs_create_kernel(X, np.zeros(4), 1.0, 0.0)
    with pytest.raises(rs.RSError):
        rs.rs_create_kernel(X, np.zeros(4), -1.0, 1.0)


@pytest.mark.parametrize("mode,kind,tau", [("explicit", "subsample", 300), ("explicit", "subsample", 120),
                                           ("explicit", "count", 260), ("gram", "subsample", 300),
                                           ("implicit", "subsample", 300)])
def test_dirty_device_memory(rs, mode, kind, tau):
    """Every device buffer is written before it is read: the same solve after the allocator's pages
    were filled with NaN (freed by torch and handed back to the driver) equals the oracle."""
    free, _ = torch.cuda.mem_get_info()
    junk = torch.full((int(min(free * 0.8, 60e9)) // 8,), float("nan"), dtype=torch.float64,
                      device="cuda")
    del junk
    torch.cuda.empty_cache()
    n, d = 2500, 900
    X, y = rsinputs.dense_problem(n, d, seed=21)
    X, y = X.numpy(), y.numpy()
    w, r, rep = _run_gpu_dense(rs, X, y, 0.7, mode, kind, tau, 0.5, 9, seed=2)
    ref = OV.solve(X, y, 0.7, kind, tau, 1.0, 0.5, 0.0, 9, seed=2)
    assert_close(w, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


# -------------------------------------------------------------- sparse explicit A (NEXT-3)
@pytest.mark.parametrize("kind,tau,k", [("count", 40, 0), ("subsample", 33, 0), ("subcount", 20, 3),
                                        ("count", 300, 0)])
def test_csr_explicit_primal(rs, kind, tau, k):
    n, d = 4000, 600
    rp, ci, v, y, Xs = _csr_primal(n, d, per_row=90, seed=9)   # rows > 64 nnz: heavy-row DMMA block
    h = rs.rs_create_csr(n, d, rp, ci, v, y, 1e-2, mode="explicit")
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 15, seed=2, subcount_k=k)
        ws, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(Xs, y, 1e-2, kind, tau, 1.0, 0.5, 0.0, 15, seed=2, subcount_k=k, explicit=True)
    assert_close(w, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


@pytest.mark.parametrize("kind,tau,k", [("subcount", 16, 4), ("subsample", 25, 0), ("count", 12, 0),
                                        ("subcount", 240, 1)])
def test_csr_explicit_dual(rs, kind, tau, k):
    n, d = 300, 5000
    rp, ci, v, y = rsinputs.csr_zipf(n, d, 60, a=1.1, seed=3)   # Zipf head: columns > 64 nnz
    Xs = rsinputs.csr_to_scipy(rp, ci, v, n, d)
    h = rs.rs_create_csr(n, d, rp, ci, v, y, 1e-1, mode="explicit")
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 15, seed=4, subcount_k=k, d=d, alpha=True)
        alpha, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(Xs, y, 1e-1, kind, tau, 1.0, 0.5, 0.0, 15, seed=4, subcount_k=k, explicit=True)
    assert_close(alpha, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)
    assert_close(w, ref["weights"], 1e-10)


def test_csr_explicit_config4_full_size(rs):
    """BASELINE.json c4 (2e4 x 1e6, Zipf) with the sparse explicit A (NEXT-3): 3 iterations equal
    the oracle's (implicit oracle: A S = X (X^T S) + lambda S, the same iterates in exact
    arithmetic)."""
    cfg, rp, ci, va, y = _csr_cfg("c4")
    h = rs.rs_create_csr(cfg.n, cfg.d, rp, ci, va, y, cfg.lam, mode="explicit")
    try:
        w, rep = rs.rs_solve(h, cfg.sketch, cfg.tau, cfg.gamma, cfg.beta, 0.0, 3, seed=0,
                             subcount_k=cfg.subcount_k, check_every=50, d=cfg.d)
        it, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    Xs = rsinputs.csr_to_scipy(rp, ci, va, cfg.n, cfg.d)
    ref = OV.solve(Xs, y, cfg.lam, cfg.sketch, cfg.tau, cfg.gamma, cfg.beta, 0.0, 3, seed=0,
                   subcount_k=cfg.subcount_k)
    assert_close(it, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


# ------------------------------------------------- process-level switches (read once per process)
_SWITCH_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import rsinputs
from paper_2105_05565_b200 import ridgesketch as rs
X, y = rsinputs.dense_problem(3001, 600, seed=4)
X, y = X.numpy(), y.numpy()
out = {}
for mode, kind, tau, k in [("explicit", "subsample", 300, 0), ("explicit", "subcount", 250, 2),
                           ("gram", "subsample", 150, 0)]:
    h = rs.rs_create_dense(X, y, 0.5, mode=mode)
    w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 12, 3, k, check_every=5)
    _, r = rs.rs_get_state(h)
    rs.rs_destroy(h)
    out[f"{mode}_{kind}_w"], out[f"{mode}_{kind}_r"] = w, r
np.savez(sys.argv[2], **out)
"""


@pytest.mark.parametrize("env", [{"RS_PDL": "0"}, {}])
def test_process_switches_parity(tmp_path, env):
    """The PDL chain off (RS_PDL=0) is read once per process: run it in a child and compare with the
    oracle (tau 300 / 250 > 224
    use the W = L^{-1} slots; 12 iterations span three check_every chunks)."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outp = tmp_path / "out.npz"
    e = dict(os.environ, **env)
    res = subprocess.run([sys.executable, "-c", _SWITCH_CHILD, root, str(outp)], env=e,
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    got = np.load(outp)
    X, y = rsinputs.dense_problem(3001, 600, seed=4)
    X, y = X.numpy(), y.numpy()
    for mode, kind, tau, k in [("explicit", "subsample", 300, 0), ("explicit", "subcount", 250, 2),
                               ("gram", "subsample", 150, 0)]:
        ref = OV.solve(X, y, 0.5, kind, tau, 1.0, 0.5, 0.0, 12, seed=3, subcount_k=k)
        assert_close(got[f"{mode}_{kind}_w"], ref["w"], 1e-10, f"{env} {mode} {kind} w")
        assert_close(got[f"{mode}_{kind}_r"], ref["r"], 1e-10, f"{env} {mode} {kind} r")


@pytest.mark.parametrize("kind,tau,k", [("subcount", 16, 4), ("subsample", 25, 0), ("subcount", 240, 1)])
def test_csr_dual_selected_rows_match_full_scan(rs, monkeypatch, kind, tau, k):
    """The dual selected-row path (k_sel_emit / k_sel_merge / k_sel_heavy) merges every touched row
    of R = X^T in the same order as the full-scan k_hash_rows, so the rows of R S are identical;
    the iterates then agree to rounding (heavy rows enter the Gram through a DMMA GEMM on the
    selected-row path and through the band kernel on the full scan, and the u = X t scatter uses
    L2 fp64 atomics).  RS_NO_SELROWS=1 selects the full scan (read per workspace)."""
    n, d = 300, 5000
    rp, ci, v, y = rsinputs.csr_zipf(n, d, 60, a=1.1, seed=3)
    out = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("RS_NO_SELROWS", env)
        h = rs.rs_create_csr(n, d, rp, ci, v, y, 1e-1, mode="gram")
        try:
            w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 15, seed=4, subcount_k=k, d=d)
            _, r = rs.rs_get_state(h)
        finally:
            rs.rs_destroy(h)
        out.append((w, r))
    assert_close(out[0][0], out[1][0], 1e-13)
    assert_close(out[0][1], out[1][1], 1e-13)


@pytest.mark.parametrize("kind,tau,k", [("subsample", 40, 0), ("subcount", 30, 2), ("count", 25, 0),
                                        ("subsample", 240, 0)])
def test_dense_dual_explicit_parity(rs, kind, tau, k):
    """Dense X with n < d: the dual route in EXPLICIT mode, A = X X^T + lambda I built
    on the lower DMMA tiles of X^T; alpha and r after 15 steps and w = X^T alpha equal the
    oracle's (tau 240 > 224: the W = L^{-1} slots)."""
    X, y = rsinputs.dense_problem(300, 900, seed=4)
    X, y = X.numpy(), y.numpy()
    h = rs.rs_create_dense(X, y, 0.5, mode="explicit")
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 15, 3, k, check_every=7, d=900, alpha=True)
        alpha, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(X, y, 0.5, kind, tau, 1.0, 0.5, 0.0, 15, seed=3, subcount_k=k)
    assert ref["route"] == "dual"
    assert_close(alpha, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)
    assert_close(rep["alpha"], ref["w"], 1e-10)
    assert_close(w, ref["weights"], 1e-10)


@pytest.mark.parametrize("kind,tau,k", [("subsample", 40, 0), ("subcount", 30, 2), ("count", 25, 0),
                                        ("subsample", 240, 0)])
@pytest.mark.parametrize("mode", ["implicit", "gram"])
def test_dense_dual_r_parity(rs, kind, tau, k, mode):
    """Dense X with n < d in IMPLICIT / GRAM mode: the primal machinery on R = X^T (d x n), whose
    A = R^T R + lambda I = X X^T + lambda I: A S = R^T (R S) + lambda S, or the Gram of
    R S and u = R^T (R S delta); alpha, r and w = X^T alpha equal the oracle's."""
    X, y = rsinputs.dense_problem(300, 900, seed=4)
    X, y = X.numpy(), y.numpy()
    h = rs.rs_create_dense(X, y, 0.5, mode=mode)
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 15, 3, k, check_every=7, d=900, alpha=True)
        alpha, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(X, y, 0.5, kind, tau, 1.0, 0.5, 0.0, 15, seed=3, subcount_k=k)
    assert ref["route"] == "dual"
    assert_close(alpha, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)
    assert_close(w, ref["weights"], 1e-10)


# ------------------------------------------------------------------ failure paths
@pytest.mark.parametrize("mode", ["implicit", "explicit", "gram"])
def test_not_spd_sketched_system(rs, mode):
    """RS_ENOTSPD: two identical columns (entries 1, squared norm 4) and lambda = 1e-300 (lost against
    4 in fp64), S = I: G = [[4, 4], [4, 4]] is exactly singular -- L11 = 2, L21 = 2, pivot 4 - 4 = 0
    (every operation exact), so the Cholesky must report it (R3)."""
    X = np.zeros((64, 2))
    X[:4, :] = 1.0
    y = np.arange(64, dtype=np.float64)
    h = rs.rs_create_dense(X, y, 1e-300, mode=mode)
    try:
        with pytest.raises(rs.RSError) as ei:
            rs.rs_solve(h, "subsample", 2, 1.0, 0.0, 0.0, 5)
        assert ei.value.status == rs.RS_ENOTSPD, str(ei.value)
    finally:
        rs.rs_destroy(h)


@pytest.mark.parametrize("mode", ["implicit", "explicit", "gram"])
def test_diverged_residual(rs, mode):
    """RS_EDIVERGED: X = 1e150 N(0,1) and y ~ 1e10 keep A = X^T X + I (~1e302) finite, but
    ||b||^2 = ||X^T y||^2 (~1e325) and ||r||^2 leave the fp64 range, so the relative residual is not
    finite (include/ridgesketch.h)."""
    X, y = rsinputs.dense_problem(300, 20, seed=1)
    X = X.numpy() * 1e150
    h = rs.rs_create_dense(X, y.numpy() * 1e10, 1.0, mode=mode)
    try:
        with pytest.raises(rs.RSError) as ei:
            rs.rs_solve(h, "subsample", 5, 1.0, 0.5, 1e-4, 50)
        assert ei.value.status == rs.RS_EDIVERGED, str(ei.value)
    finally:
        rs.rs_destroy(h)


def test_explicit_streamed_host_build(rs):
    """rs_create_dense from host memory, EXPLICIT, X >= 2 GB: the rows are copied in chunks on a copy
    stream while A = sum_c X_c^T X_c accumulates on the solver stream (the c5 e2e path).  The
    iterates equal the oracle's (A = X^T X + lambda I) within 1e-10."""
    n, d = 262_144, 1024
    X, y = rsinputs.dense_problem(n, d, seed=21, col_decay=True, noise=0.01)
    X, y = X.numpy(), y.numpy()
    h = rs.rs_create_dense(X, y, 1e-4 * n, mode="explicit")
    try:
        w, rep = rs.rs_solve(h, "subsample", 200, 1.0, 0.5, 0.0, 6, seed=2)
        _, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(X, y, 1e-4 * n, "subsample", 200, 1.0, 0.5, 0.0, 6, seed=2, explicit=True)
    assert rep["iterations"] == 6
    assert_close(w, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)


@pytest.mark.parametrize("case", ["primal_count_col", "dual_subcount_row"])
def test_csr_gram_uneven_scales(rs, case):
    """CSR GRAM accumulates the Gram bands in int64 fixed point; the scale of each band entry comes
    from its two buckets (k_bucket_scale), so one column of R scaled by 1e6 -- one bucket's
    diagonal 1e12 times the others -- leaves the other buckets their full precision and the
    iterates equal the oracle's within 1e-10 (advisor finding on the former trace(G) scale).
    Primal: R = X, a column of X; dual: R = X^T, a sample (row of X).  (Scaling a feature of the
    dual instead adds a rank-one 1e12 term across buckets: G itself becomes ill-conditioned, which
    no accumulation precision can repair.)"""
    if case.startswith("primal"):
        n, d = 4000, 600
        rp, ci, v, y = rsinputs.csr_uniform(n, d, 12, seed=1)
        v = v.copy()
        v[ci == 7] *= 1e6
        kind, tau, k, lam = "count", 40, 0, 1e-2
    else:
        n, d = 300, 5000
        rp, ci, v, y = rsinputs.csr_zipf(n, d, 40, a=1.1, seed=6)
        v = v.copy()
        v[rp[3]:rp[4]] *= 1e6                            # one sample
        kind, tau, k, lam = "subcount", 16, 4, 1e-3
    Xs = rsinputs.csr_to_scipy(rp, ci, v, n, d)
    h = rs.rs_create_csr(n, d, rp, ci, v, y, lam, mode="gram")
    try:
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 12, seed=2, subcount_k=k, d=d)
        ws, r = rs.rs_get_state(h)
    finally:
        rs.rs_destroy(h)
    ref = OV.solve(Xs, y, lam, kind, tau, 1.0, 0.5, 0.0, 12, seed=2, subcount_k=k)
    assert rep["iterations"] == 12
    assert_close(ws, ref["w"], 1e-10)
    assert_close(r, ref["r"], 1e-10)
