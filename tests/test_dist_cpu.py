"""Multi-rank host logic on CPU (gloo, world size 2): the library's shard plan (rs_shard_range,
rs_shard_rows_nnz) covers the data exactly once, and the per-rank partial products the CUDA path
allreduces sum to the full ones:
  primal  A S = sum_p X_p^T (X_p S) + lambda S,   b = sum_p X_p^T y_p,   A = sum_p X_p^T X_p + lambda I
  dual    A S = sum_p X_p (X_p^T S) + lambda S,   w = sum_p pad_p(X_p^T alpha)
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import rsinputs
from oracle import sketch as OS


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_05565_b200 import ridgesketch as rs
        out = {}
        lam = 0.3
        # ---- dense primal, row shards
        X, y = rsinputs.dense_problem(97, 13, seed=1)
        X, y = X.numpy(), y.numpy()
        b0, ln = rs.rs_shard_range(97, rank, world)
        Xp, yp = X[b0:b0 + ln], y[b0:b0 + ln]
        sk = OS.draw("count", 13, 4, 2, 9)
        S = OS.materialize(sk).toarray()
        part = torch.from_numpy(Xp.T @ (Xp @ S))
        dist.all_reduce(part)
        out["primal_AS"] = np.abs(part.numpy() + lam * S - (X.T @ (X @ S) + lam * S)).max()
        bp = torch.from_numpy(Xp.T @ yp)
        dist.all_reduce(bp)
        out["primal_b"] = np.abs(bp.numpy() - X.T @ y).max()
        Ap = torch.from_numpy(Xp.T @ Xp)
        dist.all_reduce(Ap)
        out["primal_A"] = np.abs(Ap.numpy() + lam * np.eye(13) - (X.T @ X + lam * np.eye(13))).max()
        cnt = torch.tensor([ln])
        dist.all_reduce(cnt)
        out["rows_covered"] = int(cnt.item())
        # ---- CSR primal, nnz-balanced row shards
        rp, ci, v, yc = rsinputs.csr_uniform(200, 40, 6, seed=2)
        Xs = rsinputs.csr_to_scipy(rp, ci, v, 200, 40)
        c0, cl = rs.rs_shard_rows_nnz(rp, rank, world)
        Xsp = Xs[c0:c0 + cl]
        sk2 = OS.draw("subsample", 40, 7, 0, 3)
        S2 = OS.materialize(sk2).toarray()
        part2 = torch.from_numpy(np.asarray(Xsp.T @ (Xsp @ S2)))
        dist.all_reduce(part2)
        out["csr_AS"] = np.abs(part2.numpy() - np.asarray(Xs.T @ (Xs @ S2))).max()
        # ---- dual, column (feature) shards
        Xd, yd = rsinputs.dense_problem(11, 60, seed=3)
        Xd = Xd.numpy()
        f0, fl = rs.rs_shard_range(60, rank, world)
        Xdp = Xd[:, f0:f0 + fl]
        sk3 = OS.draw("subcount", 11, 3, 1, 5, 2)
        S3 = OS.materialize(sk3).toarray()
        part3 = torch.from_numpy(Xdp @ (Xdp.T @ S3))
        dist.all_reduce(part3)
        out["dual_AS"] = np.abs(part3.numpy() - Xd @ (Xd.T @ S3)).max()
        alpha = np.linspace(-1, 1, 11)
        wpad = np.zeros(60)
        wpad[f0:f0 + fl] = Xdp.T @ alpha
        wt = torch.from_numpy(wpad)
        dist.all_reduce(wt)
        out["dual_w"] = np.abs(wt.numpy() - Xd.T @ alpha).max()
        # ---- every rank regenerates the identical sketch stream from (seed, k)
        mine = torch.from_numpy(OS.draw("subsample", 1000, 50, 17, 4)["coord"])
        other = mine.clone()
        dist.broadcast(other, src=0)
        out["sketch_equal"] = bool(torch.equal(mine, other))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_partial_sums_match_full():
    from paper_2105_05565_b200 import build
    build()
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        o = res[r]
        assert o["rows_covered"] == 97
        for k in ("primal_AS", "primal_b", "primal_A", "csr_AS", "dual_AS", "dual_w"):
            assert o[k] <= 1e-10, (r, k, o[k])
        assert o["sketch_equal"]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_dual_feature_shards_balanced_by_nnz(world):
    """c4-shaped dual (Zipf(1.1) feature popularity): bench.py shards the features as contiguous
    ranges balanced by nnz (rs_shard_rows_nnz over the column pointer).  The ranges tile [0, d)
    exactly once, every rank's nnz is within one feature's nnz of the even share, and the largest
    shard is no larger than with plain d / world feature ranges."""
    from paper_2105_05565_b200 import build
    build()
    from paper_2105_05565_b200 import ridgesketch as rs
    n, d = 2000, 100_000
    rp, ci, va, y = rsinputs.csr_zipf(n, d, 25, a=1.1, seed=0)
    cnt = np.bincount(ci, minlength=d)
    colptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    total = int(colptr[-1])
    nxt, bal, plain = 0, [], []
    for r in range(world):
        b0, ln = rs.rs_shard_rows_nnz(colptr, r, world)
        assert b0 == nxt and ln >= 0
        nxt = b0 + ln
        bal.append(int(colptr[b0 + ln] - colptr[b0]))
        assert abs(bal[-1] - total / world) <= cnt.max() + 1, (r, bal[-1], total / world)
        p0, pl = rs.rs_shard_range(d, r, world)
        plain.append(int(colptr[p0 + pl] - colptr[p0]))
    assert nxt == d and sum(bal) == total
    assert max(bal) <= max(plain), (bal, plain)
