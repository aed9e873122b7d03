"""Rank process of tests/test_gpu_multirank.py: one rank of a world that runs the library's
multi-rank path (rs_dist with world > 1) through the C ABI.  Not a test module.

usage: python multirank_worker.py RANK WORLD PORT COLLECTIVE OUTDIR CASE [CASE ...]
Each case writes OUTDIR/CASE.rankR.npz with the weights, the system iterate and the residual."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import torch  # noqa: E402
import torch.distributed as tdist  # noqa: E402

import rsinputs  # noqa: E402
from multirank_cases import CASES, csr_column_block  # noqa: E402


def main():
    rank, world, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    coll, outdir, cases = sys.argv[4], sys.argv[5], sys.argv[6:]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2105_05565_b200 import ridgesketch as rs
    device = rank % max(1, torch.cuda.device_count())
    torch.cuda.set_device(device)
    for name in cases:
        c = CASES[name]
        obj = [None]
        if rank == 0:
            obj = [rs.rs_host_coll_id() if coll == "host" else rs.rs_nccl_unique_id()]
        tdist.broadcast_object_list(obj, src=0)
        dist = dict(device=device, rank=rank, world=world, nccl_unique_id=obj[0], collective=coll)
        if c["data"] == "dense":
            X, y = rsinputs.dense_problem(c["n"], c["d"], seed=c["seed"], col_decay=True, noise=0.01)
            X, y = X.numpy(), y.numpy()
            if c.get("dual"):   # feature (column) shards; y whole
                b0, ln = rs.rs_shard_range(c["d"], rank, world)
                dist.update(shard_begin=b0, shard_len=ln)
                h = rs.rs_create_dense(np.ascontiguousarray(X[:, b0:b0 + ln]), y, c["lam"], route="dual",
                                       mode=c["mode"], n=c["n"], d=c["d"], dist=dist)
            else:
                b0, ln = rs.rs_shard_range(c["n"], rank, world)
                dist.update(shard_begin=b0, shard_len=ln)
                h = rs.rs_create_dense(np.ascontiguousarray(X[b0:b0 + ln]), np.ascontiguousarray(y[b0:b0 + ln]),
                                       c["lam"], mode=c["mode"], n=c["n"], d=c["d"], dist=dist)
        else:
            rp, ci, v, y = c["make"]()
            n, d = c["n"], c["d"]
            if d > n:   # dual: feature (column) shards, nnz-balanced through the CSC column pointer
                colptr = np.concatenate([[0], np.cumsum(np.bincount(ci, minlength=d))]).astype(np.int64)
                b0, ln = rs.rs_shard_rows_nnz(colptr, rank, world)
                rpl, cil, vl = csr_column_block(rp, ci, v, b0, ln)
                dist.update(shard_begin=b0, shard_len=ln)
                h = rs.rs_create_csr(n, d, rpl, cil, vl, y, c["lam"], mode=c["mode"], dist=dist)
            else:       # primal: nnz-balanced row shards
                b0, ln = rs.rs_shard_rows_nnz(rp, rank, world)
                e0, e1 = rp[b0], rp[b0 + ln]
                dist.update(shard_begin=b0, shard_len=ln)
                h = rs.rs_create_csr(n, d, rp[b0:b0 + ln + 1] - e0, ci[e0:e1], v[e0:e1], y[b0:b0 + ln],
                                     c["lam"], mode=c["mode"], dist=dist)
        try:
            w, rep = rs.rs_solve(h, c["kind"], c["tau"], 1.0, 0.5, 0.0, c["iters"], seed=c["sseed"],
                                 subcount_k=c.get("k", 0), check_every=c.get("check_every", 0), d=c["d"])
            ws, r = rs.rs_get_state(h)
        finally:
            rs.rs_destroy(h)
        np.savez(os.path.join(outdir, f"{name}.rank{rank}.npz"), w=w, ws=ws, r=r,
                 iterations=rep["iterations"])
        tdist.barrier()
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
