"""Small solves of every path for compute-sanitizer (memcheck / racecheck / synccheck):
c1-shaped dense in IMPLICIT / EXPLICIT / GRAM, a tau > 224 EXPLICIT solve (overlapped pipeline:
k_bf_gather, k_bfactor_lp, k_iterate), CSR primal and dual in IMPLICIT and GRAM.
usage: compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import rsinputs  # noqa: E402
from paper_2105_05565_b200 import ridgesketch as rs  # noqa: E402

X, y = rsinputs.dense_problem(1000, 50, seed=0, noise=0.1)
X, y = X.numpy(), y.numpy()
for mode in ("implicit", "explicit", "gram"):
    for kind, tau, k in (("subsample", 10, 0), ("count", 10, 0), ("subcount", 8, 3)):
        h = rs.rs_create_dense(X, y, 1e-2, mode=mode)
        w, rep = rs.rs_solve(h, kind, tau, 1.0, 0.5, 0.0, 20, 0, k, check_every=7)
        rs.rs_destroy(h)
        print(mode, kind, rep["iterations"], flush=True)
Xb, yb = rsinputs.dense_problem(2000, 300, seed=1, col_decay=True)
h = rs.rs_create_dense(Xb.numpy(), yb.numpy(), 0.5, mode="explicit")
w, rep = rs.rs_solve(h, "subsample", 260, 1.0, 0.5, 0.0, 12, 3)
rs.rs_destroy(h)
print("explicit tau 260", rep["iterations"], flush=True)
rp, ci, v, yc = rsinputs.csr_uniform(2000, 300, 10, seed=2)
for mode in ("implicit", "gram"):
    h = rs.rs_create_csr(2000, 300, rp, ci, v, yc, 1e-2, mode=mode)
    w, rep = rs.rs_solve(h, "count", 20, 1.0, 0.5, 0.0, 10, 1)
    rs.rs_destroy(h)
    print("csr primal", mode, rep["iterations"], flush=True)
rp, ci, v, yc = rsinputs.csr_zipf(200, 3000, 30, a=1.1, seed=3)
for mode in ("implicit", "gram"):
    h = rs.rs_create_csr(200, 3000, rp, ci, v, yc, 1e-3, mode=mode)
    w, rep = rs.rs_solve(h, "subcount", 12, 1.0, 0.5, 0.0, 10, 1, 3, d=3000)
    rs.rs_destroy(h)
    print("csr dual", mode, rep["iterations"], flush=True)
print("sanitize run done")
