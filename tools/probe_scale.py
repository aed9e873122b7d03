import sys, numpy as np
sys.path.insert(0, '.')
import rsinputs
from paper_2105_05565_b200 import build
build()
from paper_2105_05565_b200 import ridgesketch as rs
scale = 1e100
lam = 1e-2 * scale * scale
rp, ci, v, y = rsinputs.csr_uniform(3000, 400, 70, seed=12)
for mode in ["gram", "implicit"]:
    h = rs.rs_create_csr(3000, 400, rp, ci, v * scale, y * scale, lam, mode=mode)
    try:
        w, rep = rs.rs_solve(h, "count", 64, 1.0, 0.5, 0.0, 12, seed=5); print("primal", mode, "ok", rep["rel_residual"])
    except Exception as e: print("primal", mode, e)
    rs.rs_destroy(h)
rp, ci, v, y = rsinputs.csr_zipf(300, 5000, 60, a=1.1, seed=3)
for mode in ["gram", "implicit"]:
    h = rs.rs_create_csr(300, 5000, rp, ci, v * scale, y * scale, lam, mode=mode)
    try:
        w, rep = rs.rs_solve(h, "subcount", 16, 1.0, 0.5, 0.0, 12, seed=6, subcount_k=4, d=5000); print("dual", mode, "ok", rep["rel_residual"])
    except Exception as e: print("dual", mode, e)
    rs.rs_destroy(h)
