"""Debug: per-phase clock64 totals of the single-CTA Cholesky (k_chol_small) on a c2-shaped solve."""
import ctypes as C, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import rsinputs
from paper_2105_05565_b200 import ridgesketch as rs
tau = int(sys.argv[1]) if len(sys.argv) > 1 else 200
X, y = rsinputs.dense_problem(20000, 2000, seed=0, col_decay=True, device="cuda")
h = rs.rs_create_dense(X, y, 2.0, mode="gram", borrow=True)
rs.rs_solve(h, "subsample", tau, 1.0, 0.5, 0.0, 5, 0)
buf = (C.c_ulonglong * 8)()
rs._lib.rs_internal_chol_times(buf)
w, rep = rs.rs_solve(h, "subsample", tau, 1.0, 0.5, 0.0, 50, 0, profile=True)
rs._lib.rs_internal_chol_times(buf)
n = buf[6]
names = ["gather", "diag", "panel", "trailing", "backward", "scatter"]
tot = sum(buf[k] for k in range(6))
print(f"tau={tau} calls={n} total cycles/call={tot/n:.0f} (~{tot/n/1.9e3:.1f} us at 1.9 GHz); solve class ms/launch="
      f"{rep['kernel_ms']['solve']/max(rep['kernel_launches']['solve'],1):.4f}")
for k, nm in enumerate(names):
    print(f"  {nm:9s} {buf[k]/n:10.0f} cycles  {buf[k]/tot:6.1%}")
rs.rs_destroy(h)
