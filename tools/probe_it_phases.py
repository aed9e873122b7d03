"""Development probe: per-phase SM cycles (CTA 0) of the EXPLICIT group kernel k_iterate, from a
library built with RS_NVCC_EXTRA=-DRS_IT_PHASES.  usage: python tools/probe_it_phases.py [cfg] [iters]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import rsinputs
from paper_2105_05565_b200 import ridgesketch as rs

cfg = rsinputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 148
lib = rs._lib
lib.rs_debug_it_phases.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 12)()
X, y = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, col_decay=cfg.col_decay, noise=cfg.noise, device="cuda")
h = rs.rs_create_dense(X, y, cfg.lam, mode="explicit", borrow=True)
for rep in range(2):
    lib.rs_debug_it_phases(buf, 1)
    w, r = rs.rs_solve(h, cfg.sketch, cfg.tau, 1.0, cfg.beta, 0.0, iters, 0, cfg.subcount_k, check_every=iters, d=cfg.d)
    lib.rs_debug_it_phases(buf, 0)
ph = np.array(list(buf), dtype=np.float64)
names = ["A", "sync1", "B", "sync2", "C", "stage next", "sync3", "stop", "A: g", "A: prefetch", "A: rows"]
print(f"{cfg.name}: solve {r['solve_seconds']*1e3:.3f} ms for {iters} iterations")
for k, nm in enumerate(names):
    print(f"  {nm:11s} {ph[k] / iters / 1965:8.3f} us/iteration")
