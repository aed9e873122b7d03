"""Development probe: per-phase SM cycles of the large-tau factorisation (k_bfactor_lp), from a
library built with RS_NVCC_EXTRA=-DRS_BF_PHASES.  usage: python tools/probe_bf_phases.py [cfg] [iters] [slots factored per solve (default min(iters, 148))]"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import rsinputs
from paper_2105_05565_b200 import ridgesketch as rs

cfg = rsinputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 148
lib = rs._lib
lib.rs_debug_bf_phases.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 8)()
if cfg.kind == "kernel":
    Xk, yk = rsinputs.kernel_problem(cfg.n, cfg.d, seed=0, noise=cfg.noise)
    h = rs.rs_create_kernel(Xk, yk, cfg.lam, cfg.extra["sigma"])
    d = cfg.n
else:
    X, y = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, col_decay=cfg.col_decay, noise=cfg.noise, device="cuda")
    h = rs.rs_create_dense(X, y, cfg.lam, mode="explicit", borrow=True)
    d = cfg.d
for rep in range(2):
    lib.rs_debug_bf_phases(buf, 1)
    w, r = rs.rs_solve(h, cfg.sketch, cfg.tau, 1.0, cfg.beta, 0.0, iters, 0, cfg.subcount_k, check_every=iters, d=d)
    lib.rs_debug_bf_phases(buf, 0)
ph = np.array(list(buf), dtype=np.float64)
names = ["gather", "chol acc", "chol diag", "chol total", "inv acc", "inv total", "inv diag", "write"]
slots = int(sys.argv[3]) if len(sys.argv) > 3 else min(iters, 148)
print(f"{cfg.name}: solve {r['solve_seconds']*1e3:.3f} ms, factor ms/launch {r['kernel_ms']['factor'] if r['kernel_ms']['factor'] else 0}")
tot = ph[0] + ph[3] + ph[5] + ph[7]
for k, nm in enumerate(names):
    print(f"  {nm:11s} {ph[k] / slots / 1965e3:8.3f} ms/slot-CTA  ({ph[k] / tot:5.3f})")
print(f"  chol rest  {(ph[3]-ph[1]-ph[2]) / slots / 1965e3:8.3f}   inv rest {(ph[5]-ph[4]-ph[6]) / slots / 1965e3:8.3f}")
