"""Times rs_solve host/device overhead for a config: max_iter = 0, 1, K (wall clock + events)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import rsinputs
from paper_2105_05565_b200 import ridgesketch as rs

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c4"
mode = sys.argv[2] if len(sys.argv) > 2 else "gram"
cfg = rsinputs.CONFIGS[cfgname]
if cfg.zipf_a > 0:
    rp, ci, va, yv = rsinputs.csr_zipf(cfg.n, cfg.d, cfg.nnz_per_row, a=cfg.zipf_a, seed=0)
else:
    rp, ci, va, yv = rsinputs.csr_uniform(cfg.n, cfg.d, cfg.nnz_per_row, seed=0)
h = rs.rs_create_csr(cfg.n, cfg.d, rp, ci, va, yv, cfg.lam, mode=mode)
common = dict(kind=cfg.sketch, tau=cfg.tau, gamma=cfg.gamma, beta=cfg.beta, seed=0,
              subcount_k=cfg.subcount_k, d=cfg.d)
for it in (0, 1, 20, 20, 64, 64):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rep = rs.rs_solve(h, tol=0.0, max_iter=it, check_every=20, **common)
    torch.cuda.synchronize()
    print(f"max_iter {it}: wall {1e3*(time.perf_counter()-t0):.2f} ms, solve_seconds {rep['solve_seconds']*1e3:.2f} ms", flush=True)
rs.rs_destroy(h)
