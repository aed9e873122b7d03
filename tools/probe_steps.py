"""Probe: rs_solve wall/device time for fixed-step runs vs time-to-tolerance on one config.
usage: python tools/probe_steps.py CONFIG MODE"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import rsinputs
from paper_2105_05565_b200 import build
build()
from paper_2105_05565_b200 import ridgesketch as rs

cfg = rsinputs.CONFIGS[sys.argv[1]]
mode = sys.argv[2]
if cfg.kind == "dense":
    X, y = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, col_decay=cfg.col_decay, noise=cfg.noise, device="cuda")
    h = rs.rs_create_dense(X, y, cfg.lam, mode=mode, borrow=True)
else:
    gen = rsinputs.csr_zipf if cfg.zipf_a > 0 else rsinputs.csr_uniform
    kw = dict(a=cfg.zipf_a) if cfg.zipf_a > 0 else {}
    rp, ci, va, yv = gen(cfg.n, cfg.d, cfg.nnz_per_row, seed=0, **kw)
    h = rs.rs_create_csr(cfg.n, cfg.d, rp, ci, va, yv, cfg.lam, mode=mode)
common = dict(kind=cfg.sketch, tau=cfg.tau, gamma=cfg.gamma, beta=cfg.beta, seed=0, subcount_k=cfg.subcount_k, d=cfg.d)
for steps, ce in [(5, 148), (148, 148), (148, 148), (296, 148), (148, 0), (148, 0), (1000, 0)]:
    torch.cuda.synchronize(); t = time.perf_counter()
    _, rep = rs.rs_solve(h, tol=0.0, max_iter=steps, check_every=ce, **common)
    torch.cuda.synchronize(); t = time.perf_counter() - t
    print(f"steps {steps:5d} check_every {ce:4d}: its {rep['iterations']} solve {rep['solve_seconds']*1e3:8.3f} ms "
          f"({rep['solve_seconds']*1e3/max(rep['iterations'],1):.4f} ms/it) wall {t*1e3:8.3f} ms launches {rep.get('gpu_launches')}", flush=True)
for _ in range(2):
    _, rep = rs.rs_solve(h, tol=cfg.tol, max_iter=20000, check_every=0, **common)
    print(f"tol: its {rep['iterations']} solve {rep['solve_seconds']*1e3:.3f} ms ({rep['solve_seconds']*1e3/rep['iterations']:.4f} ms/it)", flush=True)
rs.rs_destroy(h)
