"""Profiling driver: build one BASELINE.json config on cuda:0 and run exactly `iters` iterations
(tol = 0, one graph launch), so every kernel launch under ncu is an active one.
usage: python tools/prof_step.py [config] [mode] [iters]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import rsinputs
from paper_2105_05565_b200 import build
build()
from paper_2105_05565_b200 import ridgesketch as rs

cfg = rsinputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
mode = sys.argv[2] if len(sys.argv) > 2 else "gram"
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 8
if cfg.kind == "kernel":
    Xk, yk = rsinputs.kernel_problem(cfg.n, cfg.d, seed=0, noise=cfg.noise)
    h = rs.rs_create_kernel(Xk, yk, cfg.lam, cfg.extra["sigma"])
elif cfg.kind == "dense":
    X, y = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, col_decay=cfg.col_decay, noise=cfg.noise,
                                  device="cuda")
    h = rs.rs_create_dense(X, y, cfg.lam, mode=mode, borrow=True)
else:
    gen = rsinputs.csr_zipf if cfg.zipf_a > 0 else rsinputs.csr_uniform
    kw = dict(a=cfg.zipf_a) if cfg.zipf_a > 0 else {}
    rp, ci, va, yv = gen(cfg.n, cfg.d, cfg.nnz_per_row, seed=0, **kw)
    h = rs.rs_create_csr(cfg.n, cfg.d, rp, ci, va, yv, cfg.lam, mode=mode)
w, rep = rs.rs_solve(h, cfg.sketch, cfg.tau, cfg.gamma, cfg.beta, 0.0, iters, 0, cfg.subcount_k,
                     check_every=iters, d=cfg.n if cfg.kind == "kernel" else cfg.d)
torch.cuda.synchronize()
print(f"{cfg.name} {mode}: {rep['iterations']} iterations in {rep['solve_seconds'] * 1e3:.3f} ms "
      f"({rep['solve_seconds'] * 1e3 / max(rep['iterations'], 1):.4f} ms/iter), rel res "
      f"{rep['rel_residual']:.3e}")
rs.rs_destroy(h)
