"""Probe: repeated fixed-step solves on one config, per-solve device time, to locate intermittent
timed-region stalls.  usage: python tools/probe_stall.py CONFIG MODE [reps] [steps] [chunk]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import rsinputs
from paper_2105_05565_b200 import build
build()
from paper_2105_05565_b200 import ridgesketch as rs

cfg = rsinputs.CONFIGS[sys.argv[1]]
mode = sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 12
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 1000
chunk = int(sys.argv[5]) if len(sys.argv) > 5 else 256
gen = rsinputs.csr_zipf if cfg.zipf_a > 0 else rsinputs.csr_uniform
kw = dict(a=cfg.zipf_a) if cfg.zipf_a > 0 else {}
rp, ci, va, yv = gen(cfg.n, cfg.d, cfg.nnz_per_row, seed=0, **kw)
h = rs.rs_create_csr(cfg.n, cfg.d, rp, ci, va, yv, cfg.lam, mode=mode)
common = dict(kind=cfg.sketch, tau=cfg.tau, gamma=cfg.gamma, beta=cfg.beta, seed=0,
              subcount_k=cfg.subcount_k, d=cfg.d)
rs.rs_solve(h, tol=0.0, max_iter=5, check_every=chunk, **common)
st = torch.cuda.current_stream()
for r in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); t = time.perf_counter()
    e0.record(st)
    _, rep = rs.rs_solve(h, tol=0.0, max_iter=steps, check_every=chunk, **common)
    e1.record(st)
    torch.cuda.synchronize(); t = time.perf_counter() - t
    print(f"rep {r:2d}: events {e0.elapsed_time(e1):9.3f} ms  library {rep['solve_seconds']*1e3:9.3f} ms  "
          f"wall {t*1e3:9.3f} ms  ({e0.elapsed_time(e1)/steps:.4f} ms/it)", flush=True)
rs.rs_destroy(h)
