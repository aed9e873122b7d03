"""Development probe: per-iteration completion times of the EXPLICIT group kernel (globaltimer), from
a library built with RS_NVCC_EXTRA=-DRS_IT_TIMES: where a solve's iterations wait for factor slots.
usage: python tools/probe_it_times.py [cfg] [iters]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import rsinputs
from paper_2105_05565_b200 import ridgesketch as rs

cfg = rsinputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 600
X, y = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, col_decay=cfg.col_decay, noise=cfg.noise, device="cuda")
h = rs.rs_create_dense(X, y, cfg.lam, mode="explicit", borrow=True)
for rep in range(3):
    w, r = rs.rs_solve(h, cfg.sketch, cfg.tau, 1.0, cfg.beta, 0.0, iters, rep, cfg.subcount_k,
                       trace_cap=iters, d=cfg.d)
    t = np.asarray(r["trace"], dtype=np.float64)
    dt = np.diff(t) / 1e3   # us
    solve_ms = r["solve_seconds"] * 1e3
    first = solve_ms - (t[-1] - t[0]) / 1e6   # ms from the solve's start event to iteration 1's end (approx.)
    print(f"seed {rep}: solve {solve_ms:.2f} ms, first iteration done at ~{first:.2f} ms, "
          f"median step {np.median(dt):.1f} us, p90 {np.percentile(dt, 90):.1f} us")
    big = np.argsort(dt)[-6:][::-1]
    print("   largest gaps (after iteration k: us):", [(int(k) + 1, round(float(dt[k]), 1)) for k in big])
    for lo, hi in [(0, 150), (150, 232), (232, 464), (464, iters - 1)]:
        if hi > lo and hi <= len(dt):
            print(f"   iterations {lo + 1}..{hi}: mean step {dt[lo:hi].mean():.1f} us")
