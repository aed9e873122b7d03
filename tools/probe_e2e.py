"""Phase timing (wall clock) of the bench e2e path for a dense config: pinned host X -> create ->
solve to tol -> destroy.  usage: python tools/probe_e2e.py [c2] [explicit|gram|implicit]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, rsinputs
from paper_2105_05565_b200 import ridgesketch as rs
cfg = rsinputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
mode = sys.argv[2] if len(sys.argv) > 2 else "explicit"
X, y = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, col_decay=cfg.col_decay, noise=cfg.noise, device="cuda")
Xh, yh = X.cpu().pin_memory(), y.cpu().pin_memory()
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = rs.rs_create_dense(Xh, yh, cfg.lam, mode=mode)
    t1 = time.perf_counter()
    w, rep = rs.rs_solve(h, "subsample", cfg.tau, cfg.gamma, cfg.beta, cfg.tol, 20000, seed=0)
    t2 = time.perf_counter()
    rs.rs_destroy(h)
    t3 = time.perf_counter()
    print(f"run {i}: create {1e3*(t1-t0):.1f} ms (device setup {1e3*rep['setup_seconds']:.1f}), "
          f"solve {1e3*(t2-t1):.1f} ms (device {1e3*rep['solve_seconds']:.1f}, {rep['iterations']} its), "
          f"destroy {1e3*(t3-t2):.1f} ms", flush=True)
