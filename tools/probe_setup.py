"""Wall / device time of rs_create_dense (explicit) for a config, twice."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, rsinputs
from paper_2105_05565_b200 import ridgesketch as rs
cfg = rsinputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
X, y = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, col_decay=cfg.col_decay, noise=cfg.noise, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    h = rs.rs_create_dense(X, y, cfg.lam, mode="explicit", borrow=True)
    torch.cuda.synchronize(); wall = time.perf_counter() - t
    _, rep = rs.rs_solve(h, "subsample", cfg.tau, 1.0, 0.5, 0.0, 1, seed=0)
    print(f"create {i}: wall {wall*1e3:.1f} ms, setup_seconds {rep['setup_seconds']*1e3:.1f} ms", flush=True)
    rs.rs_destroy(h)
