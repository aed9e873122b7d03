#!/usr/bin/env python
"""Benchmark of the momentum sketch-and-project hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]
                    [--mode implicit|explicit]

One "step" = one iteration of Alg. 2: sketch draw, rows of A S, S^T A S + Cholesky,
fused momentum update -- every row of SURVEY §8(a).  Workload at N=1: the largest single-GPU
BASELINE.json config, configs[4] (c5: dense primal 2e6 x 4096 fp64 = 65.5 GB, subsample
tau=1024, gamma=1, beta=0.5, lambda=1e-4 n, tol 1e-4) on the EXPLICIT route (A = X^T X + lambda I
built once by the lower-tile DMMA contraction, then per iteration the sketched rows of A), the
route with the shortest measured time to tolerance; the GRAM and IMPLICIT routes of the same data
are measured over a few iterations and reported as `alt_routes`.  Synthetic data generated on the
device from a fixed seed.

Prints ONE JSON line (rank 0).  `value` = iterations per second of the solve (device time, CUDA
events on the solver stream, max over ranks), `e2e` = the same metric through the public API from
pinned host buffers (H2D of X and y, setup, solve to tol, D2H of w inside the timed region),
`time_to_tol_s` = device seconds to ||r||/||b|| <= 1e-4 (median over sketch seeds 0..4, quartiles
in `time_to_tol_seeds`), `roofline` = the dominant kernel class against its measured peak,
`cpu_baseline` = the oracle on the host cores.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# AS route of each config's line: the one with the shortest measured time to tolerance (DESIGN.md
# §9); the dense configs' other routes are measured beside it (`alt_routes`).  c4 (CSR dual):
# EXPLICIT through the sparse A build (NEXT-3) -- 4.4x faster per iteration than the selected-row
# GRAM path in round 1 (14.2k vs 3.2k iters/s), and 0.67 + 0.3 s vs 3.05 s to 1e-4.
DEFAULT_MODE = {"c1": "gram", "c2": "gram", "c3": "gram", "c4": "explicit", "c5": "explicit",
                "k1": "explicit"}
METRIC = "sketch-and-project iters/s & s to ‖r‖/‖b‖≤1e-4; AS-pass HBM GB/s vs peak"
FP64_DMMA_PEAK = 37.1   # TFLOP/s, measured on this pool's B200 (profiles/r01_fp64_peak.txt)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled every 100 ms during the timed region, in
    process through NVML (pynvml) from a background thread: no nvidia-smi process whose start-up or
    driver queries could stall the timed region's host-side launches.  Falls back to nvidia-smi."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.samples = []   # (sm_mhz, max_mhz, set of reasons)
        self.lines = []

    def _nvml_loop(self, nv, h):
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while True:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx), {k for k, v in bits.items() if rs & v}))
            except Exception:
                pass
            self._first.set()
            if self._stop.wait(0.1):
                break

    def __enter__(self):
        import threading
        self._first, self._stop = threading.Event(), threading.Event()
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.thread = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.thread.start()
            self._first.wait(timeout=5.0)
            return self
        except Exception:
            self.thread = None
        try:   # fallback: nvidia-smi, started (and first sample taken) before the region
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self

        def reader():
            for ln in self.proc.stdout:
                if ln.strip():
                    self.lines.append(ln)
                    self._first.set()
            self._first.set()

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        self._first.wait(timeout=5.0)
        return self

    def __exit__(self, *a):
        if self.proc is None and self.thread is not None:
            time.sleep(0.06)
            self._stop.set()
            self.thread.join(timeout=5)
            return
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=5)

    def summary(self):
        sm, mx, reasons = [], None, set()
        for s_mhz, m_mhz, rs in self.samples:
            sm.append(s_mhz)
            mx = m_mhz
            reasons |= rs
        for ln in self.lines:
            p = [t.strip() for t in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.samples else "nvidia-smi"}


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------------------ reference arm
# c5's A = X^T X (3.4e13 flop) is far beyond a bounded host sample: the oracle's EXPLICIT iteration
# on the m = 4096 system costs the same for any A of that size, so the host legs build A from the
# first ORACLE_ROWS rows of the same X ("CPU oracle")
ORACLE_ROWS = 100_000


def _oracle_operator(cfg, mode, X, y):
    """The oracle's operator for `cfg` (X, y host arrays; kernel ridge: X, y are its inputs)."""
    from oracle import solver as OV
    if cfg.kind == "kernel":
        from oracle import problem as OP
        sysk = OP.build_kernel(X, y, cfg.lam, cfg.extra["sigma"])
        return OV.Operator.from_system(sysk["A"], sysk["b"])
    return OV.Operator(X, y, cfg.lam, explicit=(mode == "explicit"))


def _host_inputs(cfg, dev):
    """(X, y, sample description) on the host for the oracle legs."""
    import numpy as np
    import rsinputs
    if cfg.kind == "kernel":
        X, y = rsinputs.kernel_problem(cfg.n, cfg.d, seed=0, noise=cfg.noise)
        return X, y, "full kernel system"
    if cfg.kind == "dense":
        big = cfg.n * cfg.d * 8 > 32e9
        if big and dev == "cpu":   # no device to draw the full X on: a same-shaped row sample
            X, y = rsinputs.dense_problem(ORACLE_ROWS, cfg.d, seed=0, col_decay=cfg.col_decay,
                                          noise=cfg.noise)
            return X.numpy(), y.numpy(), (f"A = X_s^T X_s + lambda I from {ORACLE_ROWS} rows drawn "
                                          f"like X (an EXPLICIT iteration costs the same for any "
                                          f"{cfg.d} x {cfg.d} A)")
        X, y = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, col_decay=cfg.col_decay,
                                      noise=cfg.noise, device=dev)
        if big:
            X, y = X[:ORACLE_ROWS].cpu().numpy(), y[:ORACLE_ROWS].cpu().numpy()
            return X, y, (f"A = X_s^T X_s + lambda I from the first {ORACLE_ROWS} of the {cfg.n} rows "
                          f"(an EXPLICIT iteration costs the same for any {cfg.d} x {cfg.d} A)")
        return X.cpu().numpy(), y.cpu().numpy(), "full X"
    if cfg.zipf_a > 0:
        rp, ci, va, y = rsinputs.csr_zipf(cfg.n, cfg.d, cfg.nnz_per_row, a=cfg.zipf_a, seed=0)
    else:
        rp, ci, va, y = rsinputs.csr_uniform(cfg.n, cfg.d, cfg.nnz_per_row, seed=0)
    return rsinputs.csr_to_scipy(rp, ci, va, cfg.n, cfg.d), y, "full X"


def run_reference(args):
    """The oracle (oracle/, plain NumPy/SciPy fp64) on the same workload, on the host cores."""
    world, rank, _ = _dist_env()
    if rank != 0:
        return 0
    import torch
    import rsinputs
    from oracle import solver as OV
    cfg = rsinputs.CONFIGS[args.config]
    if args.mode is None:
        args.mode = DEFAULT_MODE.get(cfg.name, "gram")
    if cfg.kind == "kernel":
        args.mode = "explicit"
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    X, y, sample = _host_inputs(cfg, dev)
    if dev == "cuda":
        torch.cuda.empty_cache()
    op = _oracle_operator(cfg, args.mode, X, y)
    kw = dict(seed=0, subcount_k=cfg.subcount_k)
    OV.solve_momentum(op, cfg.sketch, cfg.tau, cfg.gamma, cfg.beta, 0.0, args.warmup, **kw)
    t0 = time.perf_counter()
    OV.solve_momentum(op, cfg.sketch, cfg.tau, cfg.gamma, cfg.beta, 0.0, args.steps, **kw)
    el = time.perf_counter() - t0
    v = args.steps / el
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(cfg, args, world),
        "cpu_baseline": {"value": v, "unit": "iters/s", "cores": cores, "kind": "oracle",
                         "sample": f"{args.steps} oracle Alg. 2 iterations of {args.config} "
                                   f"({args.mode} AS; {sample}) after {args.warmup} warm-up "
                                   f"iterations"},
        "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _config_dict(cfg, args, world):
    dual = cfg.d > cfg.n and cfg.kind != "kernel"
    if cfg.kind == "kernel":
        xb = cfg.n * cfg.n * 8
        shape = f"kernel ridge (Gaussian sigma={cfg.extra['sigma']:.3g}, A = K(K + lambda I) n x n)"
    elif cfg.kind == "dense":
        xb = cfg.n * cfg.d * 8
        shape = "dense"
    else:
        xb = cfg.n * cfg.nnz_per_row * 12
        shape = f"CSR ~{cfg.nnz_per_row} nnz/row" + (f", Zipf({cfg.zipf_a}) columns" if cfg.zipf_a
                                                      else ", uniform columns, unit rows")
    extra = f", k={cfg.subcount_k}" if cfg.sketch == "subcount" else ""
    return {"workload": f"{cfg.name}: {shape} {'dual' if dual else 'primal'} {cfg.n}x{cfg.d}, "
                        f"{cfg.sketch} tau={cfg.tau}{extra}, gamma={cfg.gamma}, beta={cfg.beta}, "
                        f"lambda={cfg.lam:g}, tol={cfg.tol:g}",
            "as_mode": args.mode, "tau": cfg.tau, "n": cfg.n, "d": cfg.d,
            "momentum": args.momentum if args.momentum == "constant" else f"{args.momentum}(eta={args.eta})",
            "parallelism": (f"X {'columns (features)' if dual else 'rows'} sharded over {world} "
                            f"GPU(s), NCCL allreduce of the partial A S"),
            "l2": "inputs larger than L2 (%s = %.2f GB > 126 MB)" % ("A" if cfg.kind == "kernel" else "X", xb / 1e9)}


def _csr_column_block(np, rowptr, colidx, vals, c0, clen):
    """Columns [c0, c0 + clen) of a CSR matrix, with local column indices (dual feature shard)."""
    keep = (colidx >= c0) & (colidx < c0 + clen)
    ck = np.concatenate([[0], np.cumsum(keep, dtype=np.int64)])
    rp = ck[rowptr].astype(np.int64)
    return rp, (colidx[keep] - c0).astype(np.int32), vals[keep]


# CSR Gram pair updates: int64 fixed-point adds (two u32 shared atomics) on random addresses,
# measured 3.26 per clock per SM (tools/ubench_atom.cu, profiles/r01_ubench_atom.txt), x 148 SMs x
# 1965 MHz, in 1e9 updates/s
SMEM_FXADD_PEAK = 3.26 * 148 * 1.965


def _traffic(cfg, args, cls, units=None):
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the
    committed capture summary profiles/traffic.json (None if not captured).  A group kernel's entry
    records the units (iterations / slots) of its captured launch; `units` = the units of a launch
    here, and the bytes are scaled to it (same per-unit basis as `achieved`)."""
    if args.traffic is not None:
        return args.traffic
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(f"{cfg.name}/{args.mode}/{cls}", {})
        b = t.get("bytes_per_launch")
        if b is not None and units and t.get("units_per_launch"):
            b = b / t["units_per_launch"] * units
        return b
    except Exception:
        return None


def _csr_pairs(rs, cfg, host):
    """Algorithmic work of the CSR Gram kernels for the sketch of iteration 0: the number of merged
    entries of R S (distinct (row, bucket) pairs) and of lower-triangle pair updates
    sum_i |v_i| (|v_i| + 1) / 2 (host NumPy over the same data)."""
    import numpy as np
    rp, ci = host[0], host[1]
    dual = cfg.d > cfg.n
    m = cfg.n if dual else cfg.d
    coord, bucket, _ = rs.rs_sketch_draw(cfg.sketch, m, cfg.tau, 0, 0, cfg.subcount_k)
    bmap = np.full(m, -1, np.int64)
    bmap[coord] = bucket
    xrow = np.repeat(np.arange(cfg.n, dtype=np.int64), np.diff(rp))
    r, b = (ci.astype(np.int64), bmap[xrow]) if dual else (xrow, bmap[ci])
    keep = b >= 0
    key = np.unique(r[keep] * cfg.tau + b[keep])
    L = np.bincount(key // cfg.tau)
    sel = None
    if dual and cfg.sketch != "count":
        # selected-row path (k_sel_emit / k_sel_merge): the X entries of the s selected samples,
        # and the entries of every R row (feature) they touch (the code scan)
        feat_nnz = np.bincount(ci, minlength=cfg.d)
        touched = np.unique(ci[keep])
        sel = (int(keep.sum()), int(feat_nnz[touched].sum()))
    return int(key.size), int((L * (L + 1) // 2).sum()), sel


def _roofline(args, cfg, world, kms, kl, dom, prof_ms, host, rs, nb=1):
    per = lambda c: max(kms[c] / max(kl[c], 1), 1e-9)   # ms per launch of class c
    share = kms[dom] / max(prof_ms, 1e-9)
    hbm = _peaks().get("hbm_gbs", 6556.5)
    hbm_src = "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    dmma_src = ("measured FP64 DMMA peak, profiles/r01_fp64_peak.txt (MEASURED_PEAKS.json has no "
                "FP64 figure)")
    n_loc = cfg.n / world
    ms = per(dom)
    roof = None
    if cfg.kind == "kernel" or (cfg.kind == "csr" and args.mode == "explicit"):
        # EXPLICIT path on the m x m system (kernel ridge: m = n; CSR: m = d primal, n dual)
        import rsinputs
        m_sys = cfg.n if (cfg.kind == "kernel" or cfg.d > cfg.n) else cfg.d
        rows_s = cfg.tau * (max(cfg.subcount_k, 1) if cfg.sketch == "subcount" else 1)
        cfg = rsinputs.Config(cfg.name, "dense", m_sys, m_sys, cfg.lam, cfg.sketch, cfg.tau,
                              extra={"rows": rows_s})
    if cfg.kind == "dense":
        if dom == "as" and args.mode == "implicit":
            w = 2.0 * n_loc * cfg.d * cfg.tau
            roof = dict(kernel="a3 A S = X^T (X S) (k_tn_gemm / TMA DMMA, split-K reduce, + lambda S)",
                        bound="tensor", achieved=w / (ms * 1e-3) / 1e12, peak=FP64_DMMA_PEAK,
                        unit="TFLOP/s", peak_source=dmma_src,
                        algorithmic_per_launch=f"{w:.3e} flop (2 n d tau)")
        elif dom == "as":
            w = n_loc * cfg.d * 8.0
            roof = dict(kernel="AS pass u = X^T (X S delta) (k_xpass_rows / k_xpass_tma: one "
                               "TMA-staged streaming read of X per iteration)", bound="hbm",
                        achieved=w / (ms * 1e-3) / 1e9, peak=hbm, unit="GB/s", peak_source=hbm_src,
                        algorithmic_per_launch=f"{w:.3e} bytes (n d 8)")
        elif dom == "gram":
            w = 1.0 * n_loc * cfg.tau * (cfg.tau + 1)   # symmetric: the lower triangle only
            roof = dict(kernel="Gram (XS)^T XS of one sketch (k_gram_xt: the tau sketched rows "
                               "of X^T, DMMA; else k_gram_fused gather or XS + TMA DMMA GEMM)",
                        bound="tensor",
                        achieved=w / (ms * 1e-3) / 1e12, peak=FP64_DMMA_PEAK, unit="TFLOP/s",
                        peak_source=dmma_src,
                        algorithmic_per_launch=f"{w:.3e} flop (n tau (tau + 1): lower triangle)")
        elif dom == "factor":
            slots = args.steps / max(kl["factor"], 1)   # iterations (G_k) per group
            # tau > 224: the slot holds W = L^{-1} (nb = 1) or the blocked inverse (W_bb = L_bb^{-1}
            # on nb diagonal super-blocks, L below), applied as triangular GEMVs
            big = cfg.tau > 224
            w = float(cfg.tau) ** 3 * ((1.0 + 1.0 / nb ** 2) / 3.0 if big else 1.0) * slots
            what = ((f"tau^3/3 Cholesky + tau^3/(3 nb^2) inverse of the nb = {nb} diagonal super-blocks"
                     if nb > 1 else "tau^3/3 Cholesky + tau^3/3 inverse") if big else
                    "tau^3/3 Cholesky + tau^3/3 inverse + tau^3/3 W^T W")
            roof = dict(kernel="batched Cholesky + triangular inverse of the group's G_k "
                               f"({'k_bf_gather + k_bfactor_lp' if big else 'k_bfactor_small'}, DMMA)",
                        bound="tensor",
                        achieved=w / (ms * 1e-3) / 1e12, peak=FP64_DMMA_PEAK, unit="TFLOP/s",
                        peak_source=dmma_src,
                        algorithmic_per_launch=f"{w:.3e} flop ({what} per G_k, x {slots:.0f} slots)",
                        _units=slots)
        elif dom == "solve" and (args.mode == "explicit" or "rows" in cfg.extra):
            w = float(cfg.tau) * cfg.tau * 8.0
            roof = dict(kernel="class solve: delta = G_k^{-1} S^T r from the factor slot (tau <= 224: "
                               "G^{-1} row GEMV; else W = L^{-1} and W^T, two triangular GEMVs, "
                               "k_apply_rows)", bound="hbm",
                        achieved=w / (ms * 1e-3) / 1e9, peak=hbm, unit="GB/s", peak_source=hbm_src,
                        algorithmic_per_launch=f"{w:.3e} bytes (tau^2 x 8: the slot's factor read once)")
        else:   # explicit: rows of A + GEMV + update (the group kernel runs a whole group per launch)
            rows_s = cfg.extra.get("rows", cfg.tau)
            its = max(1.0, round(args.steps / max(kl[dom], 1))) if kl.get("solve", 0) == 0 else 1.0
            w = (rows_s * cfg.d + 10 * cfg.d + (float(cfg.tau) * cfg.tau if its > 1 else 0.0)) * 8.0 * its
            a_mb = cfg.d * cfg.d * 8 / 1e6
            roof = dict(kernel=(f"class {dom}: the group's iterations in one persistent kernel "
                                "(k_iterate: g = S^T r, delta = G^-1 g from the factor slot, u = A S "
                                "delta from the sketched rows of A, fused momentum update)") if its > 1 else
                               (f"class {dom}: u = A S delta from the tau sketched rows of A, fused "
                                "momentum update (k_update_rows)"), bound="hbm",
                        achieved=w / (ms * 1e-3) / 1e9, peak=hbm, unit="GB/s", peak_source=hbm_src,
                        algorithmic_per_launch=f"{w:.3e} bytes ({rows_s} sketched rows of A x m x 8 + 10 m-vectors"
                                               + (f" + the tau^2 slot, x {its:.0f} iterations)" if its > 1 else ")"),
                        note=f"A = {a_mb:.0f} MB ({'fits' if a_mb < 126 else 'exceeds'} the 126 MB L2)",
                        _units=its)
    else:
        nnz = int(host[0][-1])
        m = cfg.d if cfg.d <= cfg.n else cfg.n
        if args.mode == "gram" and dom in ("gram", "xs"):
            ent, pairs, sel = _csr_pairs(rs, cfg, host)
            if dom == "gram":
                w = pairs / world
                roof = dict(kernel="k_gram_bands: G_lower += v_i v_i^T over the merged rows of R S "
                                   "(one int64 fixed-point shared-memory add per pair)", bound="alu",
                            achieved=w / (ms * 1e-3) / 1e9, peak=SMEM_FXADD_PEAK, unit="Gupdates/s",
                            peak_source="shared-memory fixed-point add on random addresses "
                                        "(2 x u32 atomics, tools/ubench_atom.cu on this pool's "
                                        "B200: 3.26 per clk per SM) x 148 SMs x 1965 MHz",
                            algorithmic_per_launch=f"{w:.3e} pair updates (sketch of iteration 0)")
            elif sel is not None:   # dual, subsample / SubCount: the selected-row path
                se, tn = sel
                rows_r = cfg.d
                w = (se * 12.0 + tn * 4.0 + ent * 20.0 + rows_r * 4.0) / world
                roof = dict(kernel="k_sel_emit + k_sel_merge + k_sel_heavy: rows of R S from the s "
                                   "selected samples", bound="hbm",
                            achieved=w / (ms * 1e-3) / 1e9, peak=hbm, unit="GB/s",
                            peak_source=hbm_src,
                            algorithmic_per_launch=f"{w:.3e} bytes ({se:.3e} selected X entries x "
                                                   f"12 B, {tn:.3e} codes of the touched R rows x "
                                                   f"4 B, {ent:.3e} merged entries x 20 B, hcnt "
                                                   f"reset)")
            else:
                w = (nnz * 16.0 + ent * 12.0) / world
                roof = dict(kernel="k_hash_rows: rows of R S, merged and bucket-sorted", bound="hbm",
                            achieved=w / (ms * 1e-3) / 1e9, peak=hbm, unit="GB/s",
                            peak_source=hbm_src,
                            algorithmic_per_launch=f"{w:.3e} bytes (R read 12 B/nnz + cmap 4 B/nnz, "
                                                   f"{ent:.3e} merged entries written)")
        elif args.mode == "gram":
            w = 2.0 * nnz * 12 / world + 4.0 * m * 8
            roof = dict(kernel=f"class {dom}: A S delta = R^T (R (S delta)) (two SpMV, k_spmv)",
                        bound="hbm", achieved=w / (ms * 1e-3) / 1e9, peak=hbm, unit="GB/s",
                        peak_source=hbm_src,
                        algorithmic_per_launch=f"{w:.3e} bytes (R as CSR and CSC read once)")
        else:
            w = 2.0 * nnz * 12 / world + m * cfg.tau * 8.0
            roof = dict(kernel=("a2+a3 CSR primal A S = X^T (X S) (warp per coordinate, CSC x CSR)"
                                if m == cfg.d else
                                "a2+a3 CSR dual A S = X (X^T S) (hashed z_b, warp per row)"),
                        bound="hbm", achieved=w / (ms * 1e-3) / 1e9, peak=hbm, unit="GB/s",
                        peak_source=hbm_src,
                        algorithmic_per_launch=f"{w:.3e} bytes (X as CSR + CSC read once, A S written)")
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = _traffic(cfg, args, dom, roof.pop("_units", None))
    roof["avg_launch_ms"] = ms
    roof["share_of_step"] = share
    return roof


# ------------------------------------------------------------------------------ our arm
def _quartiles(xs):
    xs = sorted(xs)
    if len(xs) == 1:
        return xs[0], xs[0], xs[0]
    q = statistics.quantiles(xs, n=4, method="inclusive")
    return q[0], statistics.median(xs), q[2]


def run_ours(args):
    import numpy as np
    import torch
    import rsinputs
    from paper_2105_05565_b200 import build
    build()
    from paper_2105_05565_b200 import ridgesketch as rs

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    dist = None
    pg = None
    if world > 1:
        import torch.distributed as tdist
        # NCCL's own log (stderr) shows the transport (NVLS / P2P) and each communicator's nranks
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = tdist
        obj = [rs.rs_nccl_unique_id() if rank == 0 else None]
        tdist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    cfg = rsinputs.CONFIGS[args.config]
    stream = torch.cuda.current_stream()
    if args.mode is None:
        args.mode = DEFAULT_MODE.get(cfg.name, "gram")
    big = cfg.kind == "dense" and cfg.n * cfg.d * 8 > 32e9   # c5: 65.5 GB of X
    if cfg.kind == "kernel":
        if world > 1:
            raise SystemExit("kernel ridge route: one GPU (rs_create_kernel v1)")
        Xk, yk = rsinputs.kernel_problem(cfg.n, cfg.d, seed=0, noise=cfg.noise)
        Xd, yd = torch.from_numpy(Xk).cuda(), torch.from_numpy(yk).cuda()
        b0, ln = 0, cfg.n
        host = None
        args.mode = "explicit"
    elif cfg.kind == "dense":
        Xd, yd = rsinputs.dense_problem(cfg.n, cfg.d, seed=0, col_decay=cfg.col_decay,
                                        noise=cfg.noise, device="cuda")
        b0, ln = rs.rs_shard_range(cfg.n, rank, world)
        if world > 1:
            Xd = Xd[b0:b0 + ln].contiguous()
            yd = yd[b0:b0 + ln].contiguous()
        host = None
    else:   # CSR (c3 primal: row shards balanced by nnz; c4 dual: feature (column) shards)
        if cfg.zipf_a > 0:
            rp, ci, va, yv = rsinputs.csr_zipf(cfg.n, cfg.d, cfg.nnz_per_row, a=cfg.zipf_a, seed=0)
        else:
            rp, ci, va, yv = rsinputs.csr_uniform(cfg.n, cfg.d, cfg.nnz_per_row, seed=0)
        host = (rp, ci, va, yv)
        dual = cfg.d > cfg.n
        if dual:   # contiguous feature ranges balanced by nnz (Zipf popularity: plain ranges of
                   # d / world features would give rank 0 most of the entries)
            colptr = np.concatenate([[0], np.cumsum(np.bincount(ci, minlength=cfg.d))]).astype(np.int64)
            b0, ln = rs.rs_shard_rows_nnz(colptr, rank, world)
            rp, ci, va = _csr_column_block(np, rp, ci, va, b0, ln)
        else:
            b0, ln = rs.rs_shard_rows_nnz(rp, rank, world)
            e0, e1 = rp[b0], rp[b0 + ln]
            rp, ci, va, yv = rp[b0:b0 + ln + 1] - e0, ci[e0:e1], va[e0:e1], yv[b0:b0 + ln]
        Xd = (torch.from_numpy(np.ascontiguousarray(rp)).cuda(),
              torch.from_numpy(np.ascontiguousarray(ci)).cuda(),
              torch.from_numpy(np.ascontiguousarray(va)).cuda())
        yd = torch.from_numpy(np.ascontiguousarray(yv)).cuda()
    if world > 1:
        dist = dict(device=local, rank=rank, world=world, nccl_unique_id=uid,
                    cuda_stream=stream.cuda_stream, shard_begin=b0, shard_len=ln)
    else:
        dist = dict(device=local, rank=0, world=1, cuda_stream=stream.cuda_stream,
                    shard_begin=0, shard_len=ln)

    def create(X, y, borrow, mode=None):
        if cfg.kind == "kernel":
            return rs.rs_create_kernel(X, y, cfg.lam, cfg.extra["sigma"])
        if cfg.kind == "dense":
            return rs.rs_create_dense(X, y, cfg.lam, mode=mode or args.mode, n=cfg.n, d=cfg.d,
                                      borrow=borrow, dist=dist)
        return rs.rs_create_csr(cfg.n, cfg.d, X[0], X[1], X[2], y, cfg.lam, mode=mode or args.mode,
                                dist=dist)

    def barrier():
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(ms):
        if pg is None:
            return ms
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        return float(t.item())

    def timed(h, **kw):
        """(device ms, report) of one rs_solve, CUDA events on the solver stream, max over ranks."""
        barrier()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        out = rs.rs_solve(h, **kw)
        eb.record(stream)
        barrier()
        return max_over_ranks(ea.elapsed_time(eb)), out[1]

    common = dict(kind=cfg.sketch, tau=cfg.tau, gamma=cfg.gamma, beta=cfg.beta, seed=0,
                  subcount_k=cfg.subcount_k, d=cfg.n if cfg.kind == "kernel" else cfg.d,
                  momentum=args.momentum, eta=args.eta)

    def chunk_of(mode, steps):
        # iterations per graph launch: EXPLICIT iterations are a few kernel nodes each (1024 per
        # graph); GRAM / IMPLICIT groups add several nodes per sketch-ahead slot, and a graph of
        # 10k+ nodes delays its own submission (256 per graph)
        return min(steps, 1024 if (mode == "explicit" or cfg.kind == "kernel") else 256)

    def measure(h, mode, steps, warmup, clk=None):
        """iters/s over exactly `steps` iterations (tol = 0) after `warmup` untimed ones with the
        same launch parameters (so the captured iteration graph exists before the timed region),
        then the per-class breakdown from a separate profiled run (events perturb the step)."""
        chunk = chunk_of(mode, steps)
        rs.rs_solve(h, tol=0.0, max_iter=warmup, check_every=chunk, **common)
        if clk is not None:
            with clk:
                el_ms, rep = timed(h, tol=0.0, max_iter=steps, check_every=chunk, **common)
        else:
            el_ms, rep = timed(h, tol=0.0, max_iter=steps, check_every=chunk, **common)
        assert rep["iterations"] == steps, rep
        rs.rs_solve(h, tol=0.0, max_iter=warmup, check_every=chunk, profile=True, **common)
        _, rep_prof = rs.rs_solve(h, tol=0.0, max_iter=steps, check_every=chunk, profile=True,
                                  **common)
        kms, kl = rep_prof["kernel_ms"], rep_prof["kernel_launches"]
        prof_ms = rep_prof["solve_seconds"] * 1e3
        dom = max(kms, key=lambda k: kms[k])
        saved = args.mode
        args.mode = mode
        roof = _roofline(args, cfg, world, kms, kl, dom, prof_ms, host, rs,
                         nb=int(rep_prof.get("inverse_blocks") or 1))
        others = {}
        for cls in sorted(kms, key=lambda k: -kms[k]):
            if cls != dom and kms[cls] > 0.1 * prof_ms:
                try:
                    o = _roofline(args, cfg, world, kms, kl, cls, prof_ms, host, rs,
                                  nb=int(rep_prof.get("inverse_blocks") or 1))
                    others[cls] = {k: o[k] for k in ("kernel", "bound", "achieved", "peak", "unit",
                                                     "frac", "traffic", "avg_launch_ms",
                                                     "share_of_step") if k in o}
                except Exception:
                    pass
        args.mode = saved
        ov = int(rep_prof.get("overlap_sms") or 0)
        if ov:   # overlapped pipeline: the group kernel on `ov` SMs, the factorisation on the rest
            n_sms = torch.cuda.get_device_properties(local).multi_processor_count
            for cls, o in [(dom, roof)] + list(others.items()):
                sms = ov if cls == "update" else (n_sms - ov if cls == "factor" else None)
                if sms and o.get("frac") is not None:
                    o["sms"] = sms
                    o["frac_of_sm_share"] = o["frac"] * n_sms / sms
                    o["note_sms"] = (f"runs concurrently on {sms} of {n_sms} SMs by design; "
                                     "frac_of_sm_share = achieved / (peak x sms / n_sms)")
        roof["step_share_by_class"] = {k: kms[k] / max(prof_ms, 1e-9) for k in kms}
        roof["dominant_class"] = dom
        if others:
            roof["other_classes"] = others
        return steps / (el_ms / 1e3), el_ms, rep, roof, {k: kms[k] / steps for k in kms}

    torch.cuda.synchronize()
    h = create(Xd, yd, True)
    clk = ClockSampler(local)
    value, el_ms, rep, roof, kms_step = measure(h, args.mode, args.steps, args.warmup, clk)

    # time to tolerance (second half of the metric): device time of rs_solve to ||r||/||b|| <= tol
    # for sketch seeds 0 .. seeds-1 (the paper reports medians and quartiles over runs);
    # each seed's first solve builds its graph (untimed)
    tol_runs = []
    for sd in range(args.seeds):
        kw = dict(common, seed=sd)
        rs.rs_solve(h, tol=cfg.tol, max_iter=args.max_iter_tol, check_every=0, **kw)
        ms, rp_ = timed(h, tol=cfg.tol, max_iter=args.max_iter_tol, check_every=0, **kw)
        tol_runs.append((sd, ms / 1e3, rp_["iterations"], rp_["converged"], rp_["rel_residual"]))
    setup_s = rep["setup_seconds"]
    rs.rs_destroy(h)
    t_q = _quartiles([t for _, t, _, _, _ in tol_runs])
    i_q = _quartiles([i for _, _, i, _, _ in tol_runs])
    seeds_rec = {"seeds": [s_ for s_, _, _, _, _ in tol_runs],
                 "seconds": [t for _, t, _, _, _ in tol_runs],
                 "iterations": [i for _, _, i, _, _ in tol_runs],
                 "converged": [c for _, _, _, c, _ in tol_runs],
                 "seconds_q1_median_q3": list(t_q), "iterations_q1_median_q3": list(i_q)}
    conv_all = all(c for _, _, _, c, _ in tol_runs)

    # the other routes on the same resident data (informational; device time).  EXPLICIT pays the
    # A = X^T X + lambda I build once (rs_create's setup_seconds: device work only, no allocator
    # time) and then never streams X; GRAM streams X once per iteration; IMPLICIT forms A S on the
    # FP64 tensor cores every iteration.
    alt = {}
    if cfg.kind == "dense" and world == 1 and not args.no_alt:
        routes = ["gram", "implicit"] if args.mode == "explicit" else ["explicit"]
        for mode in routes:
            if mode == args.mode:
                continue
            try:
                ha = create(Xd, yd, True, mode)
                steps_a = {"explicit": args.steps, "gram": 8 if big else args.steps,
                           "implicit": 2 if big else 20}[mode]
                warm_a = 3 if mode != "implicit" or not big else 1
                v_a, _, rep_a, roof_a, _ = measure(ha, mode, steps_a, warm_a)
                rec = {"iters_per_s": v_a, "steps": steps_a, "warmup": warm_a,
                       "setup_s": rep_a["setup_seconds"],
                       "roofline": {k: roof_a[k] for k in ("kernel", "bound", "achieved", "peak",
                                                           "unit", "frac", "dominant_class",
                                                           "share_of_step") if k in roof_a}}
                if mode == "explicit" or steps_a * 8 >= i_q[1]:
                    rs.rs_solve(ha, tol=cfg.tol, max_iter=args.max_iter_tol, check_every=0,
                                **common)
                    ms, rp_ = timed(ha, tol=cfg.tol, max_iter=args.max_iter_tol, check_every=0,
                                    **common)
                    rec.update(time_to_tol_s=ms / 1e3, iterations_to_tol=rp_["iterations"],
                               converged=rp_["converged"])
                else:   # same sketch stream, same iterates: the headline route's iteration count
                    rec.update(time_to_tol_s_extrapolated=tol_runs[0][2] / v_a,
                               note=f"extrapolated: {tol_runs[0][2]} iterations (seed 0, same "
                                    f"sketch stream) / measured iters/s")
                rec["time_to_tol_incl_setup_s"] = rec.get(
                    "time_to_tol_s", rec.get("time_to_tol_s_extrapolated", 0.0)) + rec["setup_s"]
                rs.rs_destroy(ha)
                alt[mode] = rec
            except Exception as ex:   # an informational leg must not sink the line
                alt[mode] = {"error": str(ex)[:300]}

    # end to end through the public API from pinned host buffers (rank-local shard): H2D of X and
    # y, rs_create (setup: A build / b), rs_solve to tol, w to the host -- all inside the region
    e2e = None
    Xh = None
    if not args.no_e2e:
        try:
            if cfg.kind in ("dense", "kernel"):
                Xh = torch.empty(tuple(Xd.shape), dtype=torch.float64, pin_memory=True)
                Xh.copy_(Xd)
            else:
                Xh = tuple(t.cpu().pin_memory() for t in Xd)
            yh = yd.cpu().pin_memory()
            if big:   # the device copy is the library's from here on: free the resident one
                del Xd
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
                Xd = None
            h2d = sum(t.numel() * t.element_size() for t in (Xh if isinstance(Xh, tuple) else (Xh,)))
            h2d += yh.numel() * 8
            barrier()
            e4, e5 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e4.record(stream)
            h2 = create(Xh, yh, False)
            w, rep_e2e = rs.rs_solve(h2, tol=cfg.tol, max_iter=args.max_iter_tol, check_every=0,
                                     **common)
            e5.record(stream)
            barrier()
            rs.rs_destroy(h2)
            e2e_ms = max_over_ranks(e4.elapsed_time(e5))
            e2e = {"value": rep_e2e["iterations"] / (e2e_ms / 1e3), "unit": "iters/s",
                   "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(w.size * 8),
                   "step": "one public-API solve: rs_create_(dense|csr)(pinned host X, y) + rs_solve "
                           "to tol + w to host",
                   "seconds": e2e_ms / 1e3, "iterations": rep_e2e["iterations"],
                   "setup_s": rep_e2e["setup_seconds"], "solve_s": rep_e2e["solve_seconds"]}
        except Exception as ex:
            e2e = {"skipped": f"{type(ex).__name__}: {str(ex)[:300]}"}

    # CPU baseline: the oracle on a bounded sample, rank 0, N = 1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import solver as OV
        if host is not None:
            X = rsinputs.csr_to_scipy(host[0], host[1], host[2], cfg.n, cfg.d)
            y = host[3]
            sample = "full X"
        elif cfg.kind == "kernel":
            X, y = Xk, yk
            sample = "full kernel system"
        elif big:
            src = Xh if isinstance(Xh, torch.Tensor) else Xd
            X = src[:ORACLE_ROWS].cpu().numpy()
            y = yd[:ORACLE_ROWS].cpu().numpy()
            sample = (f"A = X_s^T X_s + lambda I from the first {ORACLE_ROWS} of the {cfg.n} rows "
                      f"(an EXPLICIT iteration costs the same for any {cfg.d} x {cfg.d} A)")
        else:
            X = Xd.cpu().numpy() if Xd is not None else Xh.numpy()
            y = yd.cpu().numpy()
            sample = "full X"
        op = _oracle_operator(cfg, args.mode, X, y)
        kw = dict(seed=0, subcount_k=cfg.subcount_k)
        OV.solve_momentum(op, cfg.sketch, cfg.tau, cfg.gamma, cfg.beta, 0.0, 1, **kw)
        t0 = time.perf_counter()
        n_it = 0
        while time.perf_counter() - t0 < args.cpu_seconds:
            n_it += 1
            OV.solve_momentum(op, cfg.sketch, cfg.tau, cfg.gamma, cfg.beta, 0.0, 1, **kw)
        el = time.perf_counter() - t0
        cpu = {"value": n_it / el, "unit": "iters/s", "cores": os.cpu_count(), "kind": "oracle",
               "sample": f"{n_it} oracle Alg. 2 iterations of {cfg.name} ({args.mode} AS; "
                         f"{sample}; NumPy/SciPy fp64, BLAS on all host cores, 1 warm-up iteration "
                         f"excluded), {el:.1f} s"}
        del X, y, op

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": el_ms / args.steps,
            "higher_is_better": True, "scaling": "strong",   # one solve, X sharded over ranks
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded; DESIGN.md §5 recipe for BASELINE.json " + cfg.name + ")",
            "config": _config_dict(cfg, args, world),
            "time_to_tol_s": t_q[1], "iterations_to_tol": i_q[1],
            "time_to_tol_seeds": seeds_rec,
            "time_to_tol_incl_setup_s": t_q[1] + setup_s,
            "setup_s": setup_s,
            "setup": "device work of rs_create: b = X^T y (+ explicit A = X^T X + lambda I, CSC copy)",
            "converged": conv_all, "rel_residual": tol_runs[0][4],
            "alt_routes": alt or None,
            "e2e": e2e, "gpu_launches": rep["gpu_launches"], "roofline": roof,
            "cpu_baseline": cpu, "clocks": clk.summary(),
            "kernel_ms_per_step": kms_step,
        }
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.barrier()
        pg.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)   # a timed region of ~0.4 s on c2
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--mode", default=None, choices=["implicit", "explicit", "gram"],
                    help="how A S is formed (default: DEFAULT_MODE of the config)")
    ap.add_argument("--seeds", type=int, default=5, help="sketch seeds of the time-to-tol runs")
    ap.add_argument("--no-alt", action="store_true", help="skip the other routes' measurements")
    ap.add_argument("--max-iter-tol", type=int, default=20000)
    ap.add_argument("--momentum", default="constant", choices=["constant", "heuristic", "theory", "cor1"],
                    help="momentum schedule (BASELINE.json configs: constant gamma, beta)")
    ap.add_argument("--eta", type=float, default=0.995)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the dominant kernel (from profiles/)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
