"""Thin ctypes binding of libridgesketch.so (include/ridgesketch.h) -- argument marshalling only.

Every function has the C name; arrays may be NumPy arrays (host memory) or torch tensors (host or
CUDA memory -- CUDA tensors are passed as device pointers).  All computation happens in the
library's CUDA kernels; if the library is missing this module raises at import time: there is no
CPU fallback.

    h = rs_create_dense(X, y, lam)                 # X (n, d) float64, y (n,)
    w, rep = rs_solve(h, "subsample", tau=200, beta=0.5, tol=1e-4, max_iter=10_000)
    rs_destroy(h)

`RidgeSketch(alpha, algo_mode="mom", solver="subsample", sketch_size=...)` mirrors the paper's
package entry point.
"""

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libridgesketch.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2105_05565_b200._build` "
                      "(the CUDA library is required; there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

# ------------------------------------------------------------------------------------------ enums
RS_OK, RS_EINVAL, RS_EUNSUPPORTED, RS_ENOMEM, RS_ECUDA, RS_ENCCL, RS_ENOTSPD, RS_EDIVERGED = range(8)
ROUTES = {"auto": 0, "primal": 1, "dual": 2}
MODES = {"implicit": 0, "explicit": 1, "gram": 2}
SKETCHES = {"subsample": 0, "count": 1, "subcount": 2}
MEM_HOST, MEM_DEVICE_COPY, MEM_DEVICE_BORROW = 0, 1, 2
KERNEL_CLASSES = ("sketch", "xs", "as", "solve", "update", "gram", "pre", "factor")


class rs_dist(C.Structure):
    _fields_ = [("device", C.c_int), ("rank", C.c_int), ("world", C.c_int),
                ("nccl_unique_id", C.c_void_p), ("cuda_stream", C.c_void_p),
                ("shard_begin", C.c_int64), ("shard_len", C.c_int64), ("collective", C.c_int)]
COLLECTIVES = {"nccl": 0, "host": 1}


class rs_solve_opts(C.Structure):
    _fields_ = [("kind", C.c_int), ("tau", C.c_int64), ("subcount_k", C.c_int64),
                ("gamma", C.c_double), ("beta", C.c_double), ("tol", C.c_double),
                ("max_iter", C.c_int64), ("seed", C.c_uint64), ("check_every", C.c_int64),
                ("trace", C.c_void_p), ("trace_cap", C.c_int64), ("profile", C.c_int),
                ("momentum", C.c_int), ("eta", C.c_double)]


MOMENTUM = {"constant": 0, "heuristic": 1, "theory": 2, "cor1": 3}


class rs_report(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("converged", C.c_int), ("rel_residual", C.c_double),
                ("setup_seconds", C.c_double), ("solve_seconds", C.c_double),
                ("trace_len", C.c_int64), ("kernel_ms", C.c_double * 8),
                ("kernel_launches", C.c_int64 * 8), ("gpu_launches", C.c_int64),
                ("overlap_sms", C.c_int32), ("inverse_blocks", C.c_int32)]


_P = C.c_void_p
_lib.rs_create_dense.argtypes = [C.POINTER(_P), C.c_int64, C.c_int64, _P, C.c_int64, _P, C.c_double,
                                 C.c_int, C.c_int, C.c_int, C.POINTER(rs_dist)]
_lib.rs_create_csr.argtypes = [C.POINTER(_P), C.c_int64, C.c_int64, C.c_int64, _P, _P, _P, _P,
                               C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(rs_dist)]
_lib.rs_create_kernel.argtypes = [C.POINTER(_P), C.c_int64, C.c_int64, _P, C.c_int64, _P, C.c_double,
                                  C.c_double, C.c_int, C.POINTER(rs_dist)]
_lib.rs_solve.argtypes = [_P, C.POINTER(rs_solve_opts), _P, C.c_int, _P, C.POINTER(rs_report)]
_lib.rs_get_state.argtypes = [_P, _P, _P, C.c_int]
_lib.rs_get_info.argtypes = [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int)]
_lib.rs_sketch_draw.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int64,
                                C.c_int, _P, _P, _P, C.POINTER(C.c_int64)]
_lib.rs_shard_range.argtypes = [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                C.POINTER(C.c_int64)]
_lib.rs_shard_rows_nnz.argtypes = [C.c_int64, _P, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int64)]
_lib.rs_nccl_unique_id.argtypes = [_P]
_lib.rs_host_coll_id.argtypes = [_P]
_lib.rs_destroy.argtypes = [_P]
_lib.rs_destroy.restype = None
_lib.rs_status_string.argtypes = [C.c_int]
_lib.rs_status_string.restype = C.c_char_p
_lib.rs_last_error.restype = C.c_char_p
_lib.rs_abi_version.restype = C.c_int
_ABI = 5   # rs_report / rs_solve_opts layouts above
if _lib.rs_abi_version() != _ABI:
    raise ImportError(f"libridgesketch.so ABI {_lib.rs_abi_version()} != binding ABI {_ABI}: rebuild "
                      "(python -m paper_2105_05565_b200._build)")
for _f in ("rs_create_dense", "rs_create_csr", "rs_solve", "rs_get_state", "rs_get_info",
           "rs_sketch_draw", "rs_shard_range", "rs_shard_rows_nnz", "rs_nccl_unique_id",
           "rs_host_coll_id"):
    getattr(_lib, _f).restype = C.c_int


class RSError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        detail = _lib.rs_last_error().decode(errors="replace")
        super().__init__(f"{where}: {_lib.rs_status_string(status).decode()} -- {detail}")


def _check(st, where):
    if st != RS_OK:
        raise RSError(st, where)


def rs_status_string(s):
    return _lib.rs_status_string(int(s)).decode()


def rs_last_error():
    return _lib.rs_last_error().decode(errors="replace")


def rs_abi_version():
    return _lib.rs_abi_version()


# ------------------------------------------------------------------------------------ marshalling
def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _arr(x, dtype):
    """(pointer, mem, keepalive, is_device) for a NumPy array or torch tensor.  A CUDA tensor's
    producer stream is synchronised first: the library works on its own stream, which is not
    ordered with torch's (include/ridgesketch.h: device inputs must be complete at the call)."""
    if _is_torch(x):
        import torch
        tdt = {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32}[dtype]
        if x.dtype != tdt:
            raise TypeError(f"expected {tdt}, got {x.dtype}")
        if not x.is_contiguous():
            x = x.contiguous()
        dev = x.is_cuda
        if dev:
            torch.cuda.current_stream(x.device).synchronize()
        return x.data_ptr(), (MEM_DEVICE_COPY if dev else MEM_HOST), x, dev
    a = np.ascontiguousarray(x, dtype=dtype)
    return a.ctypes.data, MEM_HOST, a, False


def _dist(dist):
    if dist is None:
        return None
    d = rs_dist()
    d.device = dist.get("device", 0)
    d.rank = dist.get("rank", 0)
    d.world = dist.get("world", 1)
    uid = dist.get("nccl_unique_id")
    if uid is not None:
        buf = C.create_string_buffer(bytes(uid), 128)
        d._uid = buf
        d.nccl_unique_id = C.cast(buf, C.c_void_p)
    d.cuda_stream = dist.get("cuda_stream") or None
    d.shard_begin = dist.get("shard_begin", 0)
    d.shard_len = dist["shard_len"]
    d.collective = COLLECTIVES[dist.get("collective", "nccl")]
    return d


# ---------------------------------------------------------------------------------------- calls
def rs_create_dense(X, y, lam, route="auto", mode="implicit", n=None, d=None, borrow=False,
                    dist=None):
    """X: (rows, d) row-major float64 (the rank's shard when dist is given); n, d global dims."""
    rows, dd = X.shape
    n = rows if n is None else n
    d = dd if d is None else d
    xp, mem, xk, dev = _arr(X, np.float64)
    yp, ymem, yk, ydev = _arr(y, np.float64)
    if dev != ydev:
        raise ValueError("X and y must both be host or both be device arrays")
    if borrow and dev:
        mem = MEM_DEVICE_BORROW
    h = _P()
    ds = _dist(dist)
    st = _lib.rs_create_dense(C.byref(h), n, d, xp, dd, yp, float(lam), ROUTES[route], MODES[mode],
                              mem, C.byref(ds) if ds is not None else None)
    _check(st, "rs_create_dense")
    return h


def rs_create_csr(n, d, rowptr, colidx, vals, y, lam, route="auto", mode="implicit", dist=None):
    rp, mem, rk, dev = _arr(rowptr, np.int64)
    cp, _, ck, _ = _arr(colidx, np.int32)
    vp, _, vk, _ = _arr(vals, np.float64)
    yp, _, yk, _ = _arr(y, np.float64)
    nnz = int(vals.shape[0])
    h = _P()
    ds = _dist(dist)
    st = _lib.rs_create_csr(C.byref(h), n, d, nnz, rp, cp, vp, yp, float(lam), ROUTES[route],
                            MODES[mode], mem, C.byref(ds) if ds is not None else None)
    _check(st, "rs_create_csr")
    return h


def rs_create_kernel(X, y, lam, sigma, dist=None):
    """Kernel ridge regression problem (rs_create_kernel): A = K (K + lam I), b = K y with the
    Gaussian kernel of bandwidth sigma; rs_solve then returns alpha (n)."""
    n, d = X.shape
    xp, mem, xk, dev = _arr(X, np.float64)
    yp, ymem, yk, ydev = _arr(y, np.float64)
    if dev != ydev:
        raise ValueError("X and y must both be host or both be device arrays")
    h = _P()
    ds = _dist(dist)
    _check(_lib.rs_create_kernel(C.byref(h), n, d, xp, d, yp, float(lam), float(sigma), mem,
                                 C.byref(ds) if ds is not None else None), "rs_create_kernel")
    return h


def rs_get_info(h):
    m = C.c_int64()
    r = C.c_int()
    _check(_lib.rs_get_info(h, C.byref(m), C.byref(r)), "rs_get_info")
    return m.value, {1: "primal", 2: "dual"}[r.value]


def rs_solve(h, kind="subsample", tau=1, gamma=1.0, beta=0.0, tol=0.0, max_iter=100, seed=0,
             subcount_k=0, check_every=0, trace_cap=0, profile=False, w_out=None, alpha=False,
             d=None, momentum="constant", eta=0.995):
    """Run Alg. 2.  Returns (w, report_dict[, trace]) where w is a NumPy array (host), or the
    given `w_out` (a CUDA tensor: written on the device).  momentum: "constant" (gamma, beta) or
    a schedule "heuristic" | "theory" | "cor1" with parameter eta (rs_momentum)."""
    m, route = rs_get_info(h)
    o = rs_solve_opts()
    o.kind = SKETCHES[kind]
    o.tau = int(tau)
    o.subcount_k = int(subcount_k)
    o.gamma = float(gamma)
    o.beta = float(beta)
    o.tol = float(tol)
    o.max_iter = int(max_iter)
    o.seed = int(seed)
    o.check_every = int(check_every)
    trace = np.zeros(max(int(trace_cap), 1))
    o.trace = trace.ctypes.data if trace_cap else None
    o.trace_cap = int(trace_cap)
    o.profile = 1 if profile else 0
    o.momentum = MOMENTUM[momentum]
    o.eta = float(eta)
    rep = rs_report()
    if w_out is None:
        if d is None:
            d = m if route == "primal" else None
        if d is None:
            raise ValueError("dual route: pass d= (number of features) or w_out")
        w = np.zeros(d)
        wp, wmem = w.ctypes.data, MEM_HOST
    else:
        w = w_out
        wp, wmem = (w.data_ptr(), MEM_DEVICE_COPY) if _is_torch(w) and w.is_cuda else (w.ctypes.data, MEM_HOST)
    al = np.zeros(m) if (alpha and route == "dual") else None
    st = _lib.rs_solve(h, C.byref(o), wp, wmem, al.ctypes.data if al is not None else None,
                       C.byref(rep))
    _check(st, "rs_solve")
    report = dict(iterations=rep.iterations, converged=bool(rep.converged),
                  rel_residual=rep.rel_residual, setup_seconds=rep.setup_seconds,
                  solve_seconds=rep.solve_seconds,
                  kernel_ms={k: rep.kernel_ms[i] for i, k in enumerate(KERNEL_CLASSES)},
                  kernel_launches={k: rep.kernel_launches[i] for i, k in enumerate(KERNEL_CLASSES)},
                  gpu_launches=rep.gpu_launches, overlap_sms=rep.overlap_sms,
                  inverse_blocks=rep.inverse_blocks)
    if trace_cap:
        report["trace"] = trace[:rep.trace_len].copy()
    if al is not None:
        report["alpha"] = al
    return w, report


def rs_get_state(h):
    """(system iterate, maintained residual) as NumPy arrays (w in primal, alpha in dual)."""
    m, _ = rs_get_info(h)
    w = np.zeros(m)
    r = np.zeros(m)
    _check(_lib.rs_get_state(h, w.ctypes.data, r.ctypes.data, MEM_HOST), "rs_get_state")
    return w, r


def rs_sketch_draw(kind, m, tau, seed, it, subcount_k=0, device=0):
    """Entries (coord, bucket, sign) of S_it in bucket order, drawn by the library's GPU kernel."""
    coord = np.zeros(m, dtype=np.int32)
    bucket = np.zeros(m, dtype=np.int32)
    sign = np.zeros(m, dtype=np.int8)
    n = C.c_int64()
    _check(_lib.rs_sketch_draw(SKETCHES[kind], m, tau, subcount_k, C.c_uint64(seed), it, device,
                               coord.ctypes.data, bucket.ctypes.data, sign.ctypes.data,
                               C.byref(n)), "rs_sketch_draw")
    L = n.value
    return coord[:L].copy(), bucket[:L].copy(), sign[:L].copy()


def rs_shard_range(total, rank, world):
    b = C.c_int64()
    n = C.c_int64()
    _check(_lib.rs_shard_range(total, rank, world, C.byref(b), C.byref(n)), "rs_shard_range")
    return b.value, n.value


def rs_shard_rows_nnz(rowptr, rank, world):
    rp = np.ascontiguousarray(rowptr, dtype=np.int64)
    b = C.c_int64()
    n = C.c_int64()
    _check(_lib.rs_shard_rows_nnz(rp.shape[0] - 1, rp.ctypes.data, rank, world, C.byref(b),
                                  C.byref(n)), "rs_shard_rows_nnz")
    return b.value, n.value


def rs_nccl_unique_id():
    buf = C.create_string_buffer(128)
    _check(_lib.rs_nccl_unique_id(buf), "rs_nccl_unique_id")
    return buf.raw


def rs_host_coll_id():
    """128-byte name of a fresh host-staged collective group (rs_dist collective "host")."""
    buf = C.create_string_buffer(128)
    _check(_lib.rs_host_coll_id(buf), "rs_host_coll_id")
    return buf.raw


def rs_destroy(h):
    _lib.rs_destroy(h)


# ------------------------------------------------------------------------------ paper-style API
class RidgeSketch:
    """RidgeSketch(alpha, algo_mode="mom", solver="subsample", sketch_size=tau).

    algo_mode: "mom" (constant gamma, beta), "plain" (gamma=1, beta=0, Alg. 1), or a
    momentum schedule "heuristic" | "theory" | "cor1" (parameter eta; rs_momentum).
    solver: "subsample" | "count" | "subcount".  fit(X, y) accepts dense NumPy / torch arrays or a
    scipy.sparse CSR matrix, and stores the weights in `coef_`."""

    def __init__(self, alpha=1.0, algo_mode="mom", solver="subsample", sketch_size=10, gamma=1.0,
                 beta=0.5, tol=1e-4, max_iter=10_000, seed=0, subcount_k=0, as_mode="implicit",
                 route="auto", eta=0.995):
        self.alpha, self.algo_mode, self.solver, self.sketch_size = alpha, algo_mode, solver, sketch_size
        self.gamma, self.beta = (1.0, 0.0) if algo_mode == "plain" else (gamma, beta)
        self.tol, self.max_iter, self.seed, self.subcount_k = tol, max_iter, seed, subcount_k
        self.as_mode, self.route = as_mode, route
        self.momentum = algo_mode if algo_mode in ("heuristic", "theory", "cor1") else "constant"
        self.eta = eta
        self.coef_ = None
        self.report_ = None

    def fit(self, X, y):
        try:
            import scipy.sparse as sp
            sparse = sp.issparse(X)
        except ImportError:
            sparse = False
        if sparse:
            X = X.tocsr()
            X.sort_indices()
            n, d = X.shape
            h = rs_create_csr(n, d, X.indptr.astype(np.int64), X.indices.astype(np.int32),
                              X.data.astype(np.float64), np.asarray(y, dtype=np.float64),
                              self.alpha, self.route, self.as_mode)
        else:
            n, d = X.shape
            h = rs_create_dense(X, y, self.alpha, self.route, self.as_mode)
        try:
            w, rep = rs_solve(h, self.solver, self.sketch_size, self.gamma, self.beta, self.tol,
                              self.max_iter, self.seed, self.subcount_k, d=d,
                              momentum=self.momentum, eta=self.eta)
        finally:
            rs_destroy(h)
        self.coef_, self.report_ = w, rep
        return self
