"""The library's multi-rank path (rs_dist with world > 1) executed on
the GPU, each rank a separate process:

* world 2 with the host-staged collective (RS_COLL_HOST): both ranks share one GPU -- no kernel
  waits on another rank -- so this runs on a single-GPU box.  It executes every world > 1 branch
  of the engine: row shards (dense, nnz-balanced CSR), feature shards (CSR dual, nnz-balanced), the
  allreduce of A S / u / the group Grams / b / A inside the captured graphs, the dual weight
  assembly.  The ranks' iterates must agree bit for bit (the collective sums in rank order and every
  replicated kernel sees the same inputs), and equal the oracle's within 1e-10 (R18/R27).
* world 2 with NCCL (torchrun-style, one GPU per rank): skipped below 2 GPUs."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from multirank_cases import CASES
from oracle import solver as OV
from parity_util import assert_close

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def built():
    from paper_2105_05565_b200 import build
    build()
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"


def _run_world(tmp_path, world, coll, cases):
    port = _free_port()
    env = dict(os.environ)
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "multirank_worker.py"), str(r),
                               str(world), str(port), coll, str(tmp_path)] + cases,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, env=env)
             for r in range(world)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=900)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out)
    for p, out in zip(procs, outs):
        assert p.returncode == 0, out[-3000:]


def _reference(name):
    import rsinputs
    c = CASES[name]
    if c["data"] == "dense":
        X, y = rsinputs.dense_problem(c["n"], c["d"], seed=c["seed"], col_decay=True, noise=0.01)
        X, y = X.numpy(), y.numpy()
    else:
        rp, ci, v, y = c["make"]()
        X = rsinputs.csr_to_scipy(rp, ci, v, c["n"], c["d"])
    return OV.solve(X, y, c["lam"], c["kind"], c["tau"], 1.0, 0.5, 0.0, c["iters"], seed=c["sseed"],
                    subcount_k=c.get("k", 0))


@pytest.mark.parametrize("world", [2, 3])
def test_host_collective_world(built, tmp_path, world):
    names = list(CASES) if world == 2 else ["dense_gram", "csr_dual_gram", "dense_explicit_big"]
    _run_world(tmp_path, world, "host", names)
    for name in names:
        got = [np.load(tmp_path / f"{name}.rank{r}.npz") for r in range(world)]
        for r in range(1, world):   # replicated state: bit-identical on every rank
            for key in ("w", "ws", "r"):
                assert np.array_equal(got[0][key], got[r][key]), (name, key, r)
        ref = _reference(name)
        assert int(got[0]["iterations"]) == CASES[name]["iters"]
        assert_close(got[0]["ws"], ref["w"], 1e-10, f"{name} system iterate")
        assert_close(got[0]["r"], ref["r"], 1e-10, f"{name} residual")
        assert_close(got[0]["w"], ref["weights"], 1e-10, f"{name} weights")


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="NCCL world 2 needs two GPUs")
def test_nccl_world2(built, tmp_path):
    names = ["dense_gram", "dense_implicit", "csr_primal_gram", "csr_dual_gram"]
    _run_world(tmp_path, 2, "nccl", names)
    for name in names:
        got = [np.load(tmp_path / f"{name}.rank{r}.npz") for r in range(2)]
        for key in ("w", "ws", "r"):
            assert np.array_equal(got[0][key], got[1][key]), (name, key)
        ref = _reference(name)
        assert_close(got[0]["ws"], ref["w"], 1e-10, f"{name} system iterate")
        assert_close(got[0]["r"], ref["r"], 1e-10, f"{name} residual")
