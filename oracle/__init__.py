"""Plain, slow, float64 CPU oracle for momentum sketch-and-project (RidgeSketch, arXiv 2105.05565).

TEST INFRASTRUCTURE ONLY. Nothing in the product path (``paper_2105_05565_b200``) may import,
call or link anything under ``oracle/``; only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may use it.  The oracle shares no
code with the CUDA path: it has its own Philox4x32-10, its own sketch construction, and
follows the paper's algorithms step by step with NumPy/SciPy library primitives
(matmul, Cholesky) as the only building blocks.

Citations: ``P:Lnnn`` is /root/reference/PAPER.md line nnn (section / equation in the text);
``S:Lnnn`` is SPEC.md line nnn.

Modules
-------
philox   Philox4x32-10 counter-based RNG (the sketch stream's generator).
sketch   Subsample, Count and SubCount sketches
         drawn from the seeded sketch-stream contract, plus materialisation of S.
problem  Primal / dual linear system A w = b and the direct Cholesky solve.
solver   Alg. 1 and Alg. 2, literal.

Parity status: every function is pinned by a ``-m "not gpu"`` test in tests/test_oracle_*.py
except the *design* of the sketch stream (which counter/stream/bit feeds which decision), which
the paper does not fix: "parity unpinned" for that design choice; its statistical properties
(uniformity, exact structure) are pinned instead.  See DESIGN.md §4.
"""

from . import philox, sketch, problem, solver  # noqa: F401
