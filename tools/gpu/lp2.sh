set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x -k "large_tau or config5 or kernel or switches or csr_explicit or c3 or csr_primal" 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
B="timeout 1200 python bench.py --no-cpu-baseline --no-e2e"
$B --config c5 --mode explicit --steps 148 --max-iter-tol 2000 > gpurun_out/bench_c5_explicit.json 2>/dev/null
$B --config k1 --steps 148 --max-iter-tol 2000 > gpurun_out/bench_k1.json 2>/dev/null
