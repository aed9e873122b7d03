python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "csr" 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
B="timeout 1200 python bench.py --no-cpu-baseline --no-e2e"
$B --config c3 --steps 148 --max-iter-tol 3000 > gpurun_out/bench_c3.json 2>/dev/null
$B --config c4 --max-iter-tol 3000 > gpurun_out/bench_c4.json 2>/dev/null
