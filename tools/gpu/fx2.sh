python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x -k "csr_primal or c3 or config3" 2>&1 | grep -E "^E  |passed|failed|FAILED|Error" | head -20 | tee gpurun_out/pytest_gpu.log
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e"
$B --config c3 --steps 300 --max-iter-tol 300 > gpurun_out/fx2_c3.json 2>/dev/null
