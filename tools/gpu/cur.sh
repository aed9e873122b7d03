python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x -k "csr or c3 or config3" 2>&1 | tail -1 | tee gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline --no-e2e --config c3 --max-iter-tol 300 > gpurun_out/cur_c3.json 2>/dev/null
