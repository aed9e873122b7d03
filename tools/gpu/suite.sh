set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py --mode explicit --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_explicit.json 2>/dev/null
