set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "dense or config1 or config2 or explicit or abi" 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py --mode explicit --no-cpu-baseline > gpurun_out/bench_c2_explicit.json 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_gram.json 2>/dev/null
