set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x -k "gram or fused or config2 or switches or config1" 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_gram.json 2>/dev/null
RS_GX_SYNC=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_gram_sync.json 2>/dev/null
