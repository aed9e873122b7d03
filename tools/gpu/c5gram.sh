set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x -k "gram or large_tau or fused or switches" 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
RS_VERBOSE=1 timeout 1500 python bench.py --config c5 --mode gram --steps 20 --warmup 3 --max-iter-tol 400 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_gram.json 2> gpurun_out/bench_c5_gram.err
