# left-looking pair factor: GPU suite + c5 explicit / k1 / c3 (tau 500) bench lines, right-looking A/B
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --config c5 --mode explicit --steps 148 --max-iter-tol 2000 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_explicit.json 2>/dev/null

timeout 1200 python bench.py --config k1 --steps 148 --max-iter-tol 2000 --no-cpu-baseline --no-e2e > gpurun_out/bench_k1.json 2>/dev/null
timeout 900 python bench.py --config c4 --mode explicit --steps 148 --max-iter-tol 20000 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_explicit.json 2>/dev/null
