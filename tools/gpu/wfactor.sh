# W = L^{-1} factor slots (tau > 224): full GPU suite + c5 explicit / k1 / c3 bench lines
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --config c5 --mode explicit --steps 148 --max-iter-tol 2000 --no-cpu-baseline > gpurun_out/bench_c5_explicit.json 2>gpurun_out/bench_c5_explicit.err
timeout 1200 python bench.py --config k1 --steps 148 --max-iter-tol 2000 --no-cpu-baseline > gpurun_out/bench_k1.json 2>/dev/null
timeout 900 python bench.py --config c3 --steps 148 --max-iter-tol 3000 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3.json 2>/dev/null
