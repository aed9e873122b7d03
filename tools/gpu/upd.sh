python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "explicit or kernel or config1 or momentum or large_tau" 2>&1 | tail -2
timeout 600 python bench.py --mode explicit --no-cpu-baseline > gpurun_out/bench_c2_explicit.json 2>/dev/null
timeout 900 python bench.py --config c5 --mode explicit --steps 148 --max-iter-tol 2000 > gpurun_out/bench_c5_explicit.json 2>/dev/null
timeout 900 python bench.py --config k1 --steps 148 --max-iter-tol 2000 --no-cpu-baseline > gpurun_out/bench_k1.json 2>/dev/null
