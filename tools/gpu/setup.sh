python -c "import __graft_entry__ as g; g.build()" || exit 1
RS_VERBOSE=1 python tools/probe_setup.py c2 2>&1 | grep -v gemm
RS_A_BUILD_CPASYNC=1 python tools/probe_setup.py c2
timeout 600 python -m pytest tests -m gpu -x -q -k "explicit or kernel" 2>&1 | tail -1
timeout 900 python bench.py --config c5 --mode explicit --steps 148 --max-iter-tol 2000 --no-e2e > gpurun_out/bench_c5_explicit.json 2>/dev/null
timeout 900 python bench.py --config k1 --steps 148 --max-iter-tol 2000 --no-cpu-baseline --no-e2e > gpurun_out/bench_k1.json 2>/dev/null
