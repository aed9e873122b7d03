python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "kernel" 2>&1 | tail -15
timeout 900 python bench.py --config k1 --steps 148 --max-iter-tol 20000 --cpu-seconds 10 > gpurun_out/bench_k1.json 2> gpurun_out/bench_k1.err; tail -4 gpurun_out/bench_k1.err
