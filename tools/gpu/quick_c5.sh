# Quick c5 check: parity of the large-tau paths, then the default bench line without the slow legs.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "tau1024 or large_tau or kernel_ridge or process_switches or config5" 2>&1 | tail -3 > gpurun_out/quick_pytest.log
timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
cat gpurun_out/quick_pytest.log
