# Full GPU suite (per-test timeout) + default bench line (no slow legs)
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1700 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 2>&1 | tail -25 > gpurun_out/full_pytest.log
timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
cat gpurun_out/full_pytest.log
