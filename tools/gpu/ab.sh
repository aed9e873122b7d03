# A build on the lower tiles with the split-K plan over the working tiles: full suite + c5 line
python -c "import __graft_entry__ as g; g.build()" || exit 1
RS_VERBOSE=1 timeout 300 python tools/probe_setup.py c5 2>&1 | grep -v "^\[rs\] gemm" | tail -6 > gpurun_out/ab_setup.txt
timeout 600 python bench.py --no-cpu-baseline --seeds 5 > gpurun_out/ab_c5.json 2>gpurun_out/ab_c5.err
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -4 > gpurun_out/ab_pytest.log
