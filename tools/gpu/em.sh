NBS=2 bash tools/gpu/bfp.sh
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "tau1024 and (explicit or overlapped)" 2>&1 | tail -3 > gpurun_out/em_pytest.log
timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline --seeds 5 > gpurun_out/em_c5.json 2>/dev/null
timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline --config k1 --max-iter-tol 2000 --seeds 1 > gpurun_out/em_k1.json 2>/dev/null
python tools/showbench.py gpurun_out/em_*.json > gpurun_out/em_summary.txt 2>&1
