# Verification call: build, GPU suite, smoke, default bench line (c5) and the c4 / k1 EXPLICIT lines
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -6 | tee gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
B="timeout 1200 python bench.py"
$B > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
$B --config c4 --max-iter-tol 20000 --no-cpu-baseline > gpurun_out/bench_c4_explicit.json 2>/dev/null
$B --config k1 --max-iter-tol 2000 --no-cpu-baseline --seeds 1 > gpurun_out/bench_k1.json 2>/dev/null
ls gpurun_out/
