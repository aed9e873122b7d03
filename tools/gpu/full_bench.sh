# full GPU test suite + bench lines for every mode (c2) and the CSR configs
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 | tee gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for m in gram explicit implicit; do
  timeout 600 python bench.py --mode $m > gpurun_out/bench_c2_$m.json 2> gpurun_out/bench_c2_$m.err; tail -2 gpurun_out/bench_c2_$m.err
done
for c in ${CSR_CONFIGS:-}; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --max-iter-tol ${TOLITER:-3000} --cpu-seconds 20 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err
done
