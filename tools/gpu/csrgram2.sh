set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "csr or large_tau" 2>&1 | tail -25 | tee gpurun_out/pytest_csr.log
timeout 300 python tools/probe_overhead.py c4 gram 2>&1 | tail -8
for c in c3 c4; do
  RS_VERBOSE=1 timeout 600 python bench.py --config $c --mode gram --steps 64 --warmup 3 --max-iter-tol ${TOLITER:-3000} --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_gram.json 2> gpurun_out/bench_${c}_gram.err; tail -5 gpurun_out/bench_${c}_gram.err
done
