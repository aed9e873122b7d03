# CSR GRAM mode: parity tests + c3/c4 probes
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "csr" 2>&1 | tail -25 | tee gpurun_out/pytest_csr.log
for c in c3 c4; do
  RS_VERBOSE=1 timeout 600 python bench.py --config $c --mode gram --steps 20 --warmup 3 --max-iter-tol ${TOLITER:-3000} --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_gram.json 2> gpurun_out/bench_${c}_gram.err; tail -5 gpurun_out/bench_${c}_gram.err
done
