set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "csr or large_tau or sketch_ahead" 2>&1 | tail -5 | tee gpurun_out/pytest_csr.log
for c in c3 c4; do
  RS_VERBOSE=1 timeout 600 python bench.py --config $c --mode gram --steps 148 --warmup 3 --max-iter-tol ${TOLITER:-3000} --no-cpu-baseline --no-e2e > gpurun_out/bench_${c}_gram.json 2> gpurun_out/bench_${c}_gram.err; tail -3 gpurun_out/bench_${c}_gram.err
done
for c in c3 c4; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gram_bands|k_hash_rows|k_spmv|k_bfactor_big" -c 8 -o gpurun_out/ncu_${c}_gram python bench.py --config $c --mode gram --steps 3 --warmup 3 --max-iter-tol 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${c}.log 2>&1; tail -1 gpurun_out/ncu_${c}.log
done
