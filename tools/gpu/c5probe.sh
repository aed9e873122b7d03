set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -x -q -k "csr" 2>&1 | tail -3
RS_VERBOSE=1 timeout 600 python bench.py --config c3 --mode gram --steps 148 --warmup 3 --max-iter-tol 3000 --no-cpu-baseline --no-e2e > gpurun_out/bench_c3_gram.json 2> gpurun_out/bench_c3_gram.err; tail -2 gpurun_out/bench_c3_gram.err
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
for m in explicit gram; do
RS_VERBOSE=1 timeout 1200 python bench.py --config c5 --mode $m --steps 20 --warmup 3 --max-iter-tol 400 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_$m.json 2> gpurun_out/bench_c5_$m.err; tail -4 gpurun_out/bench_c5_$m.err
done
