python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "explicit or config5" 2>&1 | tail -2
timeout 600 python bench.py --mode explicit --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_explicit.json 2>/dev/null
timeout 1200 python bench.py --config c5 --mode explicit --steps 148 --max-iter-tol 2000 > gpurun_out/bench_c5_explicit.json 2> gpurun_out/c5.err; tail -2 gpurun_out/c5.err
for f in c2_explicit c5_explicit; do python -c "import json; d=json.load(open('gpurun_out/bench_$f.json')); print('$f', round(d['value'],1), 'setup_s', d['setup_s'], 'tol', d['time_to_tol_s'], d['iterations_to_tol'])"; done
