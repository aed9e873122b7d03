python -c "import __graft_entry__ as g; g.build()" || exit 1
for m in heuristic theory; do
timeout 900 python bench.py --config c3 --steps 148 --max-iter-tol 20000 --no-cpu-baseline --no-e2e --momentum $m > gpurun_out/bench_c3_$m.json 2>/dev/null
timeout 600 python bench.py --config c4 --steps 148 --max-iter-tol 20000 --no-cpu-baseline --no-e2e --momentum $m > gpurun_out/bench_c4_$m.json 2>/dev/null
timeout 600 python bench.py --config c2 --no-cpu-baseline --no-e2e --momentum $m > gpurun_out/bench_c2_$m.json 2>/dev/null
done
