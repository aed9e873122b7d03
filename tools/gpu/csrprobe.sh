set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in c3 c4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --max-iter-tol 2000 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -5 gpurun_out/bench_$c.err
done
