# usage: bash tools/gpu/quick.sh "<pytest -k expr or empty>" "<bench modes>" [steps]
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
if [ -n "$1" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$1" 2>&1 | tail -25 | tee gpurun_out/pytest_quick.log; fi
for m in $2; do
  timeout 300 python bench.py --steps ${3:-50} --warmup 5 --mode $m --no-cpu-baseline --no-e2e > gpurun_out/bench_$m.json 2> gpurun_out/bench_$m.err; tail -3 gpurun_out/bench_$m.err
done
