set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
for m in gram implicit explicit; do
  timeout 300 python bench.py --steps 50 --warmup 5 --mode $m --no-cpu-baseline > gpurun_out/bench_$m.json 2> gpurun_out/bench_$m.err; tail -3 gpurun_out/bench_$m.err
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
