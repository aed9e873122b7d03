python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_gram.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 10 > /dev/null 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 10 > gpurun_out/bench_c2_short.json 2>/dev/null
