python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -x -q -k "fused" 2>&1 | tail -2
RS_XG=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_xg.json 2> gpurun_out/bench_c2_xg.err; tail -3 gpurun_out/bench_c2_xg.err
RS_XG=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_xpass_gram1" -s 2 -c 1 -o gpurun_out/ncu_xg1 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 4 > /dev/null 2>&1
