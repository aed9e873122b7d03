# streamed-build test, the default bench line (all legs), its ncu launch list, compute-sanitizer
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -k "streamed or overlapped or tau1024" 2>&1 | tail -3 > gpurun_out/r2a_pytest.log
timeout 900 python bench.py > gpurun_out/r02_bench_c5.json 2> gpurun_out/r02_bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches_c5.csv python bench.py --steps 300 --warmup 3 --no-alt --no-e2e --no-cpu-baseline --seeds 1 > /dev/null 2>&1
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_small.py > gpurun_out/r02_sanitize_$t.txt 2>&1
  echo "$t rc=$?" >> gpurun_out/r02_sanitize_rc.txt
done
cat gpurun_out/r2a_pytest.log gpurun_out/r02_sanitize_rc.txt
