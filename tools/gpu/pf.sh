set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x -k "explicit or kernel or config5 or switches or dirty" 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
B="timeout 1200 python bench.py --no-cpu-baseline --no-e2e"
$B --config c5 --mode explicit --steps 148 --max-iter-tol 2000 > gpurun_out/bench_c5_explicit.json 2>/dev/null
RS_NO_L2PF=1 $B --config c5 --mode explicit --steps 148 --max-iter-tol 2000 > gpurun_out/bench_c5_explicit_nopf.json 2>/dev/null
$B --config c4 --mode explicit --steps 148 --max-iter-tol 20000 > gpurun_out/bench_c4_explicit.json 2>/dev/null
$B --config c4 --steps 148 --max-iter-tol 20000 > gpurun_out/bench_c4.json 2>/dev/null
$B --mode explicit > gpurun_out/bench_c2_explicit.json 2>/dev/null
$B > gpurun_out/bench_c2_gram.json 2>/dev/null
