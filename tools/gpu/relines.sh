python -c "import __graft_entry__ as g; g.build()" || exit 1
B="timeout 1200 python bench.py"
$B --mode explicit --no-cpu-baseline > gpurun_out/bench_c2_explicit.json 2>/dev/null
$B --config c4 --mode explicit --max-iter-tol 20000 --no-cpu-baseline > gpurun_out/bench_c4_explicit.json 2>/dev/null
$B --config c4 --max-iter-tol 20000 --cpu-seconds 20 > gpurun_out/bench_c4.json 2>/dev/null
$B --config c4 --max-iter-tol 20000 --no-cpu-baseline --no-e2e --momentum theory > gpurun_out/bench_c4_theory.json 2>/dev/null
$B --config c5 --mode explicit --max-iter-tol 2000 > gpurun_out/bench_c5_explicit.json 2>/dev/null
$B --config k1 --max-iter-tol 2000 --no-cpu-baseline > gpurun_out/bench_k1.json 2>/dev/null
