python -c "import __graft_entry__ as g; g.build()" || exit 1
B="timeout 1200 python bench.py --no-cpu-baseline --no-e2e"
$B > gpurun_out/chk_c2.json 2>/dev/null
$B --config c4 --max-iter-tol 3000 > gpurun_out/chk_c4.json 2>/dev/null
$B --config c4 --mode explicit --max-iter-tol 3000 > gpurun_out/chk_c4e.json 2>/dev/null
$B --mode explicit > gpurun_out/chk_c2e.json 2>/dev/null
$B --config c5 --mode explicit --max-iter-tol 2000 > gpurun_out/chk_c5e.json 2>/dev/null
