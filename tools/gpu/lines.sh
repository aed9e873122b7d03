# The EXPLICIT bench lines (c5 default with every leg, c4, c4 THEORY, k1, c2 EXPLICIT) -> gpurun_out/fin_*.json
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="timeout 1200 python bench.py"
$B > gpurun_out/fin_c5.json 2> gpurun_out/fin_c5.err
RS_VERBOSE=1 $B --config c4 --max-iter-tol 20000 --cpu-seconds 20 > gpurun_out/fin_c4_explicit.json 2> gpurun_out/fin_c4.err
$B --config c4 --max-iter-tol 20000 --no-cpu-baseline --no-e2e --seeds 1 --momentum theory > gpurun_out/fin_c4_theory.json 2>/dev/null
$B --config k1 --max-iter-tol 2000 --no-cpu-baseline --seeds 1 > gpurun_out/fin_k1.json 2>/dev/null
$B --config c2 --mode explicit --no-cpu-baseline --no-alt > gpurun_out/fin_c2_explicit.json 2>/dev/null
grep "csr explicit" gpurun_out/fin_c4.err | head -3 > gpurun_out/fin_c4_plan.txt
