# Round profile (round 2, final): full GPU suite + smoke, every bench line, the default command's ncu launch
# list, ncu DRAM traffic of the dominant kernels, and --set full captures of the c5 step's kernels.
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 2>&1 | tail -4 | tee gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
B="timeout 1200 python bench.py"
$B > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
$B --impl reference --steps 20 --warmup 3 > gpurun_out/bench_c5_reference.json 2>/dev/null
$B --config c2 > gpurun_out/bench_c2_gram.json 2>/dev/null
$B --config c2 --mode explicit --no-cpu-baseline --no-alt > gpurun_out/bench_c2_explicit.json 2>/dev/null
$B --config c2 --mode implicit --no-cpu-baseline --no-alt --steps 50 --seeds 1 > gpurun_out/bench_c2_implicit.json 2>/dev/null
RS_OV_SPLIT=0 $B --no-cpu-baseline --no-alt --no-e2e > gpurun_out/bench_c5_nosplit.json 2>/dev/null
RS_SB_NB=1 $B --no-cpu-baseline --no-alt --no-e2e > gpurun_out/bench_c5_nb1.json 2>/dev/null
$B --config c3 --max-iter-tol 20000 --cpu-seconds 20 --seeds 1 > gpurun_out/bench_c3.json 2>/dev/null
$B --config c4 --max-iter-tol 20000 --cpu-seconds 20 > gpurun_out/bench_c4_explicit.json 2>/dev/null
$B --config c4 --mode gram --max-iter-tol 20000 --no-cpu-baseline --seeds 1 > gpurun_out/bench_c4_gram.json 2>/dev/null
$B --config k1 --max-iter-tol 2000 --no-cpu-baseline --seeds 1 > gpurun_out/bench_k1.json 2>/dev/null
for c in c3 c4; do $B --config $c --max-iter-tol 20000 --no-cpu-baseline --no-e2e --seeds 1 --momentum theory > gpurun_out/bench_${c}_theory.json 2>/dev/null; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 300 --warmup 3 --no-alt --no-e2e --no-cpu-baseline --seeds 1 > /dev/null 2>&1
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
P="python tools/prof_step.py"
timeout 900 ncu $M -k regex:"k_bfactor_lp|k_bf_gather|k_iterate" -c 9 --log-file gpurun_out/tr_c5_explicit.csv $P c5 explicit 400 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_bfactor_lp|k_bf_gather|k_iterate" -c 6 --log-file gpurun_out/tr_k1.csv $P k1 explicit 300 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_iterate|k_bfactor_small" -c 6 --log-file gpurun_out/tr_c4_explicit.csv $P c4 explicit 300 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_gram_xtw|k_xpass_rows" -c 6 --log-file gpurun_out/tr_c2_gram.csv $P c2 gram 8 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_gram_bands|k_hash_rows|k_spmv" -c 12 --log-file gpurun_out/tr_c3.csv $P c3 gram 4 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_dense_xs" -c 4 --log-file gpurun_out/tr_xs_c2.csv $P c2 implicit 4 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_dense_xs" -c 2 --log-file gpurun_out/tr_xs_c5.csv $P c5 gram 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"bfactor_lp<.int.4" -c 1 -o gpurun_out/prof_c5_bfactor_full $P c5 explicit 300 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_iterate" -c 1 -o gpurun_out/prof_c5_iterate_full $P c5 explicit 300 > /dev/null 2>&1
ls gpurun_out/
