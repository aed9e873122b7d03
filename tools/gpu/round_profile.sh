# Round profile: full GPU suite + smoke, every bench line, the default command's ncu launch list,
# ncu DRAM traffic of each config's dominant kernels (prof_step: every captured launch is active),
# and one --set full capture of the default command's top kernels.
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
B="timeout 1200 python bench.py"
$B > gpurun_out/bench_c2_gram.json 2> gpurun_out/bench_c2_gram.err
$B --impl reference --steps 3 --warmup 1 > gpurun_out/bench_c2_reference.json 2>/dev/null
for m in explicit implicit; do $B --mode $m --no-cpu-baseline > gpurun_out/bench_c2_$m.json 2>/dev/null; done
for c in c3 c4; do $B --config $c --max-iter-tol 20000 --cpu-seconds 20 > gpurun_out/bench_$c.json 2>/dev/null; done
$B --config c4 --mode explicit --max-iter-tol 20000 --no-cpu-baseline > gpurun_out/bench_c4_explicit.json 2>/dev/null
for c in c2 c3 c4; do $B --config $c --max-iter-tol 20000 --no-cpu-baseline --no-e2e --momentum theory > gpurun_out/bench_${c}_theory.json 2>/dev/null; done
$B --config c5 --mode explicit --max-iter-tol 2000 > gpurun_out/bench_c5_explicit.json 2>/dev/null
$B --config k1 --max-iter-tol 2000 --no-cpu-baseline > gpurun_out/bench_k1.json 2>/dev/null
$B --config c5 --mode gram --steps 20 --max-iter-tol 400 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5_gram.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2_gram.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 10 > /dev/null 2>&1
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
P="python tools/prof_step.py"
timeout 900 ncu $M -k regex:"k_gram_xt" -c 4 --log-file gpurun_out/tr_c2_gram.csv $P c2 gram 8 > /dev/null 2>&1
RS_NO_XC=1 timeout 900 ncu $M -k regex:"k_xpass_rows" -c 4 --log-file gpurun_out/tr_c2_gram_xpass.csv $P c2 gram 8 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_spmv" -c 4 --log-file gpurun_out/tr_c4_spmv.csv $P c4 gram 4 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_tn_gemm" -c 4 --log-file gpurun_out/tr_c2_implicit.csv $P c2 implicit 4 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_update_rows|k_bfactor|k_apply_rows" -c 12 --log-file gpurun_out/tr_c2_explicit.csv $P c2 explicit 64 > /dev/null 2>&1
for c in c3 c4; do timeout 900 ncu $M -k regex:"k_gram_bands|k_hash_rows|k_sel_|k_spmv" -c 12 --log-file gpurun_out/tr_$c.csv $P $c gram 4 > /dev/null 2>&1; done
timeout 900 ncu $M -k regex:"k_update_rows|k_apply_rows" -c 8 --log-file gpurun_out/tr_c4_explicit.csv $P c4 explicit 16 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_bfactor|k_update_rows|k_apply_rows" -c 9 --log-file gpurun_out/tr_c5_explicit.csv $P c5 explicit 150 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_bfactor|k_update_rows|k_apply_rows" -c 9 --log-file gpurun_out/tr_k1.csv $P k1 explicit 150 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_xtw" -c 1 -o gpurun_out/prof_c2_gram_full $P c2 gram 8 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_xpass_rows" -c 1 -o gpurun_out/prof_c2_xpass_full $P c2 gram 8 > /dev/null 2>&1
ls gpurun_out/
