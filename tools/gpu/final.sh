# final check of the round: full GPU suite, smoke, the default bench line and the c4 lines (the
# selected-row emit changed)
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
B="timeout 1200 python bench.py"
$B > gpurun_out/fin_c2_gram.json 2> gpurun_out/fin_c2_gram.err
$B --config c4 --max-iter-tol 20000 --cpu-seconds 20 > gpurun_out/fin_c4.json 2>/dev/null
$B --config c4 --max-iter-tol 20000 --no-cpu-baseline --no-e2e --momentum theory > gpurun_out/fin_c4_theory.json 2>/dev/null
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $M -k regex:"k_gram_bands|k_hash_rows|k_sel_|k_spmv" -c 12 --log-file gpurun_out/tr_c4.csv python tools/prof_step.py c4 gram 4 > /dev/null 2>&1
