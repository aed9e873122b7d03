# fixed-point CSR Gram bands: CSR parity tests, c3 / c4 benches, ncu durations
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x -k "csr or c3 or c4 or config3 or config4 or momentum" 2>&1 | grep -E "^E  |passed|failed|FAILED|Error" | head -20 | tee gpurun_out/pytest_gpu.log
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e"
$B --config c3 --steps 300 --max-iter-tol 300 > gpurun_out/fx_c3.json 2>/dev/null
$B --config c4 > gpurun_out/fx_c4.json 2>/dev/null
$B --config c3 --momentum theory > gpurun_out/fx_c3_theory.json 2>/dev/null
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $M -k regex:"k_gram_bands|k_hash_rows|k_spmv" -c 12 --log-file gpurun_out/tr_c3.csv python tools/prof_step.py c3 gram 4 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_gram_bands|k_sel_|k_spmv" -c 12 --log-file gpurun_out/tr_c4.csv python tools/prof_step.py c4 gram 4 > /dev/null 2>&1
