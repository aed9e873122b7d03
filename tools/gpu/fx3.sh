python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x -k "csr or c3 or c4 or config3 or config4 or momentum" 2>&1 | grep -E "^E  |passed|failed|FAILED|Error" | head -20 | tee gpurun_out/pytest_gpu.log
B="timeout 900 python bench.py"
for c in c3 c4; do $B --config $c --max-iter-tol 20000 --cpu-seconds 20 > gpurun_out/f3_$c.json 2>/dev/null; done
$B --config c4 --max-iter-tol 20000 --no-cpu-baseline --no-e2e --momentum theory > gpurun_out/f3_c4_theory.json 2>/dev/null
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
P="python tools/prof_step.py"
for c in c3 c4; do timeout 900 ncu $M -k regex:"k_gram_bands|k_hash_rows|k_sel_|k_spmv" -c 12 --log-file gpurun_out/tr_$c.csv $P $c gram 4 > /dev/null 2>&1; done
