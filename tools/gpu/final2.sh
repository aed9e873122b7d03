# end-of-round check after the CSR Gram changes: full GPU suite, smoke, default line, CSR lines,
# DRAM traffic of the CSR kernels
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.log
B="timeout 1200 python bench.py"
$B > gpurun_out/f2_c2_gram.json 2> gpurun_out/f2_c2_gram.err
for c in c3 c4; do $B --config $c --max-iter-tol 20000 --cpu-seconds 20 > gpurun_out/f2_$c.json 2>/dev/null; done
for c in c3 c4; do $B --config $c --max-iter-tol 20000 --no-cpu-baseline --no-e2e --momentum theory > gpurun_out/f2_${c}_theory.json 2>/dev/null; done
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
P="python tools/prof_step.py"
for c in c3 c4; do timeout 900 ncu $M -k regex:"k_gram_bands|k_hash_rows|k_sel_|k_spmv" -c 12 --log-file gpurun_out/tr_$c.csv $P $c gram 4 > /dev/null 2>&1; done
