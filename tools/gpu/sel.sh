# k_sel_emit rewrite (4 entries per lane, aggregated append, 4-warp blocks): dual CSR parity tests,
# c4 GRAM bench, ncu durations of the selected-row kernels
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x -k "csr or config4 or c4" 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
for r in 1 2; do timeout 900 python bench.py --config c4 --no-cpu-baseline --no-e2e > gpurun_out/sel_c4_$r.json 2>/dev/null; done
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $M -k regex:"k_gram_bands|k_sel_|k_spmv" -c 12 --log-file gpurun_out/tr_c4_sel.csv python tools/prof_step.py c4 gram 4 > /dev/null 2>&1
