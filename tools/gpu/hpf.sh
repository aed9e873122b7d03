# k_hash_rows next-row prefetch (count sketch): CSR parity tests, c3 A/B, ncu durations
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x -k "csr or c3 or config3" 2>&1 | tail -2 | tee gpurun_out/pytest_gpu.log
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 300 --max-iter-tol 300 --config c3"
for r in 1 2; do
  $B > gpurun_out/hpf_c3_on_$r.json 2>/dev/null
  RS_HR_NOPF=1 $B > gpurun_out/hpf_c3_off_$r.json 2>/dev/null
done
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
timeout 900 ncu $M -k regex:"k_gram_bands|k_hash_rows|k_spmv" -c 12 --log-file gpurun_out/tr_c3.csv python tools/prof_step.py c3 gram 4 > /dev/null 2>&1
