# staged light-row pair loop in k_gram_bands: CSR GRAM parity tests, then c3 / c4 A/B
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x -k "csr or c3 or config3 or config4" 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 300"
for r in 1 2; do
for v in on off; do
  if [ $v = off ]; then export RS_GB_NOSTAGE=1; else unset RS_GB_NOSTAGE; fi
  $B --config c3 --max-iter-tol 300 > gpurun_out/gbs_c3_${v}_$r.json 2>/dev/null
  $B --config c4 --max-iter-tol 300 > gpurun_out/gbs_c4_${v}_$r.json 2>/dev/null
done; done
unset RS_GB_NOSTAGE
