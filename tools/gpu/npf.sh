# next-iteration L2 prefetch in k_update_rows: explicit parity tests, then A/B on the explicit benches
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x -k "explicit or kernel or config5 or switches" 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
B="timeout 900 python bench.py --no-cpu-baseline --no-e2e"
for r in 1 2; do
for v in on off; do
  if [ $v = off ]; then export RS_NO_NEXTPF=1; else unset RS_NO_NEXTPF; fi
  $B --config c5 --mode explicit --max-iter-tol 2000 > gpurun_out/npf_c5_${v}_$r.json 2>/dev/null
  $B --config k1 > gpurun_out/npf_k1_${v}_$r.json 2>/dev/null
  $B --config c4 --mode explicit --max-iter-tol 3000 > gpurun_out/npf_c4_${v}_$r.json 2>/dev/null
  $B --mode explicit > gpurun_out/npf_c2_${v}_$r.json 2>/dev/null
done; done
unset RS_NO_NEXTPF
