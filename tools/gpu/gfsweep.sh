python -c "import __graft_entry__ as g; g.build()" || exit 1
cp paper_2105_05565_b200/libridgesketch.so /tmp/lib_base.so
for v in base gf6 gf8; do
  if [ $v = base ]; then cp /tmp/lib_base.so paper_2105_05565_b200/libridgesketch.so; else cp tools/variants/lib_$v.so paper_2105_05565_b200/libridgesketch.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 64 --max-iter-tol 10 > gpurun_out/gf_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/gf_$v.json')); k=d['kernel_ms_per_step']; print('$v', round(d['ms_per_step'],4), 'gram', round(k['gram'],4), 'as', round(k['as'],4))"
done
cp /tmp/lib_base.so paper_2105_05565_b200/libridgesketch.so
