python -c "import __graft_entry__ as g; g.build()" || exit 1
for R in 1 2 4 8; do
  RS_XP_R=$R timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 50 --max-iter-tol 10 > gpurun_out/xp_R$R.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/xp_R$R.json')); print('R=$R', round(d['kernel_ms_per_step']['as'],4), 'ms', round(d['roofline']['frac'],3))"
done
