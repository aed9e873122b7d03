# row-owner X pass: full GPU suite + c2 GRAM bench (on / off)
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_gram.json 2>/dev/null
RS_NO_XPASS_ROWS=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_gram_old.json 2>/dev/null
for R in 1 2 4; do RS_XP_R=$R timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 50 --max-iter-tol 10 > gpurun_out/xr_R$R.json 2>/dev/null; done
