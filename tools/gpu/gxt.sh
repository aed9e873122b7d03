# Gram from X^T: GPU tests + c2 GRAM bench BK 32 / 16
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_gram.json 2>/dev/null
RS_GX_BK=16 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_gram16.json 2>/dev/null
CFG=c2 MODE=gram ITERS=64 KREGEX="k_gram_xt" COUNT=2 bash tools/gpu/ncu_step.sh > gpurun_out/ncu_c2g.log 2>&1
