# concurrent Gram / X-pass groups: GPU suite + c2 GRAM bench (xc on/off) + X-pass traffic captures
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_c2_gram_xc.json 2>gpurun_out/bench_c2_gram_xc.err
RS_NO_XC=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_gram_seq.json 2>/dev/null
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
RS_NO_XC=1 timeout 900 ncu $M -k regex:"k_xpass_rows" -c 4 --log-file gpurun_out/tr_c2_gram_xpass.csv python tools/prof_step.py c2 gram 8 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_xpass_rows|k_gram_xt" -c 8 --log-file gpurun_out/tr_c2_gram_xc.csv python tools/prof_step.py c2 gram 64 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_spmv" -c 4 --log-file gpurun_out/tr_c4_spmv.csv python tools/prof_step.py c4 gram 4 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2_gram_xc.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 10 > /dev/null 2>&1
