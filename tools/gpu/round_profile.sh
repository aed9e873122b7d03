# full GPU suite, bench lines for every config, ncu DRAM traffic of each dominant kernel
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 | tee gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
timeout 600 python bench.py > gpurun_out/bench_c2_gram.json 2> gpurun_out/bench_c2_gram.err; tail -2 gpurun_out/bench_c2_gram.err
for m in explicit implicit; do timeout 600 python bench.py --mode $m --no-cpu-baseline > gpurun_out/bench_c2_$m.json 2> gpurun_out/bench_c2_$m.err; tail -2 gpurun_out/bench_c2_$m.err; done
for c in c3 c4; do timeout 900 python bench.py --config $c --steps 148 --max-iter-tol 20000 --cpu-seconds 20 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -2 gpurun_out/bench_$c.err; done
timeout 1200 python bench.py --config c5 --mode explicit --steps 148 --max-iter-tol 2000 > gpurun_out/bench_c5_explicit.json 2> gpurun_out/bench_c5_explicit.err; tail -2 gpurun_out/bench_c5_explicit.err
# ncu: launch list of the default command and DRAM bytes of the dominant kernels
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_gram.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 10 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_xpass|k_gram_fused" -c 12 --log-file gpurun_out/tr_c2_gram.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 3 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_tn_gemm" -c 6 --log-file gpurun_out/tr_c2_implicit.csv python bench.py --mode implicit --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 3 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_update|k_bfactor" -c 12 --log-file gpurun_out/tr_c2_explicit.csv python bench.py --mode explicit --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 3 > /dev/null 2>&1
for c in c3 c4; do timeout 900 ncu $M -k regex:"k_gram_bands|k_hash_rows|k_spmv|k_bfactor" -c 16 --log-file gpurun_out/tr_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 3 > /dev/null 2>&1; done
timeout 900 ncu $M -k regex:"k_bfactor|k_update" -c 8 --log-file gpurun_out/tr_c5_explicit.csv python bench.py --config c5 --mode explicit --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 3 > /dev/null 2>&1
ls -la gpurun_out/
