# full GPU suite, bench lines for every config, ncu DRAM traffic of each dominant kernel
set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv"
timeout 600 python bench.py > gpurun_out/bench_c2_gram.json 2> gpurun_out/bench_c2_gram.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_c2_reference.json 2>/dev/null
for m in explicit implicit; do timeout 600 python bench.py --mode $m --no-cpu-baseline > gpurun_out/bench_c2_$m.json 2>/dev/null; done
for c in c3 c4; do timeout 900 python bench.py --config $c --steps 148 --max-iter-tol 20000 --cpu-seconds 20 > gpurun_out/bench_$c.json 2>/dev/null; done
for c in c2 c3 c4; do timeout 900 python bench.py --config $c --steps 148 --max-iter-tol 20000 --no-cpu-baseline --no-e2e --momentum theory > gpurun_out/bench_${c}_theory.json 2>/dev/null; done
timeout 1200 python bench.py --config c5 --mode explicit --steps 148 --max-iter-tol 2000 > gpurun_out/bench_c5_explicit.json 2>/dev/null
timeout 1200 python bench.py --config k1 --steps 148 --max-iter-tol 2000 --no-cpu-baseline > gpurun_out/bench_k1.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_gram.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 10 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_xpass_tma|k_gram_fused" -c 12 --log-file gpurun_out/tr_c2_gram.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 3 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_tn_gemm" -c 6 --log-file gpurun_out/tr_c2_implicit.csv python bench.py --mode implicit --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 3 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_update_rows|k_bfactor" -c 12 --log-file gpurun_out/tr_c2_explicit.csv python bench.py --mode explicit --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 3 > /dev/null 2>&1
for c in c3 c4; do timeout 900 ncu $M -k regex:"k_gram_bands|k_hash_rows|k_spmv|k_bfactor" -c 16 --log-file gpurun_out/tr_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 3 > /dev/null 2>&1; done
timeout 900 ncu $M -k regex:"k_bfactor|k_update_rows" -c 8 --log-file gpurun_out/tr_c5_explicit.csv python bench.py --config c5 --mode explicit --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 3 > /dev/null 2>&1
timeout 900 ncu $M -k regex:"k_bfactor|k_update_rows" -c 8 --log-file gpurun_out/tr_k1.csv python bench.py --config k1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --max-iter-tol 3 > /dev/null 2>&1
ls gpurun_out/
