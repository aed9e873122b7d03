python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x -k "csr or c3 or c4 or config3 or config4 or momentum" 2>&1 | tail -1 | tee gpurun_out/pytest_gpu.log
M="--metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 ncu $M -k regex:"k_sel_|k_gram_bands" -c 12 --log-file gpurun_out/xx_c4.csv python tools/prof_step.py c4 gram 4 > /dev/null 2>&1
B="timeout 900 python bench.py"
$B --config c4 --max-iter-tol 20000 --cpu-seconds 20 > gpurun_out/f4_c4.json 2>/dev/null
$B --config c4 --max-iter-tol 20000 --no-cpu-baseline --no-e2e --momentum theory > gpurun_out/f4_c4_theory.json 2>/dev/null
