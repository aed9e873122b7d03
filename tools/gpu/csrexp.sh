python -c "import __graft_entry__ as g; g.build()" || exit 1
RS_VERBOSE=1 timeout 900 python -m pytest tests -m gpu -x -q -k "csr_explicit" 2>&1 | grep -E "^E  |passed|failed|heavy" | head -20
RS_VERBOSE=1 timeout 900 python bench.py --config c4 --mode explicit --steps 148 --max-iter-tol 20000 --cpu-seconds 10 > gpurun_out/bench_c4_explicit.json 2> gpurun_out/c4e.err; grep -E "heavy|Error" gpurun_out/c4e.err | head -3
