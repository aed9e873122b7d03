set -x
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "explicit or kernel or switches" 2>&1 | grep -E "^E  .*Error|passed|failed|FAILED" | head | tee gpurun_out/pytest_gpu.log
B="timeout 1200 python bench.py --no-cpu-baseline --no-e2e"
for b in 4 8 16 32; do RS_UR_BPS=$b $B --config c4 --mode explicit --steps 296 --max-iter-tol 2000 > gpurun_out/ur_c4_$b.json 2>/dev/null; done
for b in 4 16; do RS_UR_BPS=$b $B --config c5 --mode explicit --steps 296 --max-iter-tol 2000 > gpurun_out/ur_c5_$b.json 2>/dev/null; done
for b in 4 16; do RS_UR_BPS=$b $B --mode explicit > gpurun_out/ur_c2_$b.json 2>/dev/null; done
