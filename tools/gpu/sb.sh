# Blocked-inverse check: parity subset, then the c5 / k1 lines at nb = 2 (default), 1, 3, 4
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 120 ./tools/ubench_ring 4096 1024 > gpurun_out/ubench_ring.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "${PYK:-tau1024 or blocked_inverse or kernel or explicit}" 2>&1 | tail -5 | tee gpurun_out/sb_pytest.log
B="timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline"
for nb in ${NBS:-2 1 3 4}; do
  RS_SB_NB=$nb $B --seeds 5 > gpurun_out/sb_c5_$nb.json 2>gpurun_out/sb_c5_$nb.err
  RS_SB_NB=$nb $B --config k1 --max-iter-tol 2000 --seeds 1 > gpurun_out/sb_k1_$nb.json 2>/dev/null
done
python tools/showbench.py gpurun_out/sb_*.json 2>&1 | tee gpurun_out/sb_summary.txt
