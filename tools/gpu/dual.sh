# Two-slots-per-SM factorisation (k_bfactor_lp<4>) in the overlapped pipeline, with the first set's
# tail factored beside the first group: large-tau parity subset, then the OV_SMS sweep of the c5
# line and the 8-warp reference (RS_BF_DUAL=0)
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "${PYK:-tau1024 or large_tau or overlapped or kernel_ridge or explicit}" 2>&1 | tail -4 | tee gpurun_out/dual_pytest.log
RS_BF_DUAL=0 timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline --seeds 2 > gpurun_out/dual0_c5.json 2>/dev/null
python tools/showbench.py gpurun_out/dual0_c5.json > gpurun_out/dual0.txt
SWEEP="${SWEEP:-22 32 34 38}" bash tools/gpu/ov_sweep.sh
