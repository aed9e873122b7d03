# Quick check: explicit / dual / multi-rank / tau = 1024 parity subset, then the OV_SMS sweep of
# the c5 line (bench without the slow legs)
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "${PYK:-explicit or dual or multirank or tau1024 or kernel or config1 or ragged or xs}" 2>&1 | tail -4 | tee gpurun_out/quick_pytest.log
SWEEP="${SWEEP:-22 26 30}" bash tools/gpu/ov_sweep.sh
