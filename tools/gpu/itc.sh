# phase C rewrite of k_iterate: parity subset, c5 at OV_SMS 22 / 32, c4 and k1 explicit lines
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "${PYK:-tau1024 or large_tau or overlapped or kernel_ridge or explicit or multirank}" 2>&1 | tail -2 | tee gpurun_out/itc_pytest.log
B="timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline"
$B --config c4 --max-iter-tol 20000 --seeds 1 > gpurun_out/itc_c4.json 2>/dev/null
$B --config k1 --max-iter-tol 2000 --seeds 1 > gpurun_out/itc_k1.json 2>/dev/null
$B --config c2 --mode explicit --seeds 1 > gpurun_out/itc_c2.json 2>/dev/null
for f in c4 k1 c2; do python -c "
import json;d=json.loads(open('gpurun_out/itc_$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value']), d['time_to_tol_s'], {k: round(v*1e3,2) for k, v in d['kernel_ms_per_step'].items() if v})"; done | tee gpurun_out/itc.txt
SWEEP="${SWEEP:-32 22 18}" bash tools/gpu/ov_sweep.sh
