# development check: build, a pytest subset (PYK), the c5 line and the c4 / k1 EXPLICIT lines
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 -k "${PYK:-tau1024 or large_tau or overlapped or kernel_ridge or explicit or multirank or abi}" 2>&1 | tail -4 | tee gpurun_out/check_pytest.log
B="timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline"
$B --seeds 3 > gpurun_out/check_c5.json 2>/dev/null
$B --config k1 --max-iter-tol 2000 --seeds 1 > gpurun_out/check_k1.json 2>/dev/null
for f in c5 k1; do python -c "
import json;d=json.loads(open('gpurun_out/check_$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value']), d['time_to_tol_seeds']['seconds_q1_median_q3'], {k: round(v*1e3,2) for k, v in d['kernel_ms_per_step'].items() if v})"; done | tee gpurun_out/check.txt
