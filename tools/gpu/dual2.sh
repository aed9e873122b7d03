# c5 line: two slots per SM + split first set (default), without the split, and the 8-warp shape
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 -k "${PYK:-tau1024 or large_tau or overlapped or kernel_ridge or explicit}" 2>&1 | tail -2 | tee gpurun_out/dual_pytest.log
B="timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline --seeds 2"
$B > gpurun_out/d2_split.json 2>/dev/null
RS_OV_SPLIT=0 $B > gpurun_out/d2_nosplit.json 2>/dev/null
RS_BF_DUAL=0 $B > gpurun_out/d2_8w.json 2>/dev/null
for f in split nosplit 8w; do python -c "
import json;d=json.loads(open('gpurun_out/d2_$f.json').read().strip().splitlines()[-1])
print('$f', round(d['value']), d['time_to_tol_seeds']['seconds'], {k: round(v*1e3,2) for k, v in d['kernel_ms_per_step'].items() if v})"; done | tee gpurun_out/d2.txt
