# k_iterate: next g gathered beside the stop rule -- parity subset and the EXPLICIT lines
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="timeout 900 python bench.py --no-alt --no-e2e --no-cpu-baseline"
$B --seeds 5 > gpurun_out/gg_c5.json 2>/dev/null
$B --config k1 --max-iter-tol 2000 --seeds 1 > gpurun_out/gg_k1.json 2>/dev/null
$B --config c4 --max-iter-tol 20000 --seeds 1 > gpurun_out/gg_c4.json 2>/dev/null
$B --config c2 --mode explicit --seeds 1 > gpurun_out/gg_c2e.json 2>/dev/null
python - <<'PY' | tee gpurun_out/gg_summary.txt
import json, glob
for f in sorted(glob.glob("gpurun_out/gg_*.json")):
    try: d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception: print(f, "unreadable"); continue
    r = d["roofline"]
    print(f, round(d["value"]), round(d["time_to_tol_s"] * 1e3, 2), d.get("time_to_tol_seeds", {}).get("seconds_q1_median_q3"), r.get("sms"), {k: round(v * 1e3, 1) for k, v in d["kernel_ms_per_step"].items() if v})
PY
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -k "explicit or tau1024 or kernel or multirank or overlapped" 2>&1 | tail -3 > gpurun_out/gg_pytest.log
