# development check: build, a pytest subset (PYK), the c5 line and the c4 / k1 EXPLICIT lines
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="timeout 900 python bench.py --no-alt --no-e2e --no-cpu-baseline"
$B --seeds ${SEEDS:-3} > gpurun_out/chk_c5.json 2>/dev/null
$B --config k1 --max-iter-tol 2000 --seeds 1 > gpurun_out/chk_k1.json 2>/dev/null
$B --config c4 --max-iter-tol 20000 --seeds 1 > gpurun_out/chk_c4.json 2>/dev/null
python - <<'PY' | tee gpurun_out/chk_summary.txt
import json, glob
for f in sorted(glob.glob("gpurun_out/chk_*.json")):
    try: d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception: print(f, "unreadable"); continue
    print(f, round(d["value"]), "iters/s; to 1e-4", d.get("time_to_tol_seeds", {}).get("seconds_q1_median_q3"),
          "s; SMs", d["roofline"].get("sms"), {k: round(v * 1e3, 1) for k, v in d["kernel_ms_per_step"].items() if v})
PY
[ -n "$PYK" ] && timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "$PYK" 2>&1 | tail -3 > gpurun_out/chk_pytest.log
true
