python -c "import __graft_entry__ as g; g.build()" || exit 1
B="timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline"
for s in 0 66; do RS_OV_SMS=$s $B --config k1 --max-iter-tol 2000 --seeds 1 > gpurun_out/k1m_$s.json 2>/dev/null; done
$B --seeds 3 > gpurun_out/k1m_c5.json 2>/dev/null
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/k1m_*.json")):
    d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
    print(f, round(d["value"]), round(d["time_to_tol_s"] * 1e3, 2), r.get("sms"), {k: round(v * 1e3, 1) for k, v in d["kernel_ms_per_step"].items() if v})
PY
