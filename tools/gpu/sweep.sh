# A/B sweep of one environment switch over bench lines (development):
#   VAR=RS_SB_NB VALUES="1 2 3" CONFIGS="c5 k1" bash tools/gpu/sweep.sh
# (VAR e.g. RS_OV_SMS, RS_SB_NB, RS_OV_SPLIT, RS_BF_DUAL; an empty value = the default)
python -c "import __graft_entry__ as g; g.build()" || exit 1
B="timeout 900 python bench.py --no-alt --no-e2e --no-cpu-baseline"
for c in ${CONFIGS:-c5}; do
  for v in ${VALUES:-""}; do
    env $VAR=$v $B --config $c --max-iter-tol 20000 --seeds ${SEEDS:-3} > gpurun_out/sweep_${c}_${VAR}_$v.json 2>/dev/null
  done
done
python - <<'PY' | tee gpurun_out/sweep_summary.txt
import json, glob
for f in sorted(glob.glob("gpurun_out/sweep_*.json")):
    try: d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception: print(f, "unreadable"); continue
    print(f, round(d["value"]), "iters/s; to 1e-4", d.get("time_to_tol_seeds", {}).get("seconds_q1_median_q3"),
          "s; SMs", d["roofline"].get("sms"), {k: round(v * 1e3, 1) for k, v in d["kernel_ms_per_step"].items() if v})
PY
