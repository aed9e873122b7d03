# k_iterate next-step row preload: parity subset, c5 / k1 lines, phase probe
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -x -k "${PYK:-tau1024 or blocked_inverse or explicit}" 2>&1 | tail -5 | tee gpurun_out/pre_pytest.log
B="timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline"
for s in ${C5S:-0 40}; do RS_OV_SMS=$s $B --seeds 5 > gpurun_out/pre_c5_$s.json 2>/dev/null; done
$B --config k1 --max-iter-tol 2000 --seeds 1 > gpurun_out/pre_k1.json 2>/dev/null
python - <<'PY' | tee gpurun_out/pre_summary.txt
import json, glob
for f in sorted(glob.glob("gpurun_out/pre_*.json")):
    try: d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e: print(f, "unreadable"); continue
    r = d["roofline"]
    print(f, round(d["value"]), "t_tol_ms", round(d["time_to_tol_s"] * 1e3, 2), d.get("time_to_tol_seeds", {}).get("seconds_q1_median_q3"), "sms", r.get("sms"),
          {k: round(v * 1e3, 1) for k, v in d["kernel_ms_per_step"].items() if v})
PY
RS_NVCC_EXTRA=-DRS_IT_PHASES python -m paper_2105_05565_b200._build --force > /dev/null 2>&1 && \
  for nb in 1 2; do RS_SB_NB=$nb timeout 300 python tools/probe_it_phases.py c5 232 2>&1 | tail -12 > gpurun_out/pre_itphases_$nb.txt; done
python -m paper_2105_05565_b200._build --force > /dev/null 2>&1
