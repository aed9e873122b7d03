# k_bfactor_lp<4> slice depth / stages variants on the c5 and k1 lines
for v in "" "-DRS_LP4_KS=8 -DRS_LP4_ST=4" "-DRS_LP4_KS=8 -DRS_LP4_ST=3"; do
  RS_NVCC_EXTRA="$v" python -m paper_2105_05565_b200._build --force > /dev/null 2>&1 || { echo "build fail $v"; continue; }
  tag=$(echo "$v" | tr -d ' =-' | tr -d 'D')
  timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline --seeds 3 > gpurun_out/lpks_c5_$tag.json 2>/dev/null
  timeout 600 python bench.py --no-alt --no-e2e --no-cpu-baseline --config k1 --max-iter-tol 2000 --seeds 1 > gpurun_out/lpks_k1_$tag.json 2>/dev/null
done
python -m paper_2105_05565_b200._build --force > /dev/null 2>&1
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/lpks_*.json")):
    try: d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception: print(f, "unreadable"); continue
    r = d["roofline"]
    print(f, round(d["value"]), round(d["time_to_tol_s"] * 1e3, 2), r.get("sms"), {k: round(v * 1e3, 1) for k, v in d["kernel_ms_per_step"].items() if v})
PY
