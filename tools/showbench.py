"""Summarise bench JSON lines (gpurun_out/bench_*.json)."""
import json, sys, glob
for f in sys.argv[1:] or sorted(glob.glob("gpurun_out/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f"{f}: {d['value']:.1f} {d['unit']}  ms/step {d['ms_per_step']:.4f}  tol it {d.get('iterations_to_tol')} "
          f"t {d.get('time_to_tol_s')}  e2e {(d.get('e2e') or {}).get('value')}")
    r = d.get("roofline", {})
    print("   roof", {k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items() if k not in ("step_share_by_class", "kernel", "peak_source")})
    print("   kms/step", {k: round(v, 4) for k, v in d.get("kernel_ms_per_step", {}).items()}, d.get("clocks"))
