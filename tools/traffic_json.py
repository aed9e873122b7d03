"""Build profiles/traffic.json from ncu CSVs (--metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum --csv): per key "config/mode/class", the mean DRAM bytes per launch of the
named kernel.  usage: python tools/traffic_json.py out.json key=kernel_regex=csv[=units_per_launch] [...]
(units_per_launch: iterations / slots of one captured launch of a group kernel; bench.py scales the
bytes to its own launches)"""
import csv, json, re, statistics, sys, os

out = sys.argv[1]
res = json.load(open(out)) if os.path.exists(out) else {}
for spec in sys.argv[2:]:
    parts = spec.split("=")
    key, kre, path = parts[0], parts[1], parts[2]
    units = float(parts[3]) if len(parts) > 3 else None
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    per = {}
    for r in csv.DictReader(lines):
        if not re.search(kre, r.get("Kernel Name", "")):
            continue
        lid = r["ID"]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "nsecond": 1e-9}.get(unit, 1)
        per.setdefault(lid, {})[r["Metric Name"]] = v * scale
    launches = [p for p in per.values() if "dram__bytes_read.sum" in p]
    if not launches:
        print("no launches for", key)
        continue
    b = [p["dram__bytes_read.sum"] + p.get("dram__bytes_write.sum", 0) for p in launches]
    t = [p.get("gpu__time_duration.sum", 0) for p in launches]
    res[key] = {"kernel_regex": kre, "bytes_per_launch": statistics.mean(b),
                "launches": len(b), "ncu_duration_s_mean": statistics.mean(t),
                "source": os.path.basename(path)}
    if units:
        res[key]["units_per_launch"] = units
    print(key, res[key])
json.dump(res, open(out, "w"), indent=1)
