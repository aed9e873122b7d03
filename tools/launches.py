"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per-kernel count, total,
mean, share of our kernels.  usage: python tools/launches.py launches.csv [prefix-filter]"""
import csv, sys, collections, re
lines = [ln for ln in open(sys.argv[1]) if not ln.startswith("==")]
rows = list(csv.DictReader(lines))
agg = collections.OrderedDict()
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"]
    m = re.search(r"(k_[A-Za-z0-9_]+)", name)
    short = m.group(1) if m else name.split("(")[0][:60]
    t = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0 if r["Metric Unit"] == "usecond" else 1e3)
    a = agg.setdefault(short, [0, 0.0])
    a[0] += 1
    a[1] += t
ours = {k: v for k, v in agg.items() if k.startswith("k_")}
tot = sum(v[1] for v in ours.values()) or 1
print(f"{'kernel':28s} {'launches':>8s} {'total_us':>11s} {'mean_us':>10s} {'share':>7s}")
for k, (c, t) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:28s} {c:8d} {t:11.1f} {t / c:10.2f} {t / tot:7.1%}")
print(f"ours total {tot:.1f} us over {sum(v[0] for v in ours.values())} launches; other kernels: "
      f"{sum(v[0] for k, v in agg.items() if k not in ours)}")
