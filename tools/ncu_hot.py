"""Summarise an ncu source page (SASS) export: top instructions by stall samples + stall totals.
usage: ncu -i rep --page source --csv -k regex:NAME --print-source sass > x.csv; python tools/ncu_hot.py x.csv"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
S = idx["Warp Stall Sampling (All Samples)"]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        v = float(r[S] or 0)
    except ValueError:
        continue
    data.append((v, r[idx["Address"]], r[idx["Source"]][:90], r[idx["Instructions Executed"]]))
    for h in stalls:
        try:
            tot[h] += float(r[idx[h]] or 0)
        except ValueError:
            pass
T = sum(d[0] for d in data) or 1
print("stall totals:", ", ".join(f"{k[6:]}={v/T:.1%}" for k, v in tot.most_common(8)))
for v, a, src, ex in sorted(data, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v/T:6.1%} {a} {src:90s} exec={ex}")
