"""Hot SASS lines of one kernel from an ncu report (source page, sass view).
usage: python tools/sass_hot.py rep.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + kre, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[0].startswith("0x")]
iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
f = lambda x: float(x) if x not in ("", "-") else 0.0
tot = sum(f(r[iW]) for r in data) or 1
totE = sum(f(r[iE]) for r in data) or 1
print(f"samples {tot:.0f}  warp-instructions {totE:.3e}")
sel = sorted(data, key=lambda r: -f(r[iW]))[:top]
for r in sorted(sel, key=lambda r: int(r[0], 16)):
    print(f"{r[0][-5:]} stall {100*f(r[iW])/tot:5.1f}%  inst {100*f(r[iE])/totE:5.1f}%  {r[iS].strip()[:90]}")
