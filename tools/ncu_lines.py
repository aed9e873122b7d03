"""Stall samples of one kernel per CUDA source line: zips the ncu SASS source page (per-instruction
samples, in program order) with `nvdisasm -g` line annotations of the same cubin.
usage: python tools/ncu_lines.py report.ncu-rep object.o kernel_substring [top]"""
import collections, csv, io, os, re, subprocess, sys, tempfile

rep, obj, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS = hdr.index("Warp Stall Sampling (All Samples)")
samples = [int(r[iS] or 0) for r in rows[2:]]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ri = [hdr.index(h) for h in reasons]
per = [[int(r[j] or 0) for j in ri] for r in rows[2:]]
sass = [r[1].strip() for r in rows[2:]]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
dis = ""
for f in sorted(os.listdir(d)):   # the cubin that holds the kernel (a .so carries one per source)
    if f.endswith(".cubin"):
        t = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, f)], capture_output=True, text=True).stdout
        if re.search(r'\.text\.\S*' + re.escape(kname), t):
            dis = t
            break
lines, cur, fn = [], None, None
for ln in dis.splitlines():
    m = re.match(r'\s*\.text\.(\S+):', ln)
    if m:
        fn = m.group(1)
        continue
    m = re.search(r'//## File ".*?", line (\d+)', ln)
    if m:
        cur = int(m.group(1))
        continue
    if fn and kname in fn and re.search(r'/\*[0-9a-f]{4,}\*/', ln):
        lines.append(cur)
n = min(len(lines), len(samples))
print(f"{len(samples)} SASS rows in report, {len(lines)} in cubin")
agg = collections.Counter()
why = collections.defaultdict(collections.Counter)
for k in range(n):
    agg[lines[k]] += samples[k]
    for nm, v in zip(reasons, per[k]):
        why[lines[k]][nm[6:]] += v
tot = sum(agg.values()) or 1
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2105_05565_b200", "csrc",
                        sys.argv[5] if len(sys.argv) > 5 else "bfactor.cu")).read().splitlines()
for line, s in agg.most_common(top):
    txt = src[line - 1].strip()[:90] if line and line <= len(src) else ""
    top3 = ", ".join(f"{k} {v / max(s, 1):.2f}" for k, v in why[line].most_common(3))
    print(f"{s:8d} {s / tot:6.3f}  L{line}: {txt}\n{'':18s}[{top3}]")
