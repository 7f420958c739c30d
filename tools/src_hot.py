"""Per-CUDA-line hot spots from an ncu report (side-by-side cuda,sass source page).
usage: ncu -i X.ncu-rep --page source --csv --kernel-name regex:K --print-source cuda,sass \\
         | python tools/src_hot.py [N] [instr] [ranges=file:a-b:name,...]"""
import csv, os, sys
from collections import defaultdict
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
mode = sys.argv[2] if len(sys.argv) > 2 else "stall"
ranges = []
for a in sys.argv[3:]:
    if a.startswith("ranges="):
        for item in a[7:].split(","):
            f, ab, name = item.split(":")
            lo, hi = ab.split("-")
            ranges.append((f, int(lo), int(hi), name))
hdr = None
fname = "?"
cur = ("?", "?", "")
agg = defaultdict(lambda: [0, 0])
for r in csv.reader(sys.stdin):
    if len(r) >= 2 and r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, r[0], r[1].strip()[:90])
    try:
        st = int(r[4]) if r[4] not in ("", "-") else 0
        ie = int(r[7]) if r[7] not in ("", "-") else 0
    except ValueError:
        continue
    a = agg[cur]
    a[0] += st
    a[1] += ie
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total stall samples {ts}, warp-instr {ti}")
key = (lambda kv: -kv[1][1]) if mode == "instr" else (lambda kv: -kv[1][0])
for (f, ln, src), (st, ie) in sorted(agg.items(), key=key)[:n]:
    print(f"{st/ts*100:5.1f}%s {ie/ti*100:5.1f}%i  {f}:{ln:>4}  {src}")
if ranges:
    print("--- by range")
    tot = defaultdict(lambda: [0, 0])
    for (f, ln, src), (st, ie) in agg.items():
        name = "other:" + f
        for rf, lo, hi, nm in ranges:
            if f == rf and lo <= int(ln) <= hi:
                name = nm
                break
        tot[name][0] += st
        tot[name][1] += ie
    for name, (st, ie) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
        print(f"{st/ts*100:5.1f}%s {ie/ti*100:5.1f}%i  {name}")
