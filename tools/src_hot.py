"""Per-CUDA-line hot spots from an ncu report (side-by-side cuda,sass source page).
usage: ncu -i X.ncu-rep --page source --csv --kernel-name regex:K --print-source cuda,sass \
         | python tools/src_hot.py [N]"""
import csv, sys
from collections import defaultdict
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
hdr = None
cur = ("?", "")
agg = defaultdict(lambda: [0, 0])
for r in csv.reader(sys.stdin):
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = (r[0], r[1].strip()[:90])
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
for (ln, src), (st, ie) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{st/ts*100:5.1f}%s {ie/ti*100:5.1f}%i  L{ln:>4}  {src}")
