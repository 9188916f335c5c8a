"""Aggregates an ncu correlated source export (--page source --csv
--print-source cuda,sass) per CUDA source line and per function-ish region:
warp instructions, thread instructions, stall samples.  Developer aid."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
f = None
hdr = None
agg = defaultdict(lambda: [0, 0, 0, ""])
tot = [0, 0, 0]
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9 or not r[0].isdigit():
        continue
    try:
        samp = int(r[4] or 0)
        wi = int(r[7] or 0)
        ti = int(r[8] or 0)
    except ValueError:
        continue
    a = agg[(f, int(r[0]))]
    a[0] += wi
    a[1] += ti
    a[2] += samp
    a[3] = r[1][:70]
    tot[0] += wi
    tot[1] += ti
    tot[2] += samp
print(f"total warp inst {tot[0]:.3e} thread inst {tot[1]:.3e} samples {tot[2]} active/warp {tot[1]/max(tot[0],1):.2f}")
key = 2 if len(sys.argv) > 3 and sys.argv[3] == "samples" else 0
for (fn, ln), (wi, ti, s, src) in sorted(agg.items(), key=lambda x: -x[1][key])[:top]:
    print(f"{fn:16s}:{ln:5d} wi {wi/tot[0]*100:5.2f}% samp {s/max(tot[2],1)*100:5.2f}% act {ti/max(wi,1):5.2f} | {src}")
