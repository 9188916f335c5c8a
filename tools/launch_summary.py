"""Per-kernel totals of an ncu launch list (`ncu --metrics gpu__time_duration.sum
--csv --log-file launches.csv ...`): launches, total ms and share of the
timed work (k_gen, the corpus generator, is outside the bench's timed step).
    python tools/launch_summary.py launches.csv "header comment" > launch_summary.csv"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1], errors="replace")) if len(r) > 10]
h = rows[0]
ki, mi, ui, vi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].strip()
    tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
timed = sum(v for k, v in tot.items() if not k.endswith("k_gen"))
print("# " + (sys.argv[2] if len(sys.argv) > 2 else "ncu launch list summary"))
print("kernel,launches,total_ms,share")
for k in sorted(tot, key=lambda k: -tot[k]):
    share = 0.0 if k.endswith("k_gen") else tot[k] / timed
    print(f"{k},{cnt[k]},{tot[k]:.2f},{share:.4f}")
