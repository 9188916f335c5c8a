"""Per-function aggregation of an ncu correlated source export: maps each
CUDA source line to the enclosing function definition in the csrc headers.
Developer aid:  python tools/ncu_funcs.py export.csv [top]"""
import csv
import os
import re
import sys
from collections import defaultdict

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2107_07809_b200", "csrc")
starts = {}
pat = re.compile(r"^\s*(?:OD_NOINL|OD_INL|OD_HD|__global__|__device__)[^(]*?\b(\w+)\s*\(")
REV = os.environ.get("REV")  # read the sources at this git revision (the profiled build)


def source_lines(f):
    if REV:
        import subprocess
        return subprocess.run(["git", "show", f"{REV}:paper_2107_07809_b200/csrc/{f}"], capture_output=True,
                              text=True, cwd=os.path.dirname(CSRC) + "/..").stdout.splitlines()
    return open(os.path.join(CSRC, f)).read().splitlines()


for f in os.listdir(CSRC):
    if not (f.endswith(".cuh") or f.endswith(".cu")):
        continue
    lst = []
    for i, line in enumerate(source_lines(f), 1):
        m = pat.match(line)
        if m:
            lst.append((i, m.group(1)))
    starts[f] = lst


def func_of(f, ln):
    best = "?"
    for i, name in starts.get(f, []):
        if i <= ln:
            best = name
        else:
            break
    return best


rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
agg = defaultdict(lambda: [0, 0])
f = None
tot = [0, 0]
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) < 9 or not r[0].isdigit():
        continue
    try:
        samp, wi = int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    k = (f, func_of(f, int(r[0])))
    agg[k][0] += samp
    agg[k][1] += wi
    tot[0] += samp
    tot[1] += wi
for (fn, name), (s, wi) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{s / max(tot[0], 1) * 100:6.2f}% samp {wi / max(tot[1], 1) * 100:6.2f}% inst  {fn}:{name}")
