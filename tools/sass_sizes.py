"""SASS code size per kernel and per called sub-function (instruction-cache
budget check).  Developer aid:  python tools/sass_sizes.py [kernel-substr ...]"""
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "paper_2107_07809_b200", "libocldec_b200.so")
want = sys.argv[1:] or ["k_front", "k_lower", "k_emit"]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True)
    dis = ""
    for cub in sorted(f for f in os.listdir(d) if ".cubin" in f):
        dis += subprocess.run(["nvdisasm", os.path.join(d, cub)], capture_output=True, text=True).stdout
per = {}
cur = None
for line in dis.splitlines():
    st = line.strip()
    if st.startswith(".section") and ".text." not in st:
        cur = None  # data sections (constant banks, tables) are not code
        continue
    if line.startswith("$_Z") or line.startswith("_Z"):
        name = line.strip().rstrip(":")
        parts = name.split("$")
        entry = parts[1] if name.startswith("$") else parts[0]
        cur = None
        for w in want:
            # exact kernel identifier (k_lower must not match k_lower_wide)
            if re.search(r"\d+" + re.escape(w) + r"E", entry):
                cur = (w, parts[-1] if name.startswith("$") else "(entry)")
        if cur:
            per.setdefault(cur, 0)
        continue
    if cur and re.match(r"\s+/\*[0-9a-f]+\*/\s+\S", line) and ".word" not in line and ".dword" not in line:
        per[cur] += 1
for w in want:
    items = sorted(((c, s) for (k, s), c in per.items() if k == w), reverse=True)
    tot = sum(c for c, _ in items)
    print(f"== {w}: {tot} instrs, {tot * 16 / 1024:.1f} KB")
    for c, s in items[:int(os.environ.get("TOP", "12"))]:
        print(f"   {c:6d} {c * 16 / 1024:6.1f} KB  {s[:80]}")
