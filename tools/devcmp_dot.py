"""Developer diff of the DOT dumps: tools/devhost (OD_DUMP=3) vs the oracle's
cfg_dot / reduction.dumps on the reference corpus, nests and generated
corpora.  Not a test."""
import json
import os
import subprocess
import sys

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
import paper_2107_07809_b200 as P  # noqa: E402


def dev_dumps(listing):
    p = subprocess.run(["build/devhost"], input=listing, capture_output=True, timeout=600,
                       env=dict(os.environ, OD_DUMP="7"))
    out = p.stdout
    g, r, m = {}, {}, {}
    pos = 0
    while pos < len(out):
        nl = out.index(b"\n", pos)
        head = out[pos:nl].split()
        pos = nl + 1
        if head[0] == b"K":
            pos += int(head[4]) + int(head[5])
        elif head[0] == b"G":
            n = int(head[2])
            g[int(head[1])] = out[pos:pos + n]
            pos += n
        elif head[0] == b"M":
            n = int(head[2])
            m[int(head[1])] = out[pos:pos + n]
            pos += n
        elif head[0] == b"R":
            n = int(head[3])
            r.setdefault(int(head[1]), []).append((int(head[2]), out[pos:pos + n]))
            pos += n
        elif head[0] == b"C":
            break
    return g, r, m


def check(name, listing):
    ref = O.decompile(listing, dump_cfg=True, dump_regions=True, reduction=True)
    g, r, mm = dev_dumps(listing)
    bad = 0
    for i, k in enumerate(ref.kernels):
        if g.get(i, b"") != k.cfg_dot:
            bad += 1
            if bad < 3:
                print(f"CFG DIFF {name} k{i}\n--- ref\n{k.cfg_dot.decode()}\n--- got\n{g.get(i, b'').decode()}")
        if mm.get(i, b"") != k.reduction:
            bad += 1
            if bad < 3:
                print(f"REDUCTION DIFF {name} k{i}\n--- ref\n{k.reduction.decode()}--- got\n{mm.get(i, b'').decode()}")
        steps = [t for _, t in sorted(r.get(i, []))]
        if steps != k.region_dumps:
            bad += 1
            if bad < 3:
                print(f"REGION DIFF {name} k{i}: {len(steps)} vs {len(k.region_dumps)} dumps")
                for a, b in zip(steps, k.region_dumps):
                    if a != b:
                        print("--- ref\n" + b.decode() + "--- got\n" + a.decode())
                        break
    return bad == 0


if __name__ == "__main__":
    ok = bad = 0
    for rec in (json.loads(x) for x in open("tests/golden/corpus.jsonl")):
        if check(rec["name"], rec["listing"].encode()):
            ok += 1
        else:
            bad += 1
    for rec in list(json.loads(x) for x in open("tests/golden/nests.jsonl"))[:200]:
        if check(rec["seed"], rec["listing"].encode()):
            ok += 1
        else:
            bad += 1
    for shape, stress, n in (("C1", 1, 50), ("C2", 0, 20), ("C3", 1, 300), ("C3", 0, 300), ("C4", 1, 50)):
        lst, _, _ = P.generate_corpus(shape, n, seed=99, stress=bool(stress))
        if check(f"{shape}/{stress}", lst):
            ok += 1
        else:
            bad += 1
    print("ok", ok, "bad", bad)
