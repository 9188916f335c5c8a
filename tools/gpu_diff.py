"""GPU debugging aid: per-kernel GPU vs oracle diff for a generated corpus."""
import sys
sys.path.insert(0, ".")
import difflib
import paper_2107_07809_b200 as P
from oracle import oracle as O

shape, stress, seed, count = (int(x) for x in sys.argv[1:5])
listing, offs, _ = P.generate_corpus(shape, count, seed=seed, stress=bool(stress))
bad = 0
for k in range(count):
    part = listing[int(offs[k]):int(offs[k + 1])]
    g = P.decompile_listing(part).combined
    r = O.decompile(part).combined
    if g != r:
        bad += 1
        if bad <= 2:
            print(f"=== kernel {k} differs")
            print(part.decode(errors="replace"))
            for l in difflib.unified_diff(r.decode(errors="replace").splitlines(),
                                          g.decode(errors="replace").splitlines(), "ref", "gpu", lineterm=""):
                print(l)
print("bad", bad, "of", count)
