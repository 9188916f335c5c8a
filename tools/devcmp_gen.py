"""Developer diff on generated corpora: whole-listing devhost output vs the
oracle for each shape (stress and plain).  Not a test (tests/ run the GPU)."""
import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from devcmp import check, gen  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
bad = 0
for shape, stress, seed in ((2, 0, 7), (2, 1, 8), (3, 0, 9), (3, 1, 10), (4, 0, 11), (4, 1, 12), (1, 1, 13), (5, 0, 14)):
    cnt = n if shape != 5 else max(2, n // 100)
    ls = gen(shape, stress, seed, 0, cnt)
    ok = check(f"gen C{shape} stress={stress} n={cnt}", ls, verbose=bad == 0)
    print(f"C{shape} stress={stress} n={cnt}: {'ok' if ok else 'DIFF'}")
    bad += not ok
print("bad", bad)
