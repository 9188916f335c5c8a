"""Times the batched semantic check (developer aid): the device check of one
generated kernel whose listing loops until the interpreter's fuel runs out
(1M steps per environment), and of a C4 sample.
    python tools/sem_time.py [--nk 20000]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_07809_b200 as P  # noqa: E402

SEED = 0x5E3A171C
ap = argparse.ArgumentParser()
ap.add_argument("--nk", type=int, default=20000)
args = ap.parse_args()


def timed(listing, on):
    o = P.DecompileOptions(semantic_check=on, semantic_seed=SEED)
    P.decompile_listing(listing, o)
    t = time.perf_counter()
    r = P.decompile_listing(listing, o)
    return time.perf_counter() - t, r


# kernel 4619 of the C4 bench corpus: `s_cbranch_vccnz` on a loop-invariant vcc
listing, _, _ = P.generate_corpus("C4", 1, seed=0x210707809C4, k0=4619)
t0, _ = timed(listing, False)
t1, r = timed(listing, True)
print(f"fuel kernel: off {t0*1e3:.1f} ms, on {t1*1e3:.1f} ms, verdict {r.kernels[0].semantic}")
listing, _, _ = P.generate_corpus("C4", args.nk, seed=0x210707809C4)
t0, _ = timed(listing, False)
t1, r = timed(listing, True)
import collections
print(f"C4 {args.nk}: off {t0:.2f} s, on {t1:.2f} s, check {args.nk/(t1-t0):.0f} kernels/s",
      collections.Counter(k.semantic[0] for k in r.kernels))
