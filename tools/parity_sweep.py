"""Randomized parity sweep (developer aid, not a test): generated corpora of
every shape and form at random seeds through the GPU, each compared with the
reference (oracle, 16 threads) on combined_source, per-kernel flags and
diagnostics.  python tools/parity_sweep.py [kernels_per_case] [cases]"""
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2107_07809_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

per = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
ncase = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rng = random.Random(int(os.environ.get("SWEEP_SEED", "20261017")))
total = bad = 0
t0 = time.time()
for c in range(ncase):
    shape = rng.choice(os.environ.get("SWEEP_SHAPES", "C1,C2,C3,C4").split(","))
    stress = rng.random() < 0.5
    seed = rng.getrandbits(48)
    k0 = rng.getrandbits(20)
    n = per if shape not in ("C1", "C5") else min(per, 500 if shape == "C1" else 100)
    listing, offs, _ = O.generate_corpus(shape, n, seed=seed, k0=k0, stress=stress)
    fold = rng.random() < 0.25
    gpu = P.decompile_listing(listing, P.DecompileOptions(fold_local_size=fold))
    ref = O.decompile_par(listing, [int(x) for x in offs[:-1]], nthreads=16, fold_local_size=fold)
    ok = gpu.combined == ref.combined and len(gpu.kernels) == len(ref.kernels)
    ok = ok and all((g.failed, g.structured, g.fallback_count) == (r.failed, r.structured, r.fallback_count)
                    for g, r in zip(gpu.kernels, ref.kernels))
    ok = ok and [(d.severity, d.line, d.message.encode("utf-8", "surrogateescape")) for d in gpu.diagnostics] == \
        [(d.severity, d.line, d.message) for d in ref.diagnostics]
    total += n
    if not ok:
        bad += 1
        print(f"MISMATCH case {c}: {shape} stress={stress} seed={seed:#x} k0={k0} fold={fold}", flush=True)
print(f"sweep: {ncase} cases, {total} kernels, {bad} mismatching cases, {time.time() - t0:.0f} s")
