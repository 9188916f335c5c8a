"""The batched semantic check on the GPU.

The device restates the reference's differential backend (oracle.cpp:
interpret_asm on the listing vs evaluate_decompiled on the lowered body) and
runs it for 8 environments per kernel (od_oracle.cuh, od_semenv.cuh).  The
reference's own interpret_asm / evaluate_decompiled, fed the same
environments (oracle/ref_driver.cpp ref_semcheck), must reach the same
verdict per kernel, with the same write-trace hashes on both sides.  Kernels
the device could not hold in its fixed per-lane room (status 3) are not
compared; they must stay rare.
"""
import collections

import pytest

import paper_2107_07809_b200 as P
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.available(), reason="oracle not built")]

SEED = 0x5E3A171C


def _check(listing, max_capacity_frac=0.05):
    res = P.decompile_listing(listing, P.DecompileOptions(semantic_check=True, semantic_seed=SEED))
    ref = O.semcheck(listing, SEED)
    assert len(ref) == len(res.kernels)
    counts = collections.Counter()
    for k, (g, r) in enumerate(zip(res.kernels, ref)):
        gs = g.semantic
        assert gs is not None
        counts[gs[0]] += 1
        if gs[0] in (3, 5):
            continue
        assert gs[0] == r[0], (k, g.name, gs, r)
        if gs[0] in (0, 1):
            assert (gs[2], gs[3]) == (r[2], r[3]), (k, g.name, gs, r)
    assert counts[3] + counts[5] <= max_capacity_frac * max(1, len(ref)), counts
    return counts


def test_reference_corpus_semantics():
    listing = b"".join(x[1] for x in O.corpus())
    counts = _check(listing)
    assert counts[0] >= 20  # the harness's comparable kernels trace identically


def test_nests_semantics():
    _check(b"".join(O.make_nest(s) for s in range(1, 201)))


@pytest.mark.parametrize("shape,stress,count", [("C1", 0, 50), ("C2", 0, 200), ("C2", 1, 200),
                                                ("C3", 0, 300), ("C3", 1, 300), ("C4", 0, 300),
                                                ("C5", 0, 48)])
def test_generated_semantics(shape, stress, count):
    listing, _, _ = O.generate_corpus(shape, count, seed=4321 + count, stress=bool(stress))
    _check(listing, max_capacity_frac=0.25)


def test_session_semantic_counts():
    """Session runs with the check on (ocldec_b200_session_set_semantic, the
    bench's --semantic leg): the device counters hold the same per-status
    kernel counts as the one-shot call's per-kernel verdicts, over chunks,
    and the combined output is unchanged by the check."""
    listing, offs, _ = O.generate_corpus("C3", 600, seed=4321 + 600, stress=True)
    res = P.decompile_listing(listing, P.DecompileOptions(semantic_check=True, semantic_seed=SEED))
    want = collections.Counter(k.semantic[0] for k in res.kernels)
    s = P.Session(0)
    try:
        d_buf, n, d_offs, _ = s.generate("C3", 600, seed=4321 + 600, stress=True)
        s.set_records(False)
        s.run(d_buf, n, [int(offs[k]) for k in (0, 150, 400)])
        plain = s.output_bytes()
        s.set_semantic(True, SEED)
        s.run(d_buf, n, [int(offs[k]) for k in (0, 150, 400)])
        got = s.semantic_counts()
        assert s.output_bytes() == plain == res.combined
        assert sum(got.values()) == 600
        for i, name in enumerate(P.Session.SEM_STATUS):
            assert got[name] == want.get(i, 0), (name, got, want)
        s.set_semantic(False)
        s.run(d_buf, n, [0])
        assert sum(s.semantic_counts().values()) == 0  # a run without the check counts nothing
    finally:
        s.close()


def test_semantic_with_pool_growth_retries():
    """Kernels re-run after a pool grows (here the DOT-dump pool, on long C5
    kernels) are checked again on their re-run: the verdicts equal a run
    without retries."""
    listing, _, _ = O.generate_corpus("C5", 3, seed=0x210707809C5)
    base = P.decompile_listing(listing, P.DecompileOptions(semantic_check=True, semantic_seed=SEED))
    grown = P.decompile_listing(listing, P.DecompileOptions(semantic_check=True, semantic_seed=SEED,
                                                            dump_regions=True))
    assert [k.semantic for k in grown.kernels] == [k.semantic for k in base.kernels]
    assert all(k.semantic[0] != 4 for k in grown.kernels)
    assert sum(len(k.region_dumps) for k in grown.kernels) > 0


@pytest.mark.parametrize("shape,count,seed", [("C2", 10_000, 0x210707809C2), ("C3", 10_000, 0x210707809C3),
                                              ("C4", 10_000, 0x210707809C4)])
def test_named_configs_semantics(shape, count, seed):
    """The named C2 and C3 corpora in full (10k kernels at the bench seeds) and
    the first 10k kernels of C4: every device verdict and trace hash equals
    the reference's (reference side on 16 threads)."""
    import os
    listing, _, _ = O.generate_corpus(shape, count, seed=seed)
    res = P.decompile_listing(listing, P.DecompileOptions(semantic_check=True, semantic_seed=SEED))
    ref = O.semcheck(listing, SEED, nthreads=min(16, os.cpu_count() or 1))
    assert len(ref) == len(res.kernels) == count
    counts = collections.Counter()
    for k, (g, r) in enumerate(zip(res.kernels, ref)):
        gs = g.semantic
        counts[gs[0]] += 1
        if gs[0] in (3, 5):
            continue
        assert gs[0] == r[0], (k, gs, r)
        if gs[0] in (0, 1):
            assert (gs[2], gs[3]) == (r[2], r[3]), (k, gs, r)
    assert counts[3] + counts[5] <= 0.05 * count, counts
    print(shape, dict(counts))


def test_deferred_recheck_with_a_tiny_budget():
    """With an exact 64-step in-wave budget nearly every kernel is deferred and
    re-checked at the run's end on the auxiliary session: verdicts and hashes
    still equal the reference's, and the session counters add up."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, json, collections; sys.path.insert(0, %r)\n"
        "import paper_2107_07809_b200 as P\n"
        "from oracle import oracle as O\n"
        "l, offs, _ = O.generate_corpus('C3', 300, seed=4621, stress=True)\n"
        "r = P.decompile_listing(l, P.DecompileOptions(semantic_check=True, semantic_seed=%d))\n"
        "s = P.Session(0); s.set_records(False); s.set_semantic(True, %d)\n"
        "d_buf, n, _, _ = s.generate('C3', 300, seed=4621, stress=True); s.run(d_buf, n, [0])\n"
        "print(json.dumps({'sem': [list(k.semantic) for k in r.kernels], 'counts': s.semantic_counts()}))\n"
        % (root, SEED, SEED))
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900,
                       env=dict(os.environ, OCLDEC_B200_SEM_BUDGET="-64"))
    assert p.returncode == 0, p.stderr[-2000:]
    out = __import__("json").loads(p.stdout.strip().splitlines()[-1])
    listing, _, _ = O.generate_corpus("C3", 300, seed=4621, stress=True)
    ref = O.semcheck(listing, SEED)
    for k, (g, r) in enumerate(zip(out["sem"], ref)):
        if g[0] in (3, 5):
            continue
        assert g[0] == r[0], (k, g, r)
        if g[0] in (0, 1):
            assert (g[2], g[3]) == (r[2], r[3]), (k, g, r)
    want = collections.Counter(g[0] for g in out["sem"])
    assert [out["counts"][n] for n in P.Session.SEM_STATUS] == [want.get(i, 0) for i in range(6)]


def test_streamed_c5_semantic_counts():
    """The check inside a streamed C5 run (ocldec_b200_session_run_generated,
    several chunks): every kernel ends in exactly one final status (deferred
    kernels re-checked at the run's end), none left deferred or unrun."""
    s = P.Session(0)
    try:
        s.set_semantic(True, SEED)
        st, _, _ = s.run_generated("C5", 1200, seed=0x210707809C5, k0=300_000, chunk_bytes=96 << 20)
        got = s.semantic_counts()
        assert st["chunks"] >= 3
        assert sum(got.values()) == 1200 and got["not_run"] == 0, got
    finally:
        s.close()
