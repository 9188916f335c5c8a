"""Inspection outputs: the DOT dumps and the
reduction record (ReduceResult's merges, root / residue).

DecompileOptions::dump_cfg gives DecompiledKernel::cfg_dot — to_dot
(cfg.cpp:400-424) of the flow graph after mask normalization
(decompiler.cpp:72-73).  dump_regions gives ReduceResult::dumps — one
region_graph_dot (structurizer.cpp:669-688) before the first merge and after
each merge (structurizer.cpp:354-390).  The sm_100a front writes both while it
runs; the tests compare them byte for byte with the reference's, through the
C ABI and through the CLI's files (<stem>.<kernel>.cfg.dot,
<stem>.<kernel>.step<N>.dot; ocldec.cpp:68-77, 150-165)."""
import json
import os
import subprocess

import pytest

import paper_2107_07809_b200 as P
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
CLI = os.path.join(ROOT, "paper_2107_07809_b200", "ocldec-b200")
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.available(), reason="oracle not built")]


def _enc(s):
    return s.encode("utf-8", "surrogateescape")


def _check(listing, cfg=True, regions=True, **kw):
    res = P.decompile_listing(listing, P.DecompileOptions(dump_cfg=cfg, dump_regions=regions, **kw))
    o = {k: (v.encode() if isinstance(v, str) else v) for k, v in kw.items()}
    ref = O.decompile(listing, dump_cfg=cfg, dump_regions=regions, **o)
    assert res.combined == ref.combined
    assert len(res.kernels) == len(ref.kernels)
    for a, b in zip(res.kernels, ref.kernels):
        assert _enc(a.cfg_dot) == b.cfg_dot, a.name
        assert [_enc(x) for x in a.region_dumps] == b.region_dumps, a.name
    return res, ref


def test_dumps_reference_corpus():
    for rec in (json.loads(x) for x in open(os.path.join(GOLDEN, "corpus.jsonl"))):
        _check(_enc(rec["listing"]))


def test_dumps_nests_and_edges():
    nests = [json.loads(x) for x in open(os.path.join(GOLDEN, "nests.jsonl"))]
    listing = b"".join(_enc(r["listing"]).replace(b".kernel nest", b".kernel nest%d" % i)
                       for i, r in enumerate(nests[:300]))
    _, ref = _check(listing)
    assert sum(len(k.region_dumps) for k in ref.kernels) > 300
    for rec in (json.loads(x) for x in open(os.path.join(GOLDEN, "edge.jsonl"))):
        _check(_enc(rec["listing"]), fold_local_size=rec["fold_local_size"], only_kernel=rec["only_kernel"])


@pytest.mark.parametrize("shape,stress,count", [("C1", 1, 100), ("C2", 0, 30), ("C3", 1, 600),
                                                ("C3", 0, 600), ("C4", 1, 60)])
def test_dumps_generated(shape, stress, count):
    listing, _, _ = P.generate_corpus(shape, count, seed=515 + count, stress=bool(stress))
    res, ref = _check(listing)
    assert any(not k.structured for k in ref.kernels) or shape in ("C1", "C2")
    # one option at a time, and with a kernel filter
    _check(listing, cfg=True, regions=False)
    _check(listing, cfg=False, regions=True, only_kernel=res.kernels[len(res.kernels) // 2].name)


@pytest.mark.parametrize("shape,stress,count", [("C1", 1, 50), ("C3", 1, 600), ("C4", 1, 40)])
def test_reduction_record(shape, stress, count):
    """ReduceResult::merges (kind, absorbed, result) in order and the root or
    residue region ids (structurizer.cpp:354-403), kernel by kernel."""
    listing, _, _ = P.generate_corpus(shape, count, seed=88 + count, stress=bool(stress))
    res = P.decompile_listing(listing, P.DecompileOptions(record_reduction=True))
    ref = O.decompile(listing, reduction=True)
    assert res.combined == ref.combined
    for a, b in zip(res.kernels, ref.kernels):
        if b.failed:
            assert a.reduction is None
            continue
        assert _enc(a.reduction.text) == b.reduction, a.name
        assert a.reduction.reduced == b.structured
    assert any(k.reduction and not k.reduction.reduced for k in res.kernels) or shape == "C1"
    for rec in (json.loads(x) for x in open(os.path.join(GOLDEN, "corpus.jsonl"))):
        r = P.decompile_listing(_enc(rec["listing"]), P.DecompileOptions(record_reduction=True))
        f = O.decompile(_enc(rec["listing"]), reduction=True)
        assert [_enc(k.reduction.text) if k.reduction else b"" for k in r.kernels] == \
               [k.reduction for k in f.kernels]


def test_dump_pool_growth():
    """C5's deep CFGs make the dumps (~37 MB per kernel) outgrow the first
    16 MB pool: the kernels that did not fit run again into a larger pool,
    and nothing is lost or doubled."""
    listing, _, _ = P.generate_corpus("C5", 3, seed=3)
    _, ref = _check(listing)
    assert sum(len(d) for k in ref.kernels for d in k.region_dumps) > 32 << 20


def test_cli_dump_files(tmp_path):
    if not os.path.exists(CLI):
        pytest.skip("CLI not built")
    listing, _, _ = P.generate_corpus("C3", 40, seed=12, stress=True)
    inp = tmp_path / "d.asm"
    inp.write_bytes(listing)
    out = tmp_path / "out.cl"
    p = subprocess.run([CLI, str(inp), "-o", str(out), "--dump-cfg", "--dump-regions"], capture_output=True)
    ref = O.decompile(listing, dump_cfg=True, dump_regions=True)
    assert out.read_bytes() == ref.combined
    want = {}
    for k in ref.kernels:
        stem = "out." + k.name.decode()
        if k.cfg_dot:
            want[stem + ".cfg.dot"] = k.cfg_dot
        for i, d in enumerate(k.region_dumps):
            want[f"{stem}.step{i}.dot"] = d
    got = {f: (tmp_path / f).read_bytes() for f in os.listdir(tmp_path) if f.endswith(".dot")}
    assert got == want
    assert p.returncode == (1 if any(k.failed for k in ref.kernels) else 0)
