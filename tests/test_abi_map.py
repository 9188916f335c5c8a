"""ABI overrides: the reference CLI's --abi-map file,
parsed by parse_abi_overrides (abi_model.cpp:109-153) and applied by
build_abi_map (abi_model.cpp:196-243) to every kernel's settings map.

CPU tests: the host parser's diagnostics equal the reference's on handwritten
and seeded random override files, and the CLI stops on a bad map before it
touches the GPU (ocldec.cpp:120-131).  GPU tests: with overrides, the
sm_100a pipeline's output, flags and diagnostics equal the reference's on the
reference corpus and on generated corpora; the CLI prints the map's
diagnostics against the map path."""
import json
import os
import random
import subprocess

import pytest

import paper_2107_07809_b200 as P
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
CLI = os.path.join(ROOT, "paper_2107_07809_b200", "ocldec-b200")
needs_oracle = pytest.mark.skipif(not O.available(), reason="oracle not built")

TARGETS = ["global_offset", "global_size", "work_dim", "local_size", "num_groups"]

MAPS = [
    b"0x0:2 = local_size:0\n0xc = num_groups:1\n0x10 = work_dim\n",
    b"0x30:2 = arg:out\n0x38 = global_size:2\n0x28 = arg:nope\n0x3c = foo\n0x40 = local_size:7\n",
    b"0x30 = arg:n\n0x34 = arg:a\n0x38:2 = arg:b\n0x40:2 = global_offset:1\n",
    b"# comment\n\n  16 : 1 = global_size : 1 \r\n0x8:2=global_offset:0x1\nbad line\n0x10:3 = work_dim\n",
]

HAND = [
    b"", b"\n\n# only comments\n", b"nokv\n", b"0x10:3 = arg:a\n", b"zz = arg:a\n", b"0x10 =   \n",
    b"0x10:2 = global_size:1\n  12 : 1 = work_dim \r\n0x = x\n0x1g = y\n4294967296 = a\n4294967295=b\n",
    b"0x10: = a\n:1 = b\n=c\n 0X10 = d\n+5 = e\n0x10:0x2 = f\n\t# x\n0x10:2=\x00\n",
    b"a=b=c\n0x8=arg:a:b", b"0x8 = local_size:\n0x8 = local_size:-1\n0x8 = arg:\n",
]


def random_map(rng, names=(b"n", b"a", b"b", b"out", b"in")):
    lines = []
    for _ in range(rng.randrange(1, 12)):
        r = rng.random()
        if r < 0.06:
            lines.append(rng.choice([b"", b"# c", b"   ", b"junk", b"=x", b"0x10 ="]))
            continue
        off = rng.randrange(0, 0x60, 4)
        key = (b"0x%x" % off) if rng.random() < 0.6 else b"%d" % off
        if rng.random() < 0.5:
            key += b":" + rng.choice([b"1", b"2", b"2", b"3", b"0x1", b""])
        if rng.random() < 0.4:
            tgt = b"arg:" + rng.choice(list(names) + [b"_.global_offset_0", b"nope"])
        else:
            tgt = rng.choice(TARGETS + ["bogus"]).encode()
            if rng.random() < 0.7:
                tgt += b":" + rng.choice([b"0", b"1", b"2", b"3", b"x", b"0x2"])
        sp = rng.choice([b"", b" ", b"\t"])
        lines.append(sp + key + sp + b"=" + sp + tgt + sp)
    return b"\n".join(lines) + rng.choice([b"", b"\n"])


def _diags(ds):
    return [(d.severity, d.line, d.message.encode("utf-8", "surrogateescape")) for d in ds]


def _ref_diags(ds):
    return [(d.severity, d.line, d.message) for d in ds]


@needs_oracle
def test_override_parse_matches_reference():
    rng = random.Random(2107)
    probe = b".kernel a\n  .text\n  s_endpgm\n"
    for m in HAND + MAPS + [random_map(rng) for _ in range(300)]:
        ref = O.decompile(probe, abi_map=m)
        assert _diags(P.check_abi_map(m)) == _ref_diags(ref.abi_diagnostics), m


def test_cli_bad_abi_map_stops_before_decompiling(tmp_path):
    if not os.path.exists(CLI):
        pytest.skip("CLI not built")
    inp = tmp_path / "k.asm"
    inp.write_text(".kernel k\n  .text\n  s_endpgm\n")
    amap = tmp_path / "m.txt"
    amap.write_text("0x10 = work_dim\nnokv\n0x10:3 = arg:a\n")
    p = subprocess.run([CLI, str(inp), "--abi-map", str(amap)], capture_output=True, text=True)
    assert p.returncode == 1
    assert p.stderr == (f"{amap}:2: error: override line is not key=value\n"
                        f"{amap}:3: error: override width must be 1 or 2 dwords\n")
    assert not (tmp_path / "k.cl").exists()
    p = subprocess.run([CLI, str(inp), "--abi-map", str(tmp_path / "none.txt")], capture_output=True, text=True)
    assert p.returncode == 1 and "cannot open" in p.stderr


def _check(listing, amap, **kw):
    res = P.decompile_listing(listing, P.DecompileOptions(abi_map=amap, **kw))
    o = {k: (v.encode() if isinstance(v, str) else v) for k, v in kw.items()}
    ref = O.decompile(listing, abi_map=amap, **o)
    assert res.combined == ref.combined
    assert [(k.name.encode("utf-8", "surrogateescape"), k.failed, k.structured, k.fallback_count)
            for k in res.kernels] == [(k.name, k.failed, k.structured, k.fallback_count) for k in ref.kernels]
    assert _diags(res.diagnostics) == _ref_diags(ref.diagnostics)
    assert _diags(res.abi_diagnostics) == _ref_diags(ref.abi_diagnostics)
    return res, ref


@pytest.mark.gpu
@needs_oracle
def test_overrides_reference_corpus():
    recs = [json.loads(line) for line in open(os.path.join(GOLDEN, "corpus.jsonl"))]
    rng = random.Random(9)
    changed = 0
    for rec in recs:
        listing = rec["listing"].encode("utf-8", "surrogateescape")
        for m in MAPS + [random_map(rng) for _ in range(3)]:
            _, ref = _check(listing, m)
            changed += ref.combined != rec["combined"].encode("utf-8", "surrogateescape")
    assert changed > 10  # the maps do change the output


@pytest.mark.gpu
@needs_oracle
@pytest.mark.parametrize("shape,count", [("C1", 300), ("C3", 800), ("C4", 200)])
def test_overrides_generated_corpora(shape, count):
    listing, _, _ = P.generate_corpus(shape, count, seed=31 + count)
    base = O.decompile(listing)
    rng = random.Random(count)
    changed = 0
    for m in MAPS + [random_map(rng) for _ in range(2)]:
        _, ref = _check(listing, m)
        changed += ref.combined != base.combined
    _check(listing, MAPS[0], fold_local_size=True)
    _check(listing, MAPS[2], only_kernel=P.decompile_listing(listing).kernels[1].name)
    assert changed >= 2


@pytest.mark.gpu
@needs_oracle
def test_cli_abi_map_matches_reference(tmp_path):
    if not os.path.exists(CLI):
        pytest.skip("CLI not built")
    listing, _, _ = P.generate_corpus("C3", 200, seed=8)
    inp = tmp_path / "c.asm"
    inp.write_bytes(listing)
    amap = tmp_path / "m.txt"
    amap.write_bytes(MAPS[3].replace(b"bad line\n", b"").replace(b"0x10:3 = work_dim\n", b"")
                     + b"0x30 = arg:nope\n")
    p = subprocess.run([CLI, str(inp), "--abi-map", str(amap), "-o", str(tmp_path / "c.cl")],
                       capture_output=True)
    ref = O.decompile(listing, abi_map=amap.read_bytes())
    sev = ("note", "warning", "error")
    want = b"".join(f"{amap}:{d.line}: {sev[d.severity]}: ".encode() + d.message + b"\n"
                    for d in ref.abi_diagnostics)
    want += b"".join(f"{inp}:{d.line}: {sev[d.severity]}: ".encode() + d.message + b"\n"
                     for d in ref.diagnostics)
    assert p.stderr == want
    assert (tmp_path / "c.cl").read_bytes() == ref.combined
