"""GPU parity tests: the sm_100a pipeline, called through the C ABI, must
produce byte-identical combined_source (and identical per-kernel flags) to
the reference on the same inputs (bit-exact: the path is integer/byte work).

Checked against: the reference's CLI golden pair, the committed corpus /
nest / edge fixtures, the live oracle (oracle/_ref, the reference compiled
from its sources) on generated corpora of every shape, and — at sizes the
oracle cannot finish — size-independent properties (determinism, chunking
invariance, host/device generator identity, per-kernel independence).
"""
import hashlib
import json
import os

import pytest

import paper_2107_07809_b200 as P
from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
pytestmark = pytest.mark.gpu


def _jsonl(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [json.loads(line) for line in f]


def _flags(res):
    return [(k.name, k.failed, k.structured, k.fallback_count) for k in res.kernels]


def test_copy_golden():
    listing = open(os.path.join(GOLDEN, "copy.asm"), "rb").read()
    res = P.decompile_listing(listing)
    assert res.combined == open(os.path.join(GOLDEN, "copy.cl"), "rb").read()
    assert _flags(res) == [("copy", False, True, 0)]
    assert res.kernels[0].instructions == 12


def test_reference_corpus():
    for rec in _jsonl("corpus.jsonl"):
        res = P.decompile_listing(rec["listing"])
        assert res.combined_source() == rec["combined"], rec["name"]
        k = rec["kernels"][0]
        assert _flags(res) == [(k["name"], k["failed"], k["structured"], k["fallbacks"])], rec["name"]
        assert res.kernels[0].fallback_count == rec["expected_fallbacks"]


def test_reference_corpus_as_one_listing():
    recs = _jsonl("corpus.jsonl")
    listing = "".join(r["listing"] for r in recs)
    res = P.decompile_listing(listing)
    if O.available():
        assert res.combined == O.decompile(listing.encode()).combined
    assert res.combined_source() == "\n".join(r["combined"] for r in recs)


def test_nest_fixtures():
    recs = _jsonl("nests.jsonl")
    listing = "".join(r["listing"] for r in recs)
    res = P.decompile_listing(listing)
    assert res.combined_source() == "\n".join(r["combined"] for r in recs)
    assert all(k.structured for k in res.kernels)


@pytest.mark.skipif(not O.available(), reason="oracle not built")
def test_1000_nests_vs_oracle():
    listing = b"".join(O.make_nest(s) for s in range(1, 1001))
    res = P.decompile_listing(listing)
    ref = O.decompile(listing)
    assert res.combined == ref.combined
    assert [(k.failed, k.structured, k.fallback_count) for k in res.kernels] == \
           [(k.failed, k.structured, k.fallback_count) for k in ref.kernels]


def test_edge_cases():
    for rec in _jsonl("edge.jsonl"):
        res = P.decompile_listing(rec["listing"].encode("utf-8", "surrogateescape"),
                                  P.DecompileOptions(fold_local_size=rec["fold_local_size"],
                                                     only_kernel=rec["only_kernel"]))
        assert res.combined_source() == rec["combined"], rec["name"]
        want = [(k["name"], k["failed"], k["structured"], k["fallbacks"]) for k in rec["kernels"]]
        assert _flags(res) == want, rec["name"]
        errs = [d for d in rec["diagnostics"] if d[0] == 2 and not rec["kernels"]]
        if errs:  # split_kernels errors: zero kernels + one error at that line
            assert [(d.severity, d.line, d.message) for d in res.diagnostics] == [tuple(errs[0])]


@pytest.mark.parametrize("g", json.load(open(os.path.join(GOLDEN, "gen.json"))),
                         ids=lambda g: f"C{g['shape']}s{g['stress']}")
def test_generated_fixture_hashes(g):
    listing, _, ni = P.generate_corpus(g["shape"], g["count"], seed=g["seed"], stress=bool(g["stress"]))
    assert hashlib.sha256(listing).hexdigest() == g["listing_sha256"]
    res = P.decompile_listing(listing)
    assert hashlib.sha256(res.combined).hexdigest() == g["combined_sha256"]
    assert len(res.combined) == g["combined_len"]
    assert sum(k.failed for k in res.kernels) == g["failed"]
    assert sum(k.fallback_count for k in res.kernels) == g["fallbacks"]
    assert sum(k.instructions for k in res.kernels) == ni


@pytest.mark.skipif(not O.available(), reason="oracle not built")
@pytest.mark.parametrize("shape,stress,count", [("C1", 1, 300), ("C2", 0, 200), ("C2", 1, 200),
                                                ("C3", 0, 1000), ("C3", 1, 1000), ("C4", 0, 150),
                                                ("C4", 1, 150)])
def test_generated_vs_oracle(shape, stress, count):
    listing, offs, _ = P.generate_corpus(shape, count, seed=1234 + count, stress=bool(stress))
    res = P.decompile_listing(listing)
    ref = O.decompile(listing)
    assert res.combined == ref.combined
    assert [(k.failed, k.structured, k.fallback_count) for k in res.kernels] == \
           [(k.failed, k.structured, k.fallback_count) for k in ref.kernels]


@pytest.mark.skipif(not O.available(), reason="oracle not built")
def test_long_kernels_sample_vs_oracle():
    listing, offs, ni = P.generate_corpus("C5", 3, seed=0x210707809C5, k0=1000)
    res = P.decompile_listing(listing)
    assert res.combined == O.decompile(listing).combined
    assert ni > 20000


def test_session_device_generation_matches_host():
    s = P.Session(0)
    try:
        for shape in ("C2", "C3"):
            d_buf, n, d_offs, ni = s.generate(shape, 64, seed=77)
            host, offs, hni = P.generate_corpus(shape, 64, seed=77)
            assert n == len(host) and ni == hni
            s.run(d_buf, n, [0])
            dev_out = s.output_bytes()
            assert dev_out == P.decompile_listing(host).combined
    finally:
        s.close()


def test_chunked_run_matches_single_chunk():
    """Chunking at .kernel boundaries is invisible in the output."""
    s = P.Session(0)
    try:
        d_buf, n, d_offs, ni = s.generate("C3", 200, seed=5, stress=False)
        host, offs, _ = P.generate_corpus("C3", 200, seed=5)
        s.run(d_buf, n, [0])
        one = s.output_bytes()
        s.run(d_buf, n, [int(offs[k]) for k in (0, 1, 17, 99, 150, 199)])
        many = s.output_bytes()
        st = s.stats()
        assert one == many and st["kernels"] == 200
    finally:
        s.close()


def test_small_arena_retry_path():
    """Kernels that outgrow the per-thread arena are re-run with a larger one."""
    listing, _, _ = P.generate_corpus("C4", 40, seed=3)
    a = P.decompile_listing(listing, P.DecompileOptions(arena_bytes=64 << 10))
    b = P.decompile_listing(listing)
    assert a.combined == b.combined


def test_empty_and_preamble_only():
    assert P.decompile_listing("").kernels == []
    r = P.decompile_listing(".amdcl2\n.gpu Fiji\n")
    assert r.kernels == [] and r.combined == b"" and r.diagnostics == []


@pytest.mark.skipif(not O.available(), reason="oracle not built")
def test_larger_c4_sample_vs_oracle():
    """A 1,500-kernel C4 sample (both size classes, straight and branching,
    stress syntax) in one listing: one decompile wave with the size-sorted
    interleaving, compared byte for byte with the reference."""
    listing, offs, ni = P.generate_corpus("C4", 1500, seed=0x210707809C4 + 1, stress=True)
    res = P.decompile_listing(listing)
    ref = O.decompile(listing)
    assert res.combined == ref.combined
    assert [(k.failed, k.structured, k.fallback_count) for k in res.kernels] == \
           [(k.failed, k.structured, k.fallback_count) for k in ref.kernels]


@pytest.mark.skipif(not O.available(), reason="oracle not built")
def test_host_chunking_vs_oracle(monkeypatch):
    """The host path cuts the listing into chunks at .kernel lines
    (OCLDEC_B200_CHUNK_BYTES); every chunk runs all phases, the state of a
    kernel moves between phase launches, and the combined output must not
    change."""
    listing, offs, _ = P.generate_corpus("C3", 1200, seed=91, stress=True)
    ref = O.decompile(listing).combined
    monkeypatch.setenv("OCLDEC_B200_CHUNK_BYTES", str(len(listing) // 7))
    res = P.decompile_listing(listing, P.DecompileOptions(arena_bytes=(96 << 20) + 4096))
    assert res.combined == ref


@pytest.mark.skipif(not O.available(), reason="oracle not built")
@pytest.mark.parametrize("pinned", [True, False])
def test_session_run_host_overlapped_chunks(monkeypatch, pinned):
    """session_run_host loads chunk c+1 and stores chunk c's output on a copy
    stream while chunk c runs (two text buffers).  The stored bytes must be
    the reference's combined output, with pinned or pageable host buffers,
    and a too-small output buffer must give -2 and the needed length."""
    import numpy as np
    import torch
    listing, _, _ = P.generate_corpus("C4", 500, seed=17, stress=True)
    ref = O.decompile(listing).combined
    monkeypatch.setenv("OCLDEC_B200_CHUNK_BYTES", str(len(listing) // 5))
    cap = 2 * len(listing) + 4096
    if pinned:
        hin = torch.frombuffer(bytearray(listing), dtype=torch.uint8).pin_memory()
        hout = torch.empty(cap, dtype=torch.uint8).pin_memory()
        pin_ptr, out_ptr = hin.data_ptr(), hout.data_ptr()
    else:
        hin = np.frombuffer(listing, dtype=np.uint8).copy()
        hout = np.zeros(cap, dtype=np.uint8)
        pin_ptr, out_ptr = hin.ctypes.data, hout.ctypes.data
    s = P.Session()
    try:
        for _ in range(2):  # buffers reused across calls
            n = s.run_host(pin_ptr, len(listing), out_ptr, cap)
            got = bytes(hout[:n].numpy()) if pinned else hout[:n].tobytes()
            assert got == ref
        with pytest.raises(RuntimeError, match="-2"):
            s.run_host(pin_ptr, len(listing), out_ptr, len(ref) // 2)
    finally:
        s.close()


def _one_huge_kernel(shape, count, seed):
    """The first kernel's header, then the .text lines of `count` generated
    kernels as one kernel (labels renamed apart, s_endpgm dropped but the
    last)."""
    import re
    listing, _, _ = P.generate_corpus(shape, count, seed=seed)
    head, body, seen_text, in_text, k = [], [], False, False, 0
    for line in listing.split(b"\n"):
        s = line.strip()
        if s.startswith(b".kernel"):
            in_text = False
            k += 1
            continue
        line = re.sub(rb"\bL(\d+)\b", b"L\\1_%d" % k, line)  # labels unique per source kernel
        if s.startswith(b".text"):
            in_text = True
            seen_text = True
            continue
        if in_text:
            if s != b"s_endpgm":
                body.append(line)
        elif not seen_text:
            head.append(line)
    return b"\n".join([b".kernel huge"] + head + [b"  .text"] + body + [b"    s_endpgm", b""])


@pytest.mark.skipif(not O.available(), reason="oracle not built")
def test_huge_kernel_and_long_lines():
    """Maximum sizes: one kernel of ~25k branching instructions (arena
    budget, one thread doing the whole kernel), and lines far longer than the
    decode stage (the decoder reads those from HBM)."""
    big = _one_huge_kernel("C3", 300, seed=21)
    ref = O.decompile(big)
    assert len(ref.kernels) == 1 and not ref.kernels[0].failed
    res = P.decompile_listing(big)
    assert res.combined == ref.combined
    assert res.kernels[0].instructions > 15_000
    long_arg = b"s" * 40_000
    listing = (b".kernel k\n  .text\n  v_mov_b32 v1, v2 ; " + b"c" * 70_000 + b"\n"
               b"  s_nop " + long_arg + b"\n  v_add_u32 v1, vcc, " + b"0x" + b"0" * 30_000 + b"5, v1\n"
               b"  s_endpgm\n")
    r = P.decompile_listing(listing)
    f = O.decompile(listing)
    assert r.combined == f.combined
    assert [(d.severity, d.line, d.message.encode()) for d in r.diagnostics] == \
           [(d.severity, d.line, d.message) for d in f.diagnostics]


@pytest.mark.skipif(not O.available(), reason="oracle not built")
def test_session_batch_names_and_diagnostics():
    """The batch (session) form returns what SURVEY §8(b) lists for it: per
    kernel source spans, flags and fallbacks, name spans into the caller's
    listing, and the diagnostics in sink order, over a multi-chunk run."""
    import numpy as np
    listing, offs, _ = P.generate_corpus("C3", 700, seed=314, stress=True)
    ref = O.decompile(listing)
    s = P.Session(0)
    try:
        d_buf, n, _, _ = s.generate("C3", 700, seed=314, stress=True)
        assert n == len(listing)
        s.run(d_buf, n, [int(offs[k]) for k in (0, 200, 450)])
        noff, nlen = s.names()
        names = [listing[int(o):int(o) + int(ln)] for o, ln in zip(noff, nlen)]
        assert names == [k.name for k in ref.kernels]
        koff, klen, kfl, kfb = s.kernels()
        out = s.output_bytes()
        srcs = [out[int(o):int(o) + int(ln)] for o, ln in zip(koff, klen)]
        assert srcs == [k.source for k in ref.kernels]
        assert [bool(f & 1) for f in kfl] == [k.failed for k in ref.kernels]
        assert list(kfb) == [k.fallback_count for k in ref.kernels]
        assert [(d.severity, d.line, d.message.encode("utf-8", "surrogateescape")) for d in s.diagnostics()] == \
               [(d.severity, d.line, d.message) for d in ref.diagnostics]
        assert len(ref.diagnostics) > 50
    finally:
        s.close()


def test_comment_heavy_chunk_retries_smaller(monkeypatch):
    """A chunk whose comment-stripped copies would push it past the u32
    offset range (chunk + aux >= 4 GiB) is re-run in smaller chunks by the
    host path, with the same output as the listing without the comments."""
    listing, _, _ = P.generate_corpus("C2", 300_000, seed=5)
    assert len(listing) > (2 << 30) - (128 << 20)
    commented = listing.replace(b"\n", b" /* c */\n")  # every line needs the aux copy
    monkeypatch.setenv("OCLDEC_B200_CHUNK_BYTES", str(7 << 29))  # one 3.5 GiB chunk: overflows
    a = P.decompile_listing(commented)
    monkeypatch.setenv("OCLDEC_B200_CHUNK_BYTES", str(1 << 30))
    b = P.decompile_listing(listing)
    assert a.combined == b.combined and len(a.kernels) == 300_000


def test_session_without_host_records_matches():
    """ocldec_b200_session_set_records(0): the same combined output and totals
    as a run that keeps per-kernel host records (the bench's device path)."""
    listing, offs, ni = P.generate_corpus("C3", 3000, seed=71, stress=True)
    import ctypes
    s = P.Session(0)
    try:
        buf = ctypes.create_string_buffer(listing, len(listing))
        out = []
        for keep in (True, False):
            s.set_records(keep)
            cap = len(listing) * 3 + (1 << 20)
            host_out = ctypes.create_string_buffer(cap)
            n = s.run_host(ctypes.addressof(buf), len(listing), ctypes.addressof(host_out), cap)
            st = s.stats()
            out.append((host_out.raw[:n], st["instructions"], st["failed"], st["goto_form"], st["fallbacks"]))
        assert out[0] == out[1]
        assert out[0][0] == P.decompile_listing(listing).combined and out[0][1] == ni
    finally:
        s.close()
