"""Parity at the named configs' bench seeds.

The whole C2 and C3 corpora the bench names (10,000 kernels each, seeds
0x210707809C2 / 0x210707809C3) and a 128-kernel C5 sample spread over the
1M-kernel index range (seed 0x210707809C5) are decompiled on the GPU through
the C ABI and compared with the reference (oracle/_ref, the reference
compiled from its own sources) kernel by kernel: source bytes, name,
failed / structured flags, fallback count, the diagnostics list (severity,
listing-global line, message) and combined_source.  Bit-exact: the path is
byte and integer work.

The oracle runs decompile_listing over slices of the listing in parallel
(ref_decompile_par); slices are independent by construction
(decompiler.cpp:55-101) and their results are joined exactly as
combined_source joins kernels (decompiler.cpp:105-115).
"""
import os

import numpy as np
import pytest

import paper_2107_07809_b200 as P
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.available(), reason="oracle not built")]

SEEDS = {"C2": 0x210707809C2, "C3": 0x210707809C3, "C5": 0x210707809C5}


def _compare(listing, kstarts, res):
    ref = O.decompile_par(listing, kstarts)
    assert len(res.kernels) == len(ref.kernels)
    for i, (g, r) in enumerate(zip(res.kernels, ref.kernels)):
        assert g.name.encode() == r.name, i
        assert (g.failed, g.structured, g.fallback_count) == (r.failed, r.structured, r.fallback_count), \
            (i, g.name)
        assert g.source.encode("utf-8", "surrogateescape") == r.source, (i, g.name)
    got_d = [(d.severity, d.line, d.message.encode("utf-8", "surrogateescape")) for d in res.diagnostics]
    want_d = [(d.severity, d.line, d.message) for d in ref.diagnostics]
    assert got_d == want_d
    assert res.combined == ref.combined
    return ref


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_full_named_corpus_vs_oracle(cfg):
    listing, offs, ni = O.generate_corpus(cfg, 10_000, seed=SEEDS[cfg])
    # the product's generator builds the same bytes (the bench corpus)
    plisting, poffs, pni = P.generate_corpus(cfg, 10_000, seed=SEEDS[cfg])
    assert plisting == listing and pni == ni
    res = P.decompile_listing(listing)
    assert sum(k.instructions for k in res.kernels) == ni
    _compare(listing, offs[:-1], res)


def _c5_sample(n=128, span=1_000_000):
    ks = [int(i * (span - 1) // (n - 1)) for i in range(n)]
    parts, starts, ni, pos = [], [], 0, 0
    for k in ks:
        b, _, i = O.generate_corpus("C5", 1, seed=SEEDS["C5"], k0=k)
        starts.append(pos)
        parts.append(b)
        pos += len(b)
        ni += i
    return b"".join(parts), np.array(starts, dtype=np.uint64), ni, ks


def test_c5_sample_vs_oracle():
    """128 kernels of the 1M-kernel C5 corpus, k spread evenly over
    [0, 1M): long (~10k-instruction) deep-CFG kernels with 64-bit pairs."""
    listing, starts, ni, ks = _c5_sample()
    assert ni > 128 * 7000
    res = P.decompile_listing(listing)
    assert sum(k.instructions for k in res.kernels) == ni
    ref = _compare(listing, starts, res)
    assert sum(k.structured for k in ref.kernels) > 0


def test_c5_device_generated_sample_matches_host():
    """The device generator (the bench's C5 input) builds the sampled kernels
    byte for byte as the host generator the oracle consumed."""
    s = P.Session(0)
    try:
        for k in (0, 499_999, 999_999):
            d_buf, n, d_offs, ni = s.generate("C5", 1, seed=SEEDS["C5"], k0=k)
            host = bytearray(n)
            import ctypes
            P.copy(ctypes.addressof((ctypes.c_char * n).from_buffer(host)), d_buf, n)
            want, _, wni = O.generate_corpus("C5", 1, seed=SEEDS["C5"], k0=k)
            assert bytes(host) == want and ni == wni
    finally:
        s.close()


def test_vertical_tab_and_formfeed_separators():
    """Operands separated by \\v, \\f and a mid-line \\r (isspace bytes the
    reference's tokenizer splits on, asm_frontend.cpp:80-107) are sized and
    decoded like spaces, on every line including the listing's last."""
    body = (".kernel vt\n  .config\n    .dims x\n  .text\n"
            "    v_mov_b32 v0\vv1\vv2\n"
            "    v_add_u32\fv3,\fvcc,\fv0,\vv1\n"
            "    s_mov_b32 s0\r\vs1\n"
            "    v_mul_lo_u32 v4\vv3\fv0\vv1\fv2\n"
            "    s_endpgm\v\f")
    for listing in (body.encode(), body.encode() + b"\n", (body + "\n" + body.replace(".kernel vt", ".kernel vt2")).encode()):
        res = P.decompile_listing(listing)
        ref = O.decompile(listing)
        assert res.combined == ref.combined
        assert [(k.failed, k.structured, k.fallback_count) for k in res.kernels] == \
               [(k.failed, k.structured, k.fallback_count) for k in ref.kernels]
        assert [(d.severity, d.line, d.message.encode()) for d in res.diagnostics] == \
               [(d.severity, d.line, d.message) for d in ref.diagnostics]


def test_streamed_generation_matches_reference_hashes():
    """ocldec_b200_session_run_generated (the C5 streaming path: generate a
    chunk on the device, decompile it, next chunk) forced into several
    chunks: the sampled kernels' source hashes equal the reference's, and the
    totals equal a resident run of the same corpus."""
    s = P.Session(0)
    try:
        for cfg, n, stride in (("C5", 40, 3), ("C3", 3000, 97)):
            st, hs, ls = s.run_generated(cfg, n, seed=SEEDS[cfg], k0=11, chunk_bytes=2 << 20 if cfg == "C5" else 1 << 18,
                                         sample_stride=stride)
            assert st["chunks"] > 2 and st["kernels"] == n and st["failed"] == 0
            ks = [k for k in range(11, 11 + n) if k % stride == 0]
            parts = [O.generate_corpus(cfg, 1, seed=SEEDS[cfg], k0=k) for k in ks]
            listing = b"".join(p[0] for p in parts)
            offs = np.cumsum([0] + [len(p[0]) for p in parts]).astype(np.uint64)
            _, _, rh, rl = O.decompile_batch(listing, offs, os.cpu_count() or 1, want_hashes=True)
            assert list(hs) == list(rh) and list(ls) == list(rl)
            # totals equal the whole-corpus run
            host, _, ni = P.generate_corpus(cfg, n, seed=SEEDS[cfg], k0=11)
            assert st["instructions"] == ni and st["in_bytes"] == len(host)
            # each chunk's combined output, joined by combined_source's "\n"
            assert st["out_bytes"] + st["chunks"] - 1 == len(P.decompile_listing(host).combined)
    finally:
        s.close()


def test_wide_lowering_option_matches_reference():
    """OCLDEC_B200_WIDE_LOWER=1 (k_lower_wide: long kernels lowered by the whole
    warp, lane-parallel merge_join / collect_delta) gives the reference's
    bytes on a C5 sample."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.');"
        "import paper_2107_07809_b200 as P; from oracle import oracle as O;"
        "parts = [O.generate_corpus('C5', 1, seed=0x210707809C5, k0=k)[0] for k in range(0, 1000000, 41667)];"
        "listing = b''.join(parts);"
        "res = P.decompile_listing(listing);"
        "offs = np.cumsum([0] + [len(p) for p in parts]).astype(np.uint64);"
        "ref = O.decompile_par(listing, offs[:-1]);"
        "assert res.combined == ref.combined;"
        "print('ok', len(parts))")
    env = dict(os.environ, OCLDEC_B200_WIDE_LOWER="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0 and "ok" in p.stdout, p.stderr[-2000:]


def test_c5_chunk_on_two_wave_streams():
    """A chunk of long C5 kernels large enough (>= 1024 kernels) for the two
    wave streams the session uses on long-kernel chunks: the combined output,
    flags and diagnostics equal the reference's, with the streams on (the
    default for such chunks) and forced off."""
    import subprocess
    import sys
    listing, offs, _ = O.generate_corpus("C5", 1100, seed=SEEDS["C5"], k0=500_000)
    ref = O.decompile_par(listing, [int(x) for x in offs[:-1]], nthreads=min(16, os.cpu_count() or 1))
    res = P.decompile_listing(listing)
    assert res.combined == ref.combined
    assert [(k.failed, k.structured, k.fallback_count) for k in res.kernels] == \
           [(k.failed, k.structured, k.fallback_count) for k in ref.kernels]
    # the same listing with the second stream disabled (a fresh process: the
    # mode is read when a session is created)
    code = ("import sys, hashlib; sys.path.insert(0, %r); import paper_2107_07809_b200 as P; "
            "from oracle import oracle as O; "
            "l, _, _ = O.generate_corpus('C5', 1100, seed=%d, k0=500000); "
            "print(hashlib.sha256(P.decompile_listing(l).combined).hexdigest())"
            % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))), SEEDS["C5"]))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900,
                         env=dict(os.environ, OCLDEC_B200_TWO_STREAMS="0"))
    import hashlib
    assert out.stdout.strip() == hashlib.sha256(ref.combined).hexdigest(), out.stderr[-2000:]
