"""Diagnostics parity: DecompileResult::diagnostics —
severity, line and message text, in the order the reference's DiagnosticSink
records them (diagnostics.hpp:20-57; catalogue SURVEY A.4) — produced by the
sm_100a pipeline through the C ABI must equal the reference's on the same
listing: the committed fixtures (reference corpus, nests, edge listings) and
the live oracle on generated stress corpora (operand ParseErrors, bad config
directives, undefined labels, unsupported branches, mask warnings, goto form,
unreachable code)."""
import json
import os
import subprocess

import pytest

import paper_2107_07809_b200 as P
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
pytestmark = pytest.mark.gpu


def _jsonl(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [json.loads(line) for line in f]


def _ours(res):
    return [(d.severity, d.line, d.message.encode("utf-8", "surrogateescape")) for d in res.diagnostics]


def _fixture(diags):
    return [(s, l, m.encode("utf-8", "surrogateescape")) for s, l, m in diags]


def test_edge_fixture_diagnostics():
    for rec in _jsonl("edge.jsonl"):
        res = P.decompile_listing(rec["listing"].encode("utf-8", "surrogateescape"),
                                  P.DecompileOptions(fold_local_size=rec["fold_local_size"],
                                                     only_kernel=rec["only_kernel"]))
        assert _ours(res) == _fixture(rec["diagnostics"]), rec["name"]


def test_reference_corpus_diagnostics():
    for rec in _jsonl("corpus.jsonl"):
        res = P.decompile_listing(rec["listing"])
        assert _ours(res) == _fixture(rec["diagnostics"]), rec["name"]


def test_nest_diagnostics():
    for rec in _jsonl("nests.jsonl"):
        res = P.decompile_listing(rec["listing"])
        assert _ours(res) == _fixture(rec["diagnostics"]), rec["seed"]


@pytest.mark.skipif(not O.available(), reason="oracle not built")
@pytest.mark.parametrize("shape,stress,count", [("C1", 1, 400), ("C2", 1, 300), ("C3", 1, 1500),
                                                ("C3", 0, 1500), ("C4", 1, 300)])
def test_generated_diagnostics_vs_oracle(shape, stress, count):
    listing, _, _ = P.generate_corpus(shape, count, seed=4242 + count, stress=bool(stress))
    res = P.decompile_listing(listing)
    ref = O.decompile(listing)
    assert _ours(res) == [(d.severity, d.line, d.message) for d in ref.diagnostics]


@pytest.mark.skipif(not O.available(), reason="oracle not built")
def test_handwritten_diagnostics_vs_oracle():
    """Every message kind of the catalogue in one listing, plus options."""
    listing = (
        ".kernel a\n  .config\n  .dims xq\n  .cws 1, 2, 3, 4\n  .cws 64, -1\n  .sgprsnum x\n"
        "  .vgprsnum -3\n  .arg only_two, \"int\"\n  .arg p, \"foo*\", foo*\n  .text\n"
        "  v_mov_b32 v[0:1, v1\n  v_mov_b32 v2, s[2-3]\n  v_mov_b32 v2, s[3:2]\n  v_mov_b32 v2, v-1\n"
        "  v_mov_b32 v300, v1\n  s_mov_b32 s200, s1\n  s_load_dword s3, s[4:5], 0x999\n"
        "  v_addc_u32 v3, vcc, v1, v2, vcc\n  s_endpgm\n"
        ".kernel b\n  .text\n  s_branch L_nowhere\n  s_endpgm\n"
        ".kernel c\n  .text\n  s_cbranch_foo L1\nL1:\n  s_endpgm\n"
        ".kernel d\n  .text\n  s_cbranch_scc1 L2\nL2:\n  s_cbranch_scc0 L2\n"
        ".kernel e\n  .text\n  s_branch\n  s_endpgm\n"
        ".kernel f\n  .text\n  s_endpgm\n  v_mov_b32 v1, v2\n  s_endpgm\n"
        ".kernel g\n  .text\nL_loop:\n  s_add_u32 s9, s9, 1\n  s_cmp_lt_u32 s9, 8\n"
        "  s_cbranch_scc1 L_loop\n  s_endpgm\n"
    )
    res = P.decompile_listing(listing)
    ref = O.decompile(listing.encode())
    assert _ours(res) == [(d.severity, d.line, d.message) for d in ref.diagnostics]
    assert len(res.diagnostics) >= 12
    for fold in (False, True):
        for only in (None, "b", "zz"):
            r = P.decompile_listing(listing, P.DecompileOptions(fold_local_size=fold, only_kernel=only))
            f = O.decompile(listing.encode(), fold_local_size=fold,
                            only_kernel=only.encode() if only else None)
            assert _ours(r) == [(d.severity, d.line, d.message) for d in f.diagnostics], (fold, only)


@pytest.mark.skipif(not O.available(), reason="oracle not built")
def test_cli_prints_reference_diagnostics(tmp_path):
    cli = os.path.join(ROOT, "paper_2107_07809_b200", "ocldec-b200")
    if not os.path.exists(cli):
        pytest.skip("CLI not built")
    listing, _, _ = P.generate_corpus("C3", 300, seed=77, stress=True)
    inp = tmp_path / "s.asm"
    inp.write_bytes(listing)
    p = subprocess.run([cli, str(inp), "-o", str(tmp_path / "s.cl")], capture_output=True)
    ref = O.decompile(listing)
    want = b"".join(f"{inp}:{d.line}: {('note', 'warning', 'error')[d.severity]}: ".encode() + d.message + b"\n"
                    for d in ref.diagnostics)
    assert p.stderr == want
    assert (tmp_path / "s.cl").read_bytes() == ref.combined
    assert p.returncode == (1 if any(k.failed for k in ref.kernels) else 0)
