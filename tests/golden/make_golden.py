"""Regenerates the golden fixtures in tests/golden/ from the reference.

Run in the build container (needs /root/reference and `make -C oracle`):
    python tests/golden/make_golden.py

Sources of truth:
  * copy.asm / copy.cl       — the reference's own CLI golden pair
                               (proj/tests/data, cli_roundtrip.cmake:10-27)
  * corpus.jsonl             — the reference's 26-kernel corpus
                               (proj/tests/support/corpus.cpp:44-664) with the
                               oracle's outputs
  * nests.jsonl              — make_nest(seed) listings (nestgen.cpp:219-243)
  * edge.jsonl               — hand-written edge cases (split errors, failed
                               kernels, comments, CRLF, options)
  * gen.json                 — oracle output hashes for synthetic corpora
"""
import hashlib
import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

REF_DATA = "/root/reference/proj/tests/data"


def ref_record(listing: bytes, **kw):
    r = O.decompile(listing, **kw)
    return {
        "combined": r.combined.decode("utf-8", "surrogateescape"),
        "kernels": [{"name": k.name.decode(), "source": k.source.decode("utf-8", "surrogateescape"),
                     "failed": k.failed, "structured": k.structured, "fallbacks": k.fallback_count}
                    for k in r.kernels],
        "diagnostics": [[d.severity, d.line, d.message.decode("utf-8", "surrogateescape")]
                        for d in r.diagnostics],
    }


EDGE = [
    ("empty", b"", {}),
    ("preamble_only", b".amdcl2\n.gpu Fiji\n# nothing here\n", {}),
    ("text_before_kernel", b".text\n.kernel k\n  .text\n  s_endpgm\n", {}),
    ("config_before_kernel", b"  .config\n.kernel k\n  .text\n  s_endpgm\n", {}),
    ("nameless_kernel", b".kernel k\n .text\n s_endpgm\n.kernel # no name\n", {}),
    ("no_text", b".kernel k\n  .config\n  .dims x\n", {}),
    ("crlf", b".kernel k\r\n  .config\r\n    .dims x\r\n    .useargs\r\n"
             b"    .arg out, \"uint*\", uint*, global\r\n  .text\r\n"
             b"    s_load_dwordx2 s[0:1], s[4:5], 0x0\r\n    s_waitcnt lgkmcnt(0)\r\n"
             b"    v_mov_b32 v1, s0\r\n    v_mov_b32 v2, s1\r\n    flat_store_dword v[1:2], v0\r\n"
             b"    s_endpgm\r\n", {}),
    ("comments", b"; header\n.kernel k /* c */ # x\n  .config\n    .dims x ; y\n  .text\n"
                 b"  v_mov_b32 v1, /* mid */ 5 # tail\n  v_mov_b32 v2, v1 /* unterminated\n"
                 b"  flat_store_dword v[3:4], v1 ; t\n  s_endpgm\n", {}),
    ("trailing_labels", b".kernel k\n  .text\n  s_cmp_eq_u32 s2, 0\n  s_cbranch_scc1 L_end\n"
                        b"  v_mov_b32 v1, 1\nL_end:\nL_other: \n", {}),
    ("undefined_label", b".kernel k\n  .text\n  s_branch L_nowhere\n  s_endpgm\n", {}),
    ("unsupported_cbranch", b".kernel k\n  .text\n  s_cbranch_cdbgsys L\nL:\n  s_endpgm\n", {}),
    ("cbranch_at_end", b".kernel k\n  .text\nL:\n  s_cbranch_scc0 L\n", {}),
    ("branch_no_label", b".kernel k\n  .text\n  s_branch 12\n  s_endpgm\n", {}),
    ("bad_register", b".kernel k\n  .text\n  v_mov_b32 v1, s[5:3]\n  v_mov_b32 v2, v[1:300]\n"
                     b"  v_mov_b32 v3, s-1\n  s_mov_b32 s1, s[2\n  s_endpgm\n", {}),
    ("two_kernels_one_failed", b".kernel a\n  .text\n  s_branch L_x\n.kernel b\n  .text\n  v_mov_b32 v1, 7\n"
                               b"  flat_store_dword v[2:3], v1\n  s_endpgm\n", {}),
    ("only_kernel", b".kernel a\n  .text\n  flat_store_dword v[2:3], v1\n  s_endpgm\n"
                    b".kernel b\n  .text\n  flat_store_dword v[4:5], v1\n  s_endpgm\n", {"only_kernel": b"b"}),
    ("fold_local_size", b".kernel k\n  .config\n    .dims xy\n    .cws 64, 4, 1\n    .useargs\n"
                        b"    .arg out, \"uint*\", uint*, global\n  .text\n"
                        b"  s_load_dwordx2 s[0:1], s[4:5], 0x0\n  s_mul_i32 s9, s6, 64\n"
                        b"  s_mul_i32 s10, s7, 4\n  v_mov_b32 v3, s9\n  v_mov_b32 v4, s10\n"
                        b"  v_mov_b32 v5, s0\n  v_mov_b32 v6, s1\n  flat_store_dword v[5:6], v3\n"
                        b"  flat_store_dword v[5:6], v4\n  s_endpgm\n", {"fold_local_size": True}),
    ("num_groups", b".kernel k\n  .config\n    .dims x\n    .cws 64\n    .useargs\n  .text\n"
                   b"  s_load_dword s2, s[4:5], 0xc\n  s_lshr_b32 s3, s2, 6\n  v_mov_b32 v1, s3\n"
                   b"  flat_store_dword v[2:3], v1\n  s_endpgm\n", {}),
    ("dims_errors", b".kernel k\n  .config\n    .dims q\n    .cws 0, 2\n    .cws 1,2,3,4\n    .sgprsnum x\n"
                    b"    .arg only_two, \"int\"\n    .arg p, \"weird\", weird\n    .foo bar\n  .text\n"
                    b"  v_mov_b32 v1, 3\n  flat_store_dword v[2:3], v1\n  s_endpgm\n", {}),
    ("mask_multi_join", b".kernel k\n  .text\n  v_cmp_lt_u32 vcc, v0, 4\n  s_and_saveexec_b64 s[10:11], vcc\n"
                        b"  s_cbranch_scc1 L_a\n  v_mov_b32 v1, 1\n  s_or_b64 exec, exec, s[10:11]\n  s_branch L_end\n"
                        b"L_a:\n  s_or_b64 exec, exec, s[10:11]\nL_end:\n  s_endpgm\n", {}),
    ("exec_branch_goto", b".kernel k\n  .text\nL_top:\n  v_cmp_lt_u32 vcc, v0, 4\n  s_cbranch_execz L_top\n"
                         b"  s_cbranch_vccnz L_top\n  s_endpgm\n", {}),
    ("sixty_four_bit", b".kernel k\n  .config\n    .dims x\n    .useargs\n"
                       b"    .arg _.global_offset_0, \"size_t\", long\n    .arg a, \"long*\", long*, global\n"
                       b"    .arg b, \"ulong\", ulong\n  .text\n"
                       b"  s_load_dwordx4 s[0:3], s[4:5], 0x8\n  s_load_dwordx2 s[8:9], s[4:5], 0x10\n"
                       b"  s_mov_b64 s[12:13], s[0:1]\n  s_and_b64 s[14:15], s[2:3], s[8:9]\n"
                       b"  s_lshl_b64 s[16:17], s[14:15], 3\n  v_mov_b32 v1, s12\n  v_mov_b32 v2, s13\n"
                       b"  v_mov_b32 v3, s16\n  v_mov_b32 v4, s17\n  flat_store_dwordx2 v[1:2], v[3:4]\n"
                       b"  flat_load_dwordx2 v[5:6], v[1:2]\n  flat_store_dwordx2 v[1:2], v[5:6]\n  s_endpgm\n", {}),
]

GEN = [  # (shape, stress, seed, count)
    (1, 0, 1, 64), (2, 0, 0x210707809C2, 64), (3, 0, 0x210707809C3, 256), (4, 0, 0x210707809C4, 64),
    (1, 1, 5, 64), (2, 1, 6, 64), (3, 1, 7, 256), (4, 1, 8, 64), (5, 0, 0x210707809C5, 2),
]


def main():
    os.makedirs(HERE, exist_ok=True)
    shutil.copy(os.path.join(REF_DATA, "copy.asm"), os.path.join(HERE, "copy.asm"))
    shutil.copy(os.path.join(REF_DATA, "copy.cl"), os.path.join(HERE, "copy.cl"))
    with open(os.path.join(HERE, "corpus.jsonl"), "w") as f:
        for name, listing, comparable, fb in O.corpus():
            rec = {"name": name.decode(), "listing": listing.decode(), "comparable": comparable,
                   "expected_fallbacks": fb}
            rec.update(ref_record(listing))
            f.write(json.dumps(rec) + "\n")
    with open(os.path.join(HERE, "nests.jsonl"), "w") as f:
        for seed in range(1, 201):
            listing = O.make_nest(seed)
            rec = {"seed": seed, "listing": listing.decode()}
            rec.update(ref_record(listing))
            f.write(json.dumps(rec) + "\n")
    with open(os.path.join(HERE, "edge.jsonl"), "w") as f:
        for name, listing, kw in EDGE:
            rec = {"name": name, "listing": listing.decode("utf-8", "surrogateescape"),
                   "fold_local_size": bool(kw.get("fold_local_size", False)),
                   "only_kernel": kw["only_kernel"].decode() if "only_kernel" in kw else None}
            rec.update(ref_record(listing, **kw))
            f.write(json.dumps(rec) + "\n")
    import paper_2107_07809_b200 as P
    gens = []
    for shape, stress, seed, count in GEN:
        listing, offs, ni = P.generate_corpus(shape, count, seed=seed, stress=bool(stress))
        ref = O.decompile(listing)
        gens.append({"shape": shape, "stress": stress, "seed": seed, "count": count,
                     "listing_sha256": hashlib.sha256(listing).hexdigest(), "instructions": ni,
                     "combined_sha256": hashlib.sha256(ref.combined).hexdigest(),
                     "combined_len": len(ref.combined),
                     "failed": sum(k.failed for k in ref.kernels),
                     "goto_form": sum((not k.structured) and (not k.failed) for k in ref.kernels),
                     "fallbacks": sum(k.fallback_count for k in ref.kernels)})
    with open(os.path.join(HERE, "gen.json"), "w") as f:
        json.dump(gens, f, indent=1)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
