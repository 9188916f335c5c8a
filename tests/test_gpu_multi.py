"""Multi-device product path on the GPU.

1. ocldec_b200_decompile_multi: the C-ABI call that shards a listing by
   kernel sections across devices, one host thread per shard, places each
   shard's text at its scanned offset and shifts its diagnostic lines.  On the
   one-GPU box the shards are several sessions on cuda:0 (devices [0, 0, ...]);
   the code path is the same as on 8 GPUs.  Checked against the single-device
   call and the reference.
2. Two ranks (processes) on cuda:0 exchanging their tuples over gloo
   (dist.exchange, the all_gather bench.py runs over NCCL): the assembled
   output equals the reference's combined_source of the whole listing.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_2107_07809_b200 as P
from oracle import oracle as O
from paper_2107_07809_b200 import dist as D

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.available(), reason="oracle not built")]


def _same(a, b):
    assert a.combined == b.combined
    assert [(k.name, k.source, k.failed, k.structured, k.fallback_count, k.instructions) for k in a.kernels] == \
           [(k.name, k.source, k.failed, k.structured, k.fallback_count, k.instructions) for k in b.kernels]
    assert [(d.severity, d.line, d.message) for d in a.diagnostics] == \
           [(d.severity, d.line, d.message) for d in b.diagnostics]


def _vs_ref(res, ref):
    assert res.combined == ref.combined
    assert [(k.failed, k.structured, k.fallback_count) for k in res.kernels] == \
           [(k.failed, k.structured, k.fallback_count) for k in ref.kernels]
    assert [(d.severity, d.line, d.message.encode("utf-8", "surrogateescape")) for d in res.diagnostics] == \
           [(d.severity, d.line, d.message) for d in ref.diagnostics]


@pytest.mark.parametrize("ndev", [2, 3, 8])
def test_multi_matches_single_and_reference(ndev):
    listing, _, _ = P.generate_corpus("C3", 400, seed=31, stress=True)
    listing = b"; preamble line ignored by split_kernels\n\n" + listing
    one = P.decompile_listing(listing)
    multi = P.decompile_listing(listing, devices=[0] * ndev)
    _same(multi, one)
    _vs_ref(multi, O.decompile(listing))


def test_multi_options_and_dumps():
    listing, _, _ = P.generate_corpus("C3", 60, seed=5, stress=True)
    names = [k.name for k in P.decompile_listing(listing).kernels]
    for opts in (P.DecompileOptions(only_kernel=names[45]), P.DecompileOptions(fold_local_size=True),
                 P.DecompileOptions(dump_cfg=True, dump_regions=True, record_reduction=True)):
        one = P.decompile_listing(listing, opts)
        multi = P.decompile_listing(listing, opts, devices=[0, 0, 0])
        _same(multi, one)
        assert [(k.cfg_dot, k.region_dumps) for k in multi.kernels] == \
               [(k.cfg_dot, k.region_dumps) for k in one.kernels]


def test_multi_split_error_in_a_later_shard():
    """A nameless .kernel anywhere voids the whole listing (decompiler.cpp:
    120-125): zero kernels and one error at its listing-global line."""
    listing, offs, _ = P.generate_corpus("C2", 40, seed=8)
    k = 33
    bad = listing[:int(offs[k])] + b".kernel\n" + listing[int(offs[k]):]
    multi = P.decompile_listing(bad, devices=[0, 0, 0, 0])
    ref = O.decompile(bad)
    assert not multi.kernels and multi.combined == b""
    assert [(d.severity, d.line, d.message.encode()) for d in multi.diagnostics] == \
           [(d.severity, d.line, d.message) for d in ref.diagnostics]


def test_multi_more_devices_than_kernels():
    listing = open(os.path.join(os.path.dirname(__file__), "golden", "copy.asm"), "rb").read()
    multi = P.decompile_listing(listing, devices=[0, 0, 0, 0])
    assert multi.combined == open(os.path.join(os.path.dirname(__file__), "golden", "copy.cl"), "rb").read()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, listing, offsets, ranges, q):
    import torch.distributed as dist
    import paper_2107_07809_b200 as P
    from paper_2107_07809_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k0, k1 = ranges[rank]
    part = listing[int(offsets[k0]):int(offsets[k1])] if rank else listing[:int(offsets[k1])]
    r = P.decompile_listing(part)  # the GPU path, this rank's shard
    err = r.diagnostics[0].line if (r.diagnostics and not r.kernels and part) else 0
    table = D.exchange(len(r.combined), part.count(b"\n"), err, len(r.kernels))
    pl = D.place(table, rank)
    diags = [(d.severity, d.line + pl.line_base if d.line else 0, d.message) for d in r.diagnostics]
    q.put((rank, r.combined, table.tolist(), diags))
    dist.destroy_process_group()


def test_two_gpu_ranks_gloo_assemble_to_reference():
    listing, offs, _ = P.generate_corpus("C3", 64, seed=44, stress=True)
    offs = [int(x) for x in offs]
    ranges = D.shard_ranges(offs, 2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, listing, offs, ranges, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    table = np.array(got[0][2])
    ref = O.decompile(listing)
    assert D.assemble([g[1] for g in got], table) == ref.combined
    assert got[0][3] + got[1][3] == [(d.severity, d.line, d.message.decode("utf-8", "surrogateescape"))
                                      for d in ref.diagnostics]


def test_cli_devices_flag(tmp_path):
    """The CLI's --devices shards through the same C-ABI call; the output file
    equals the reference's combined_source."""
    import subprocess
    cli = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2107_07809_b200",
                       "ocldec-b200")
    listing, _, _ = P.generate_corpus("C3", 120, seed=12)
    src = tmp_path / "k.asm"
    src.write_bytes(listing)
    p = subprocess.run([cli, str(src), "--devices", "0,0,0"], capture_output=True, timeout=300)
    assert p.returncode in (0, 1), p.stderr
    assert (tmp_path / "k.cl").read_bytes() == O.decompile(listing).combined


def test_multi_semantic_check_and_exports():
    """Sharded runs key each kernel's environments by its ordinal in the whole
    listing, so the semantic verdicts and trace hashes equal the one-device
    run's; the body and cfg exports also travel through the shards."""
    listing, _, _ = P.generate_corpus("C2", 300, seed=77, stress=True)
    opts = P.DecompileOptions(semantic_check=True, semantic_seed=0x5E3A171C, export_body=True)
    one = P.decompile_listing(listing, opts)
    multi = P.decompile_listing(listing, opts, devices=[0, 0, 0])
    _same(multi, one)
    assert [k.semantic for k in multi.kernels] == [k.semantic for k in one.kernels]
    assert [(k.body_text, k.cfg_text) for k in multi.kernels] == [(k.body_text, k.cfg_text) for k in one.kernels]
    assert sum(1 for k in one.kernels if k.cfg_text) >= 290
