"""World-size-2 gloo test of the multi-GPU host logic (dist.py): shards are
contiguous kernel ranges balanced by bytes; the one all_gather of the
per-rank tuple yields placements whose assembly equals the unsharded
combined_source.  Per-shard texts come from the oracle (CPU) here; on the
GPU box the same code runs over NCCL with GPU shards."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2107_07809_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, listing, offsets, ranges, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("GLOO_SOCKET_IFNAME", "lo")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k0, k1 = ranges[rank]
    part = listing[int(offsets[k0]):int(offsets[k1])]
    r = O.decompile(part) if part else O.RefResult()
    lines = part.count(b"\n")
    err = r.diagnostics[0].line if (r.diagnostics and not r.kernels and part) else 0
    table = D.exchange(len(r.combined), lines, err, len(r.kernels))
    pl = D.place(table, rank)
    q.put((rank, r.combined, table.tolist(), pl.out_offset, pl.line_base))
    dist.destroy_process_group()


@pytest.mark.skipif(not O.available(), reason="oracle not built")
@pytest.mark.parametrize("with_error", [False, True])
def test_two_rank_exchange_matches_unsharded(with_error):
    import paper_2107_07809_b200 as P
    listing, offs, _ = P.generate_corpus("C3", 24, seed=21, stress=True)
    offs = [int(x) for x in offs]
    if with_error:
        # a nameless .kernel in the second half voids the whole listing
        k = 18
        listing = listing[:offs[k]] + b".kernel\n" + listing[offs[k]:]
        offs = offs[:k + 1] + [o + 8 for o in offs[k + 1:]]
        offs[k] = offs[k]  # the bad line belongs to kernel k-1's section
    ranges = D.shard_ranges(offs, 2)
    assert ranges[0][0] == 0 and ranges[-1][1] == 24 and ranges[0][1] == ranges[1][0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, listing, offs, ranges, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    table = np.array(got[0][2])
    parts = [g[1] for g in got]
    whole = O.decompile(listing)
    assert D.assemble(parts, table) == whole.combined
    if with_error:
        assert whole.combined == b"" and D.place(table, 0).split_error_line == whole.diagnostics[0].line
    else:
        assert got[1][4] == listing[:offs[ranges[1][0]]].count(b"\n")


def test_shard_ranges_balanced():
    offs = np.cumsum([0] + [100] * 10 + [1000] * 2)
    r = D.shard_ranges(offs, 3)
    assert r[0][0] == 0 and r[-1][1] == 12
    assert all(a <= b for a, b in r)


def test_place_separators():
    t = np.array([[10, 5, 0, 2], [0, 3, 0, 1], [7, 4, 0, 1]])
    assert D.place(t, 0).out_offset == 0
    assert D.place(t, 2).out_offset == 11 and D.place(t, 2).leading_newline
    assert D.place(t, 2).total_bytes == 18
    assert D.assemble([b"a" * 10, b"", b"b" * 7], t) == b"a" * 10 + b"\n" + b"b" * 7
