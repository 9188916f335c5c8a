"""Multi-GPU sharding of a listing by kernel.

Kernels are independent units (decompiler.cpp:55-101), so a corpus shards
into contiguous kernel ranges balanced by input bytes, one range per rank,
with no data-path collective.  The only exchange is one all_gather of a
4 x int64 tuple per rank — {out_bytes, lines, split_error_line, kernels} —
from which every rank derives what combined_source (decompiler.cpp:105-115)
needs across shards:
  * its byte offset in the combined output (a "\\n" separates non-empty
    sources, so empty shards contribute nothing),
  * its listing-global line base (diagnostic line numbers),
  * the global split error (a split_kernels ParseError anywhere voids the
    whole result, decompiler.cpp:120-125).
The text itself is then written by each rank at its offset (a pinned host
buffer or a file); nothing but the tuple crosses NVLink.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

import numpy as np


def shard_ranges(offsets: Sequence[int], world: int) -> List[tuple]:
    """Contiguous kernel ranges [k0, k1) balanced by bytes.  offsets holds
    nkernels+1 byte offsets of the kernel sections."""
    offs = np.asarray(offsets, dtype=np.int64)
    nk = len(offs) - 1
    total = int(offs[-1] - offs[0])
    bounds = [0]
    for r in range(1, world):
        target = offs[0] + total * r // world
        k = int(np.searchsorted(offs, target, side="left"))
        k = max(bounds[-1], min(k, nk))
        bounds.append(k)
    bounds.append(nk)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


@dataclass
class ShardPlacement:
    out_offset: int      # where this rank's text starts in the combined output
    leading_newline: bool  # write "\n" at out_offset - 1
    line_base: int       # listing-global line number of this shard's first line, minus 1
    total_bytes: int     # combined output length
    split_error_line: int  # > 0: the whole result is void (zero kernels)
    kernels_before: int


def place(tuples: np.ndarray, rank: int) -> ShardPlacement:
    """tuples: [world, 4] int64 rows (out_bytes, lines, split_error_line_local, kernels)."""
    t = np.asarray(tuples, dtype=np.int64)
    world = t.shape[0]
    lines_before = np.concatenate([[0], np.cumsum(t[:, 1])])
    err = 0
    for r in range(world):
        if t[r, 2] > 0:
            err = int(lines_before[r] + t[r, 2])
            break
    contrib = np.where(t[:, 0] > 0, t[:, 0] + 1, 0)
    before = int(contrib[:rank].sum())
    total = int(contrib.sum()) - (1 if contrib.sum() > 0 else 0)
    if err:
        return ShardPlacement(0, False, int(lines_before[rank]), 0, err, int(t[:rank, 3].sum()))
    return ShardPlacement(before, bool(before > 0 and t[rank, 0] > 0), int(lines_before[rank]), total, 0,
                          int(t[:rank, 3].sum()))


def exchange(out_bytes: int, lines: int, split_error_line: int, kernels: int, device=None) -> np.ndarray:
    """The single collective: all_gather of the per-rank tuple (NCCL on GPUs,
    gloo on CPU).  Returns the [world, 4] table."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    mine = torch.tensor([out_bytes, lines, split_error_line, kernels], dtype=torch.int64, device=device)
    out = torch.empty(world * 4, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, mine)
    return out.view(world, 4).cpu().numpy()


def assemble(parts: Sequence[bytes], tuples: np.ndarray) -> bytes:
    """Host-side assembly of the combined output from per-rank texts at their
    placements (what rank 0 / a file writer does)."""
    world = len(parts)
    p0 = place(tuples, 0)
    if p0.split_error_line:
        return b""
    buf = bytearray(p0.total_bytes)
    for r in range(world):
        pl = place(tuples, r)
        if pl.leading_newline:
            buf[pl.out_offset - 1] = 0x0A
        buf[pl.out_offset:pl.out_offset + len(parts[r])] = parts[r]
    return bytes(buf)
