"""Parity at BASELINE.json's full single-GPU size (C4: 1,000,000 kernels,
~5.5e8 instructions, ~19 GB of listing): the bench's own workload, generated
on the device, decompiled in the bench's chunks.  The reference cannot run a
corpus this size inside a test, so the check is:

- a deterministic sample of kernels (every 997th, regenerated on the host
  from the same counter-based seed) is byte-identical to the reference's
  output for that kernel, with the same flags;
- size-independent properties of the whole run: every kernel produced,
  instruction count equal to the generator's, no failures, each source
  starts with "__kernel void" and the spans tile combined_source with one
  "\\n" between sources;
- a second run over the same input gives the same bytes (hash)."""
import hashlib

import numpy as np
import pytest

import paper_2107_07809_b200 as P
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.available(), reason="oracle not built")]

SEED_C4 = 0x210707809C4  # bench.py SEEDS["C4"]
NK = 1_000_000


def _chunks(offs, target=5 << 29):
    starts, nxt = [0], target
    for o in offs[1:-1]:
        if o >= nxt:
            starts.append(int(o))
            nxt = int(o) + target
    return starts


def _out_hash(s):
    """sha256 of the device output, copied out 256 MB at a time."""
    p, n = s.output()
    h = hashlib.sha256()
    buf = np.zeros(256 << 20, dtype=np.uint8)
    for o in range(0, n, len(buf)):
        m = min(len(buf), n - o)
        P.copy(buf.ctypes.data, p + o, m)
        h.update(memoryview(buf)[:m])
    return h.hexdigest()


def test_c4_full_size():
    s = P.Session(0)
    try:
        d_buf, nbytes, d_offs, ni = s.generate("C4", NK, seed=SEED_C4)
        offs = np.zeros(NK + 1, dtype=np.uint64)
        P.copy(offs.ctypes.data, d_offs, (NK + 1) * 8)
        assert int(offs[-1]) == nbytes and nbytes > 16e9
        s.run(d_buf, nbytes, _chunks(offs))
        st = s.stats()
        assert st["kernels"] == NK and st["instructions"] == ni and st["failed"] == 0
        koff, klen, kfl, kfb = s.kernels()
        p_out, n_out = s.output()
        # spans tile the output: sources back to back with one "\n" between
        assert np.all(klen > 0)
        assert np.array_equal(koff[1:], koff[:-1] + klen[:-1] + 1)
        assert int(koff[-1] + klen[-1]) == n_out
        # every 997th kernel against the reference
        sample = list(range(0, NK, 997)) + [NK - 1]
        for k in sample:
            src = np.zeros(int(klen[k]), dtype=np.uint8)
            P.copy(src.ctypes.data, p_out + int(koff[k]), int(klen[k]))
            listing, _, _ = P.generate_corpus("C4", 1, seed=SEED_C4, k0=k)
            ref = O.decompile(listing)
            assert src.tobytes() == ref.combined, k
            assert bool(kfl[k] & 2) == ref.kernels[0].structured and kfb[k] == ref.kernels[0].fallback_count
        # whole-output hash, then a second run over the same input
        h1 = _out_hash(s)
        s.run(d_buf, nbytes, _chunks(offs))
        assert _out_hash(s) == h1
    finally:
        s.close()
