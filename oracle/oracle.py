"""TEST INFRASTRUCTURE ONLY — the parity oracle, never the product path.

ctypes wrapper over ``oracle/_ref/libocldec_ref.so``: the unmodified reference
decompiler (``/root/reference/proj/core/src``) compiled by ``oracle/Makefile``.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module, and only as the checker or
the timed CPU arm.

Wrapped reference entry points:
  * ``ocldec::decompile_listing``        proj/core/src/decompiler.cpp:117-133
  * ``DecompileResult::combined_source`` proj/core/src/decompiler.cpp:105-115
  * ``ocldec_tests::corpus``             proj/tests/support/corpus.cpp:44-664
  * ``ocldec_tests::make_nest``          proj/tests/support/nestgen.cpp:219-243
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import List, Optional

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libocldec_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"oracle library missing: {LIB_PATH} (run `make -C oracle`)")
        L = ctypes.CDLL(LIB_PATH)
        L.ref_decompile.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_char_p,
                                    ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]
        L.ref_decompile.restype = ctypes.c_int
        L.ref_decompile_abi.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_char_p,
                                        ctypes.c_char_p, ctypes.c_size_t,
                                        ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]
        L.ref_decompile_abi.restype = ctypes.c_int
        L.ref_decompile_ex.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_char_p,
                                       ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]
        L.ref_decompile_ex.restype = ctypes.c_int
        L.ref_free.argtypes = [ctypes.c_void_p]
        L.ref_decompile_batch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.POINTER(ctypes.c_uint64)]
        L.ref_decompile_batch.restype = ctypes.c_double
        L.ref_corpus_count.restype = ctypes.c_int
        L.ref_corpus_get.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                                     ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.ref_make_nest.argtypes = [ctypes.c_uint64, ctypes.POINTER(ctypes.c_int)]
        L.ref_make_nest.restype = ctypes.c_void_p
        L.ref_gen_host.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                   ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
        L.ref_gen_host.restype = ctypes.c_int64
        L.ref_decompile_par.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                        ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]
        L.ref_decompile_par.restype = ctypes.c_int
        L.ref_semcheck.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_void_p,
                                   ctypes.c_size_t]
        L.ref_semcheck.restype = ctypes.c_int64
        L.ref_semcheck_at.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_void_p, ctypes.c_size_t]
        L.ref_semcheck_at.restype = ctypes.c_int64
        _lib = L
    return _lib


@dataclass
class RefKernel:
    name: bytes
    source: bytes
    failed: bool
    structured: bool
    fallback_count: int
    cfg_dot: bytes = b""                                   # DecompiledKernel::cfg_dot (dump_cfg)
    region_dumps: List[bytes] = field(default_factory=list)  # ReduceResult::dumps (dump_regions)
    reduction: bytes = b""  # merges + root/residue as text (ref_driver.cpp serialization)


@dataclass
class RefDiag:
    severity: int  # 0 note, 1 warning, 2 error (diagnostics.hpp:16)
    line: int
    message: bytes


@dataclass
class RefResult:
    kernels: List[RefKernel] = field(default_factory=list)
    diagnostics: List[RefDiag] = field(default_factory=list)
    combined: bytes = b""
    abi_diagnostics: List[RefDiag] = field(default_factory=list)  # parse_abi_overrides


def _take(ptr: int, n: int) -> bytes:
    return ctypes.string_at(ptr, n)


def _parse(blob: bytes) -> "RefResult":
    res = RefResult()
    pos = 0
    while pos < len(blob):
        nl = blob.index(b"\n", pos)
        head = blob[pos:nl].split()
        pos = nl + 1
        if head[0] == b"K":
            failed, structured, fb, nlen, slen = (int(x) for x in head[1:])
            name = blob[pos:pos + nlen]
            pos += nlen
            src = blob[pos:pos + slen]
            pos += slen
            res.kernels.append(RefKernel(name, src, bool(failed), bool(structured), fb))
        elif head[0] == b"D":
            sev, line, mlen = (int(x) for x in head[1:])
            res.diagnostics.append(RefDiag(sev, line, blob[pos:pos + mlen]))
            pos += mlen
        elif head[0] == b"A":
            sev, line, mlen = (int(x) for x in head[1:])
            res.abi_diagnostics.append(RefDiag(sev, line, blob[pos:pos + mlen]))
            pos += mlen
        elif head[0] == b"G":
            ki, glen = int(head[1]), int(head[2])
            res.kernels[ki].cfg_dot = blob[pos:pos + glen]
            pos += glen
        elif head[0] == b"R":
            ki, step, rlen = int(head[1]), int(head[2]), int(head[3])
            assert step == len(res.kernels[ki].region_dumps)
            res.kernels[ki].region_dumps.append(blob[pos:pos + rlen])
            pos += rlen
        elif head[0] == b"M":
            ki, mlen = int(head[1]), int(head[2])
            res.kernels[ki].reduction = blob[pos:pos + mlen]
            pos += mlen
        elif head[0] == b"C":
            clen = int(head[1])
            res.combined = blob[pos:pos + clen]
            pos += clen
        else:  # pragma: no cover
            raise ValueError(f"bad oracle record {head!r}")
    return res


def decompile(listing: bytes, fold_local_size: bool = False, only_kernel: Optional[bytes] = None,
              abi_map: Optional[bytes] = None, dump_cfg: bool = False,
              dump_regions: bool = False, reduction: bool = False) -> RefResult:
    if isinstance(listing, str):
        listing = listing.encode()
    L = lib()
    out = ctypes.c_void_p()
    n = ctypes.c_size_t()
    if isinstance(abi_map, str):
        abi_map = abi_map.encode()
    dumps = int(dump_cfg) | (2 if dump_regions else 0) | (4 if reduction else 0)
    if dumps:
        L.ref_decompile_ex(listing, len(listing), int(fold_local_size), only_kernel, abi_map,
                           len(abi_map) if abi_map is not None else 0, dumps, ctypes.byref(out), ctypes.byref(n))
    elif abi_map is None:
        L.ref_decompile(listing, len(listing), int(fold_local_size), only_kernel, ctypes.byref(out), ctypes.byref(n))
    else:
        L.ref_decompile_abi(listing, len(listing), int(fold_local_size), only_kernel, abi_map, len(abi_map),
                            ctypes.byref(out), ctypes.byref(n))
    blob = _take(out.value, n.value)
    L.ref_free(out)
    return _parse(blob)


def decompile_par(listing: bytes, kernel_starts, nthreads: int = 0, per: int = 64,
                  fold_local_size: bool = False) -> RefResult:
    """decompile_listing of the whole listing, computed in parallel over slices
    of `per` kernels (ref_driver.cpp ref_decompile_par): same kernels,
    diagnostics (listing-global lines) and combined_source as decompile()."""
    import numpy as np
    L = lib()
    ks = np.ascontiguousarray(kernel_starts, dtype=np.uint64)
    out = ctypes.c_void_p()
    n = ctypes.c_size_t()
    L.ref_decompile_par(listing, len(listing), ks.ctypes.data, len(ks), per, nthreads or (os.cpu_count() or 1),
                        int(fold_local_size), ctypes.byref(out), ctypes.byref(n))
    blob = _take(out.value, n.value)
    L.ref_free(out)
    return _parse(blob)


def semcheck(listing: bytes, seed: int, cap: int = 1 << 20, nthreads: int = 1):
    """The reference's interpret_asm / evaluate_decompiled (oracle.cpp:620-842)
    per kernel over the semantic check's 8 environments (od_semenv.cuh):
    [(status, envs, hash_asm, hash_body)], statuses as the device check's.
    nthreads > 1 cuts the listing at ".kernel" lines into slices checked on
    that many threads (each slice keyed by its kernels' ordinals in the whole
    listing); for listings without a preamble or commented-out sections."""
    import numpy as np
    L = lib()
    if nthreads <= 1:
        out = np.zeros(4 * cap, dtype=np.uint64)
        n = L.ref_semcheck(listing, len(listing), seed, out.ctypes.data, cap)
        return [tuple(int(x) for x in out[4 * k:4 * k + 4]) for k in range(min(n, cap))]
    starts = [0] if listing.startswith(b".kernel") else []
    pos = listing.find(b"\n.kernel")
    while pos >= 0:
        starts.append(pos + 1)
        pos = listing.find(b"\n.kernel", pos + 1)
    if not starts or starts[0] != 0:
        raise ValueError("semcheck(nthreads > 1) needs a listing that starts with .kernel")
    per = max(1, (len(starts) + 4 * nthreads - 1) // (4 * nthreads))
    slices = []
    for i in range(0, len(starts), per):
        b = starts[i]
        e = starts[i + per] if i + per < len(starts) else len(listing)
        slices.append((i, listing[b:e], min(per, len(starts) - i)))

    def run(sl):
        kb, text, nk = sl
        out = np.zeros(4 * nk, dtype=np.uint64)
        n = L.ref_semcheck_at(text, len(text), seed, kb, out.ctypes.data, nk)
        return [tuple(int(x) for x in out[4 * k:4 * k + 4]) for k in range(min(n, nk))]

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(nthreads) as ex:
        parts = list(ex.map(run, slices))
    return [x for p in parts for x in p][:cap]


SHAPES = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5}


def generate_corpus(shape, count: int, seed: int = 1, k0: int = 0, stress: bool = False, nthreads: int = 0):
    """The synthetic corpus (od_gen.cuh, host build linked into the oracle
    library): byte-identical to paper_2107_07809_b200.generate_corpus, without
    loading the product library.  Returns (listing, offsets[count+1], instrs)."""
    import numpy as np
    L = lib()
    shape = SHAPES.get(shape, shape) if isinstance(shape, str) else shape
    nt = nthreads or min(16, os.cpu_count() or 1)
    offs = np.zeros(count + 1, dtype=np.uint64)
    ni = ctypes.c_uint64()
    need = L.ref_gen_host(shape, int(stress), seed, k0, count, None, 0, offs.ctypes.data, ctypes.byref(ni), nt)
    buf = ctypes.create_string_buffer(int(need) + 1)
    n = L.ref_gen_host(shape, int(stress), seed, k0, count, ctypes.cast(buf, ctypes.c_void_p), need + 1,
                       offs.ctypes.data, ctypes.byref(ni), nt)
    if n < 0:
        raise RuntimeError("oracle corpus generation failed")
    return buf.raw[:n], offs, int(ni.value)


def corpus():
    """[(name, listing, comparable, expected_fallbacks)] — corpus.cpp:44-664."""
    L = lib()
    out = []
    for i in range(L.ref_corpus_count()):
        nm, ls = ctypes.c_void_p(), ctypes.c_void_p()
        cmp_, fb = ctypes.c_int(), ctypes.c_int()
        L.ref_corpus_get(i, ctypes.byref(nm), ctypes.byref(ls), ctypes.byref(cmp_), ctypes.byref(fb))
        out.append((ctypes.string_at(nm.value), ctypes.string_at(ls.value), bool(cmp_.value), fb.value))
        L.ref_free(nm)
        L.ref_free(ls)
    return out


def make_nest(seed: int) -> bytes:
    L = lib()
    c = ctypes.c_int()
    p = L.ref_make_nest(seed, ctypes.byref(c))
    s = ctypes.string_at(p)
    L.ref_free(p)
    return s


def decompile_batch(corpus_bytes: bytes, offsets, nthreads: int, want_hashes: bool = False):
    """Times the reference on per-kernel listings corpus[offsets[k]:offsets[k+1]].

    Returns (seconds, instructions, hashes|None, lengths|None)."""
    import numpy as np
    L = lib()
    offs = np.ascontiguousarray(offsets, dtype=np.uint64)
    nk = len(offs) - 1
    buf = ctypes.create_string_buffer(corpus_bytes, len(corpus_bytes)) if isinstance(corpus_bytes, bytes) else corpus_bytes
    hashes = np.zeros(nk, dtype=np.uint64) if want_hashes else None
    lens = np.zeros(nk, dtype=np.uint64) if want_hashes else None
    ninstr = ctypes.c_uint64()
    secs = L.ref_decompile_batch(ctypes.cast(buf, ctypes.c_void_p), offs.ctypes.data, nk, nthreads,
                                 hashes.ctypes.data if hashes is not None else None,
                                 lens.ctypes.data if lens is not None else None,
                                 ctypes.byref(ninstr))
    return secs, ninstr.value, hashes, lens
