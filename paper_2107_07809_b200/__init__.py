"""ocldec-b200: B200-native batch decompiler of AMD GCN listings to OpenCL C.

Host-side mirror of the reference's front door (``ocldec::decompile_listing``,
/root/reference/proj/core/include/ocldec/decompiler.hpp:29-62): same names,
argument meaning and error behaviour.  Every call runs the sm_100a pipeline
through the C ABI in ``include/ocldec_b200.h``; there is no CPU path.

    >>> from paper_2107_07809_b200 import decompile_listing
    >>> res = decompile_listing(open("copy.asm").read())
    >>> print(res.combined_source())
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Union

from . import _lib

__all__ = ["DecompileOptions", "DecompiledKernel", "Reduction", "Diagnostic", "DecompileResult",
           "decompile_listing", "check_abi_map", "generate_corpus", "Session", "SHAPES"]

# Synthetic corpus shapes (BASELINE.json configs).
SHAPES = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5}


@dataclass
class DecompileOptions:
    """DecompileOptions (decompiler.hpp:29-35).  ``abi_map`` is the override
    file text the reference CLI's --abi-map reads (parse_abi_overrides,
    abi_model.cpp:109-153) standing for ``abi_overrides``."""
    fold_local_size: bool = False           # FoldOptions (sym_state.hpp:27-29)
    only_kernel: Optional[str] = None       # restrict to one kernel by name
    abi_map: Optional[Union[str, bytes]] = None
    dump_cfg: bool = False                  # DecompiledKernel.cfg_dot (to_dot, cfg.cpp:400-424)
    dump_regions: bool = False              # region_dumps (region_graph_dot, structurizer.cpp:669-688)
    record_reduction: bool = False          # DecompiledKernel.reduction (merges, root / residue)
    export_body: bool = False               # DecompiledKernel.body_text (LoweredBody, lower.hpp:20-41)
    semantic_check: bool = False            # DecompiledKernel.semantic (the batched semantic check)
    semantic_seed: int = 0x5E3A171C
    device: int = 0
    arena_bytes: int = 0                    # per-thread arena, 0 = default


@dataclass
class Diagnostic:
    """Diagnostic (diagnostics.hpp:20-27).  severity: 0 note, 1 warning, 2 error."""
    severity: int
    line: int
    message: str

    def render(self, file: str) -> str:
        sev = ("note", "warning", "error")[self.severity]
        return f"{file}:{self.line}: {sev}: {self.message}"


@dataclass
class Reduction:
    """ReduceResult's inspection part (structurizer.hpp:54-58, 98-104):
    merges as (kind, result, absorbed) with kind 1 Linear, 2 IfThen,
    3 IfElse; root when reduced, else the residue (region ids)."""
    merges: List[tuple] = field(default_factory=list)
    reduced: bool = False
    root: int = 0
    residue: List[int] = field(default_factory=list)
    text: str = ""

    @staticmethod
    def parse(text: str) -> "Reduction":
        r = Reduction(text=text)
        for line in text.splitlines():
            w = line.split()
            if w and w[0] == "merge":
                r.merges.append((int(w[1]), int(w[2]), [int(x) for x in w[3:]]))
            elif w and w[0] == "root":
                r.reduced, r.root = True, int(w[1])
            elif w and w[0] == "residue":
                r.residue = [int(x) for x in w[1:]]
        return r


@dataclass
class DecompiledKernel:
    """DecompiledKernel (decompiler.hpp:39-52): printed source and flags."""
    name: str
    source: str
    structured: bool
    failed: bool
    fallback_count: int
    instructions: int
    cfg_dot: str = ""                                        # when dump_cfg
    region_dumps: List[str] = field(default_factory=list)   # reduction.dumps when dump_regions
    reduction: Optional["Reduction"] = None                 # when record_reduction
    body_text: str = ""                                     # when export_body (od_lower.cuh body_text)
    cfg_text: str = ""                                      # when export_body: the flow graph (od_kernel.cuh cfg_text)
    semantic: Optional[tuple] = None  # when semantic_check: (status, envs, hash_asm, hash_body);
    # status 0 equal, 1 mismatch, 2 unsupported, 3 not compared (device room), 4 not run


@dataclass
class DecompileResult:
    """DecompileResult (decompiler.hpp:54-60)."""
    kernels: List[DecompiledKernel] = field(default_factory=list)
    diagnostics: List[Diagnostic] = field(default_factory=list)
    abi_diagnostics: List[Diagnostic] = field(default_factory=list)  # parse_abi_overrides' sink
    combined: bytes = b""
    device_ms: float = 0.0

    def combined_source(self) -> str:
        """decompiler.cpp:105-115: non-empty sources joined by newlines."""
        return self.combined.decode("utf-8", errors="surrogateescape")


_SPLIT_MESSAGES = {1: ".kernel directive without a name",
                   2: ".config outside of a .kernel section",
                   3: ".text outside of a .kernel section"}


def decompile_listing(listing: Union[str, bytes], opts: Optional[DecompileOptions] = None,
                      devices: Optional[Sequence[int]] = None) -> DecompileResult:
    """ocldec::decompile_listing (decompiler.cpp:117-133) on the GPU.

    ``devices``: shard the listing by kernel sections across these CUDA
    devices, one host thread per device (ocldec_b200_decompile_multi); the
    result is identical to the single-device call.

    A split_kernels ParseError yields zero kernels and one error diagnostic,
    as in the reference (decompiler.cpp:120-125); a kernel-level ParseError
    marks that kernel ``failed`` with empty source (decompiler.cpp:95-99).
    """
    L = _lib.load()
    if isinstance(listing, str):
        listing = listing.encode("utf-8", errors="surrogateescape")
    opts = opts or DecompileOptions()
    amap = opts.abi_map
    if isinstance(amap, str):
        amap = amap.encode("utf-8", errors="surrogateescape")
    o = _lib.Options(int(opts.fold_local_size),
                     opts.only_kernel.encode() if opts.only_kernel is not None else None,
                     opts.device, opts.arena_bytes, amap, len(amap) if amap is not None else 0,
                     int(opts.dump_cfg), int(opts.dump_regions), int(opts.record_reduction),
                     int(opts.export_body), int(opts.semantic_check), opts.semantic_seed)
    out = ctypes.POINTER(_lib.Result)()
    if devices:
        devs = (ctypes.c_int * len(devices))(*devices)
        rc = L.ocldec_b200_decompile_multi(listing, len(listing), ctypes.byref(o), devs, len(devices),
                                           ctypes.byref(out))
    else:
        rc = L.ocldec_b200_decompile(listing, len(listing), ctypes.byref(o), ctypes.byref(out))
    if rc != 0:
        raise RuntimeError(f"ocldec_b200_decompile failed ({rc}): {_lib.last_error()}")
    try:
        r = out.contents
        res = DecompileResult(device_ms=r.device_ms)
        combined = ctypes.string_at(r.combined, r.combined_len) if r.combined_len else b""
        names = ctypes.string_at(r.names) if r.names else b""
        res.combined = combined
        for i in range(r.nkernels):
            k = r.kernels[i]
            src = combined[k.src_off:k.src_off + k.src_len] if k.src_len else b""
            res.kernels.append(DecompiledKernel(
                name=names[k.name_off:k.name_off + k.name_len].decode(errors="surrogateescape"),
                source=src.decode("utf-8", errors="surrogateescape"),
                structured=bool(k.structured), failed=bool(k.failed),
                fallback_count=k.fallback_count, instructions=k.instructions))
            if r.sem:
                sc = r.sem[i]
                res.kernels[-1].semantic = (sc.status, sc.envs, sc.hash_asm, sc.hash_body)
        if r.ndumps:
            dl = [r.dumps[i] for i in range(r.ndumps)]
            dtext = ctypes.string_at(r.dump_text, max(d.off + d.len for d in dl))
            for d in dl:
                txt = dtext[d.off:d.off + d.len].decode("utf-8", errors="surrogateescape")
                k = res.kernels[d.kernel]
                if d.step == -1:
                    k.cfg_dot = txt
                elif d.step == -2:
                    k.reduction = Reduction.parse(txt)
                elif d.step == -3:
                    k.body_text = txt
                elif d.step == -4:
                    k.cfg_text = txt
                else:
                    k.region_dumps.append(txt)
        alld = [r.diags[i] for i in range(r.ndiags)] + [r.abi_diags[i] for i in range(r.nabi_diags)]
        tlen = max((d.msg_off + d.msg_len for d in alld), default=0)
        text = ctypes.string_at(r.diag_text, tlen) if r.diag_text and tlen else b""
        for i, d in enumerate(alld):
            msg = text[d.msg_off:d.msg_off + d.msg_len].decode("utf-8", errors="surrogateescape")
            (res.diagnostics if i < r.ndiags else res.abi_diagnostics).append(
                Diagnostic(d.severity, d.line, msg))
        return res
    finally:
        L.ocldec_b200_free(out)


def check_abi_map(text: Union[str, bytes]) -> List[Diagnostic]:
    """parse_abi_overrides (abi_model.cpp:109-153) alone: the diagnostics the
    reference CLI prints for an --abi-map file before decompiling."""
    L = _lib.load()
    if isinstance(text, str):
        text = text.encode("utf-8", errors="surrogateescape")
    cap = 4096 + 4 * len(text)
    while True:
        buf = ctypes.create_string_buffer(cap)
        rc = L.ocldec_b200_abi_map_check(text, len(text), buf, cap)
        if rc != -2:
            break
        cap *= 2
    if rc < 0:
        raise RuntimeError(f"ocldec_b200_abi_map_check failed ({rc}): {_lib.last_error()}")
    out = []
    for line in buf.value.split(b"\n"):
        if line:
            sev, ln, msg = line.split(b" ", 2)
            out.append(Diagnostic(int(sev), int(ln), msg.decode("utf-8", errors="surrogateescape")))
    return out


def generate_corpus(shape: Union[int, str], count: int, seed: int = 1, k0: int = 0, stress: bool = False):
    """Host generation of the synthetic corpus (od_gen.cuh; identical bytes to
    the device generator).  Returns (listing bytes, per-kernel offsets list,
    instruction count)."""
    import numpy as np
    L = _lib.load()
    shape = SHAPES.get(shape, shape) if isinstance(shape, str) else shape
    offs = np.zeros(count + 1, dtype=np.uint64)
    ni = ctypes.c_uint64()
    need = ctypes.c_uint64()
    L.ocldec_b200_gen_host(shape, int(stress), seed, k0, count, None, 0, offs.ctypes.data,
                           ctypes.byref(ni), ctypes.byref(need))
    buf = ctypes.create_string_buffer(int(need.value) + 1)
    n = L.ocldec_b200_gen_host(shape, int(stress), seed, k0, count, buf, need.value + 1, offs.ctypes.data,
                               ctypes.byref(ni), ctypes.byref(need))
    if n < 0:
        raise RuntimeError("corpus generation failed")
    return buf.raw[:n], offs, int(ni.value)


class Session:
    """HBM-resident batch runs (bench, multi-GPU shards): ocldec_b200_session_*."""

    def __init__(self, device: int = 0, arena_bytes: int = 0):
        self._L = _lib.load()
        self._s = self._L.ocldec_b200_session_create(device, arena_bytes)
        if not self._s:
            raise RuntimeError(f"session create failed: {_lib.last_error()}")
        self.device = device

    def close(self):
        if self._s:
            self._L.ocldec_b200_session_destroy(self._s)
            self._s = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream_ptr(self) -> int:
        return self._L.ocldec_b200_session_stream(self._s) or 0

    def generate(self, shape: Union[int, str], count: int, seed: int = 1, k0: int = 0, stress: bool = False):
        """Device generation; returns (device ptr, length, device offsets ptr, instructions)."""
        shape = SHAPES.get(shape, shape) if isinstance(shape, str) else shape
        buf, ln, offs, ni = ctypes.c_void_p(), ctypes.c_uint64(), ctypes.c_void_p(), ctypes.c_uint64()
        rc = self._L.ocldec_b200_gen_device(self._s, shape, int(stress), seed, k0, count, ctypes.byref(buf),
                                            ctypes.byref(ln), ctypes.byref(offs), ctypes.byref(ni))
        if rc:
            raise RuntimeError(f"gen_device failed: {_lib.last_error()}")
        return buf.value, ln.value, offs.value, ni.value

    def run(self, d_listing: int, length: int, chunk_starts: Sequence[int], fold_local_size: bool = False,
            sync: bool = True):
        import numpy as np
        cs = np.ascontiguousarray(np.asarray(chunk_starts, dtype=np.uint64))
        rc = self._L.ocldec_b200_session_run(self._s, d_listing, length,
                                             cs.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(cs),
                                             int(fold_local_size), int(sync))
        if rc:
            raise RuntimeError(f"session_run failed ({rc}): {_lib.last_error()}")

    def set_records(self, keep: bool):
        """Keep per-kernel host records (names, spans, flags, diagnostics) of
        later runs (default True); False leaves them on the device and only
        totals and combined_source come back."""
        self._L.ocldec_b200_session_set_records(self._s, int(keep))

    SEM_STATUS = ("equal", "mismatch", "unsupported", "capacity", "not_run", "indeterminate")

    def set_semantic(self, on: bool, seed: int = 0):
        """Run the batched semantic check (8 environments per kernel) in
        every later session run, with this environment seed."""
        if self._L.ocldec_b200_session_set_semantic(self._s, int(on), int(seed)):
            raise RuntimeError(f"set_semantic failed: {_lib.last_error()}")

    def semantic_counts(self) -> dict:
        """Kernels of the last run per semantic-check status (SEM_STATUS)."""
        c = (ctypes.c_uint64 * 6)()
        if self._L.ocldec_b200_session_semantic_counts(self._s, c):
            raise RuntimeError(f"semantic_counts failed: {_lib.last_error()}")
        return dict(zip(self.SEM_STATUS, (int(x) for x in c)))

    def run_generated(self, shape: Union[int, str], count: int, seed: int = 1, k0: int = 0, stress: bool = False,
                      chunk_bytes: int = 0, sample_stride: int = 0, fold_local_size: bool = False):
        """Streams kernels [k0, k0+count) of a generated corpus through the
        pipeline chunk by chunk (ocldec_b200_session_run_generated): no
        whole-corpus buffer.  Returns (stats dict, sample hashes, sample lengths)."""
        import numpy as np
        shape = SHAPES.get(shape, shape) if isinstance(shape, str) else shape
        ns = 0
        if sample_stride:
            ns = (k0 + count + sample_stride - 1) // sample_stride - (k0 + sample_stride - 1) // sample_stride
        hs = np.zeros(max(ns, 1), dtype=np.uint64)
        ls = np.zeros(max(ns, 1), dtype=np.uint64)
        st = _lib.StreamStats()
        rc = self._L.ocldec_b200_session_run_generated(self._s, shape, int(stress), seed, k0, count, chunk_bytes,
                                                       int(fold_local_size), sample_stride, hs.ctypes.data,
                                                       ls.ctypes.data, ctypes.byref(st))
        if rc:
            raise RuntimeError(f"run_generated failed ({rc}): {_lib.last_error()}")
        d = {n: getattr(st, n) for n, _ in _lib.StreamStats._fields_}
        return d, hs[:ns], ls[:ns]

    def run_host(self, host_ptr: int, length: int, out_ptr: int, out_cap: int, fold_local_size: bool = False) -> int:
        """Host buffers in and out (ocldec_b200_session_run_host); returns output length."""
        n = ctypes.c_uint64()
        rc = self._L.ocldec_b200_session_run_host(self._s, host_ptr, length, int(fold_local_size), out_ptr,
                                                  out_cap, ctypes.byref(n))
        if rc:
            raise RuntimeError(f"session_run_host failed ({rc}): {_lib.last_error()}")
        return n.value

    def stats(self) -> dict:
        st = _lib.Stats()
        self._L.ocldec_b200_session_stats(self._s, ctypes.byref(st))
        d = {n: getattr(st, n) for n, _ in _lib.Stats._fields_}
        d["prof_cycles"] = list(d["prof_cycles"])
        return d

    def kernels(self):
        """Per-kernel (offset, length, flags, fallbacks) of the last run as numpy
        arrays; flags bit0 failed, bit1 structured (ocldec_b200_session_kernels)."""
        import numpy as np
        n = int(self.stats()["kernels"])
        off = np.zeros(n + 1, dtype=np.uint64)
        ln = np.zeros(n + 1, dtype=np.uint64)
        fl = np.zeros(n + 1, dtype=np.uint32)
        fb = np.zeros(n + 1, dtype=np.uint32)
        rc = self._L.ocldec_b200_session_kernels(self._s, off.ctypes.data, ln.ctypes.data, fl.ctypes.data,
                                                 fb.ctypes.data)
        if rc:
            raise RuntimeError(f"session_kernels failed ({rc}): {_lib.last_error()}")
        return off[:n], ln[:n], fl[:n], fb[:n]

    def names(self):
        """(listing offset, length) of each kernel's name in the last run
        (offset 2**64-1: not a single listing span); ocldec_b200_session_names."""
        import numpy as np
        n = int(self.stats()["kernels"])
        off = np.zeros(n + 1, dtype=np.uint64)
        ln = np.zeros(n + 1, dtype=np.uint32)
        rc = self._L.ocldec_b200_session_names(self._s, off.ctypes.data, ln.ctypes.data)
        if rc:
            raise RuntimeError(f"session_names failed ({rc}): {_lib.last_error()}")
        return off[:n], ln[:n]

    def diagnostics(self) -> List[Diagnostic]:
        """DecompileResult::diagnostics of the last run (ocldec_b200_session_diagnostics)."""
        need = ctypes.c_uint64()
        self._L.ocldec_b200_session_diagnostics(self._s, None, 0, ctypes.byref(need))
        buf = ctypes.create_string_buffer(need.value)
        rc = self._L.ocldec_b200_session_diagnostics(self._s, buf, need.value, ctypes.byref(need))
        if rc < 0:
            raise RuntimeError(f"session_diagnostics failed ({rc}): {_lib.last_error()}")
        out = []
        for line in buf.raw[:need.value - 1].split(b"\n"):
            if line:
                sev, ln, msg = line.split(b" ", 2)
                out.append(Diagnostic(int(sev), int(ln), msg.decode("utf-8", errors="surrogateescape")))
        return out

    def output(self):
        p, n = ctypes.c_void_p(), ctypes.c_uint64()
        self._L.ocldec_b200_session_output(self._s, ctypes.byref(p), ctypes.byref(n))
        return p.value, n.value

    def output_bytes(self) -> bytes:
        """D2H copy of the last run's combined output (via torch for the copy)."""
        import torch
        p, n = self.output()
        if n == 0:
            return b""
        host = torch.empty(n, dtype=torch.uint8, pin_memory=True)
        _cudart_memcpy(host.data_ptr(), p, n)
        return host.numpy().tobytes()


def _cudart_memcpy(dst: int, src: int, n: int):
    """cudaMemcpyDefault through the library (UVA: either direction)."""
    rc = _lib.load().ocldec_b200_copy(dst, src, n)
    if rc:
        raise RuntimeError(f"copy failed: {_lib.last_error()}")


def copy(dst: int, src: int, n: int):
    _cudart_memcpy(dst, src, n)
