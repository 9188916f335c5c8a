"""ctypes binding of the C ABI in include/ocldec_b200.h.

The shared library is built in-tree (``make -C paper_2107_07809_b200/csrc``
or ``__graft_entry__.build()``) for sm_100a.  There is no fallback: if the
library is missing, importing the decompiler raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# OCLDEC_B200_LIB selects an alternative in-tree build (tuning experiments).
LIB_PATH = os.environ.get("OCLDEC_B200_LIB") or os.path.join(_HERE, "libocldec_b200.so")


class Options(ctypes.Structure):
    _fields_ = [("fold_local_size", ctypes.c_int), ("only_kernel", ctypes.c_char_p),
                ("device", ctypes.c_int), ("arena_bytes", ctypes.c_size_t),
                ("abi_map", ctypes.c_char_p), ("abi_map_len", ctypes.c_size_t),
                ("dump_cfg", ctypes.c_int), ("dump_regions", ctypes.c_int),
                ("record_reduction", ctypes.c_int), ("export_body", ctypes.c_int),
                ("semantic_check", ctypes.c_int), ("semantic_seed", ctypes.c_uint64)]


class Kernel(ctypes.Structure):
    _fields_ = [("name_off", ctypes.c_uint64), ("name_len", ctypes.c_uint64),
                ("src_off", ctypes.c_uint64), ("src_len", ctypes.c_uint64),
                ("failed", ctypes.c_int32), ("structured", ctypes.c_int32),
                ("fallback_count", ctypes.c_int32), ("instructions", ctypes.c_uint32)]


class Diag(ctypes.Structure):
    _fields_ = [("severity", ctypes.c_int32), ("line", ctypes.c_int32),
                ("msg_off", ctypes.c_uint64), ("msg_len", ctypes.c_uint64)]


class Dump(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_uint64), ("step", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("off", ctypes.c_uint64), ("len", ctypes.c_uint64)]


class SemCheck(ctypes.Structure):
    _fields_ = [("status", ctypes.c_uint32), ("envs", ctypes.c_uint32), ("hash_asm", ctypes.c_uint64),
                ("hash_body", ctypes.c_uint64)]


class Result(ctypes.Structure):
    _fields_ = [("nkernels", ctypes.c_uint64), ("kernels", ctypes.POINTER(Kernel)),
                ("names", ctypes.c_void_p), ("combined", ctypes.c_void_p),
                ("combined_len", ctypes.c_uint64), ("split_error_line", ctypes.c_int32),
                ("split_error_kind", ctypes.c_int32), ("instructions", ctypes.c_uint64),
                ("device_ms", ctypes.c_double), ("ndiags", ctypes.c_uint64),
                ("diags", ctypes.POINTER(Diag)), ("diag_text", ctypes.c_void_p),
                ("nabi_diags", ctypes.c_uint64), ("abi_diags", ctypes.POINTER(Diag)),
                ("ndumps", ctypes.c_uint64), ("dumps", ctypes.POINTER(Dump)), ("dump_text", ctypes.c_void_p),
                ("sem", ctypes.POINTER(SemCheck))]


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "kernels", "instructions", "lines", "in_bytes", "out_bytes", "failed", "goto_form",
        "fallbacks", "retried", "decompile_launches", "total_launches")] + [
        ("ms_parse", ctypes.c_double), ("ms_decompile", ctypes.c_double), ("ms_emit", ctypes.c_double),
        ("prof_cycles", ctypes.c_uint64 * 16),
        ("ms_front", ctypes.c_double), ("ms_lower", ctypes.c_double), ("ms_render", ctypes.c_double),
        ("ms_fold", ctypes.c_double)]


class StreamStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "kernels", "instructions", "in_bytes", "out_bytes", "chunks", "failed", "goto_form", "fallbacks")] + [
        ("ms_decompile", ctypes.c_double), ("ms_generate", ctypes.c_double), ("ms_wall", ctypes.c_double)]


EXPORTS = [
    "ocldec_b200_decompile", "ocldec_b200_decompile_multi", "ocldec_b200_free", "ocldec_b200_last_error", "ocldec_b200_version",
    "ocldec_b200_session_create", "ocldec_b200_session_destroy", "ocldec_b200_session_stream",
    "ocldec_b200_session_run", "ocldec_b200_session_stats", "ocldec_b200_session_output",
    "ocldec_b200_session_kernels", "ocldec_b200_gen_host", "ocldec_b200_gen_device",
    "ocldec_b200_session_run_host", "ocldec_b200_copy", "ocldec_b200_abi_map_check",
    "ocldec_b200_session_names", "ocldec_b200_session_diagnostics", "ocldec_b200_session_run_generated",
    "ocldec_b200_session_set_records", "ocldec_b200_session_set_semantic", "ocldec_b200_session_semantic_counts",
]

_lib = None


def load():
    """Loads the CUDA library; raises if it is absent (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"ocldec-b200 CUDA library not built: {LIB_PATH} "
                          "(run __graft_entry__.build() or make -C paper_2107_07809_b200/csrc)")
    L = ctypes.CDLL(LIB_PATH)
    vp, u64, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
    L.ocldec_b200_decompile.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(Options),
                                        ctypes.POINTER(ctypes.POINTER(Result))]
    L.ocldec_b200_decompile_multi.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(Options),
                                              ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                              ctypes.POINTER(ctypes.POINTER(Result))]
    L.ocldec_b200_decompile_multi.restype = i32
    L.ocldec_b200_decompile.restype = i32
    L.ocldec_b200_free.argtypes = [ctypes.POINTER(Result)]
    L.ocldec_b200_abi_map_check.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t]
    L.ocldec_b200_abi_map_check.restype = i32
    L.ocldec_b200_last_error.restype = ctypes.c_char_p
    L.ocldec_b200_version.restype = i32
    L.ocldec_b200_session_create.argtypes = [i32, ctypes.c_size_t]
    L.ocldec_b200_session_create.restype = vp
    L.ocldec_b200_session_destroy.argtypes = [vp]
    L.ocldec_b200_session_stream.argtypes = [vp]
    L.ocldec_b200_session_stream.restype = vp
    L.ocldec_b200_session_run.argtypes = [vp, vp, ctypes.c_size_t, ctypes.POINTER(u64), ctypes.c_size_t,
                                          i32, i32]
    L.ocldec_b200_session_run.restype = i32
    L.ocldec_b200_session_run_host.argtypes = [vp, vp, ctypes.c_size_t, i32, vp, u64, ctypes.POINTER(u64)]
    L.ocldec_b200_session_run_host.restype = i32
    L.ocldec_b200_copy.argtypes = [vp, vp, u64]
    L.ocldec_b200_copy.restype = i32
    L.ocldec_b200_session_stats.argtypes = [vp, ctypes.POINTER(Stats)]
    L.ocldec_b200_session_output.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(u64)]
    L.ocldec_b200_session_kernels.argtypes = [vp, vp, vp, vp, vp]
    L.ocldec_b200_session_names.argtypes = [vp, vp, vp]
    L.ocldec_b200_session_diagnostics.argtypes = [vp, ctypes.c_char_p, u64, ctypes.POINTER(u64)]
    L.ocldec_b200_gen_host.argtypes = [i32, i32, u64, u64, u64, vp, u64, vp, ctypes.POINTER(u64),
                                       ctypes.POINTER(u64)]
    L.ocldec_b200_gen_host.restype = ctypes.c_int64
    L.ocldec_b200_gen_device.argtypes = [vp, i32, i32, u64, u64, u64, ctypes.POINTER(vp),
                                         ctypes.POINTER(u64), ctypes.POINTER(vp), ctypes.POINTER(u64)]
    L.ocldec_b200_gen_device.restype = i32
    L.ocldec_b200_session_run_generated.argtypes = [vp, i32, i32, u64, u64, u64, u64, i32, u64, vp, vp,
                                                    ctypes.POINTER(StreamStats)]
    L.ocldec_b200_session_run_generated.restype = i32
    L.ocldec_b200_session_set_records.argtypes = [vp, i32]
    L.ocldec_b200_session_set_records.restype = i32
    L.ocldec_b200_session_set_semantic.argtypes = [vp, i32, u64]
    L.ocldec_b200_session_set_semantic.restype = i32
    L.ocldec_b200_session_semantic_counts.argtypes = [vp, ctypes.POINTER(u64)]
    L.ocldec_b200_session_semantic_counts.restype = i32
    _lib = L
    return L


def last_error() -> str:
    return load().ocldec_b200_last_error().decode(errors="replace")
