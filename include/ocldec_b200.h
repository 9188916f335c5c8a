/* ocldec-b200: C ABI of the B200-native batch GCN -> OpenCL decompiler.
 *
 * Drop-in boundary for the reference's pipeline front door
 *   ocldec::decompile_listing(const std::string&, const DecompileOptions&)
 *       /root/reference/proj/core/include/ocldec/decompiler.hpp:62
 * and its result types
 *   DecompileOptions      decompiler.hpp:29-35   -> ocldec_b200_options
 *   DecompiledKernel      decompiler.hpp:39-52   -> ocldec_b200_kernel
 *   DecompileResult       decompiler.hpp:54-60   -> ocldec_b200_result
 *   combined_source()     decompiler.cpp:105-115 -> ocldec_b200_result.combined
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 * All decompilation runs on the GPU (sm_100a); there is no CPU path.  Every
 * entry point returns 0 on success and a negative code on API misuse or CUDA
 * failure (ocldec_b200_last_error() has the message).  Data errors (a kernel
 * that fails to parse, a listing-level split error) are reported in the
 * result exactly as the reference reports them, never as a return code.
 */
#ifndef OCLDEC_B200_H
#define OCLDEC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCLDEC_B200_ABI_VERSION 5

/* DecompileOptions (decompiler.hpp:29-35). */
typedef struct ocldec_b200_options {
    int fold_local_size;     /* FoldOptions::fold_local_size (sym_state.hpp:27-29) */
    const char *only_kernel; /* restrict to one kernel by name, NULL = all        */
    int device;              /* CUDA device ordinal                               */
    size_t arena_bytes;      /* decompile arena pool per wave, 0 = default         */
    const char *abi_map;     /* ABI override file text (the CLI's --abi-map), NULL = none:
                                parse_abi_overrides abi_model.cpp:109-153 */
    size_t abi_map_len;
    int dump_cfg;            /* DecompileOptions::dump_cfg: DecompiledKernel::cfg_dot (to_dot, cfg.cpp:400-424) */
    int dump_regions;        /* DecompileOptions::dump_regions: ReduceResult::dumps
                                (region_graph_dot, structurizer.cpp:669-688, one per reduction step) */
    int record_reduction;    /* DecompiledKernel::reduction's merges and root / residue as a
                                step -2 dump (text: "merge <kind> <result> <absorbed...>" lines,
                                then "root <id>" or "residue <ids...>"; structurizer.hpp:54-104) */
    int export_body;         /* DecompiledKernel::body (LoweredBody, lower.hpp:20-41) as a step -3
                                dump: expression nodes and the statement tree in the text format
                                of od_lower.cuh's body_text (ABI v5); and DecompiledKernel::cfg
                                (cfg.hpp:60-84, after normalize_if_else) as a step -4 dump, one
                                line per block (od_kernel.cuh cfg_text) */
    int semantic_check;      /* the batched semantic check (ABI v5): per kernel,
                                the reference's differential backend (interpret_asm vs
                                evaluate_decompiled, oracle.cpp) restated on the device, over 8
                                sampled environments; results in ocldec_b200_result.sem */
    uint64_t semantic_seed;  /* environment stream seed (od_semenv.cuh) */
} ocldec_b200_options;

/* DecompiledKernel (decompiler.hpp:39-52): the printed source and flags. */
typedef struct ocldec_b200_kernel {
    uint64_t name_off, name_len;  /* into ocldec_b200_result.names  */
    uint64_t src_off, src_len;    /* into ocldec_b200_result.combined (0 len when failed) */
    int32_t failed;               /* hard parse error; source empty */
    int32_t structured;           /* false: goto residue was needed */
    int32_t fallback_count;       /* LoweredBody::fallback_count    */
    uint32_t instructions;        /* parse_text instruction count    */
} ocldec_b200_kernel;

/* Diagnostic (diagnostics.hpp:20-27): severity 0 note, 1 warning, 2 error;
 * message at diag_text[msg_off, msg_off + msg_len); Diagnostic::render
 * (diagnostics.cpp:22-26) is "<file>:<line>: <severity>: <message>". */
typedef struct ocldec_b200_diag {
    int32_t severity;
    int32_t line;
    uint64_t msg_off, msg_len;
} ocldec_b200_diag;

/* One dump of a kernel: step -1 is cfg_dot, step -2 the reduction record,
 * step -3 the lowered body and step -4 the flow graph (export_body), step
 * i >= 0 is reduction.dumps[i]
 * ("step<i>"); text at
 * dump_text[off, off + len). */
typedef struct ocldec_b200_dump {
    uint64_t kernel;              /* index into ocldec_b200_result.kernels */
    int32_t step;
    int32_t reserved;
    uint64_t off, len;
} ocldec_b200_dump;

/* One kernel's semantic check: status 0 equal traces in every environment,
 * 1 a mismatch, 2 unsupported (either side left the interpreted subset, as
 * OracleUnsupported), 3 not compared (the device's trace / variable room ran
 * out), 4 not run (failed or skipped kernel), 5 indeterminate (an operation
 * met two NaNs with different payloads, whose result IEEE 754 leaves open, so
 * the traces depend on the host compiler); the hashes sum, over the
 * environments, a mix of each write trace's FNV-1a hash and length
 * (od_semenv.cuh), for the assembly and the decompiled body. */
typedef struct ocldec_b200_semcheck {
    uint32_t status;
    uint32_t envs;
    uint64_t hash_asm;
    uint64_t hash_body;
} ocldec_b200_semcheck;

typedef struct ocldec_b200_result {
    uint64_t nkernels;
    ocldec_b200_kernel *kernels;
    char *names;                  /* kernel names, concatenated */
    char *combined;               /* combined_source(): sources joined by "\n" */
    uint64_t combined_len;
    int32_t split_error_line;     /* >0: split_kernels ParseError at this line (zero kernels) */
    int32_t split_error_kind;     /* 1 nameless .kernel, 2 .config outside, 3 .text outside */
    uint64_t instructions;        /* total parse_text instructions */
    double device_ms;             /* device time of the pipeline (CUDA events) */
    uint64_t ndiags;              /* DecompileResult::diagnostics, in sink order */
    ocldec_b200_diag *diags;
    char *diag_text;
    uint64_t nabi_diags;          /* parse_abi_overrides' own sink (the CLI prints these
                                     against the map file and stops on errors) */
    ocldec_b200_diag *abi_diags;  /* messages also in diag_text */
    uint64_t ndumps;              /* DOT dumps (options dump_cfg / dump_regions), by kernel then step */
    ocldec_b200_dump *dumps;
    char *dump_text;
    ocldec_b200_semcheck *sem;    /* per kernel (aligned with kernels) when semantic_check, else NULL */
} ocldec_b200_result;

/* decompile_listing: host buffer in, host result out (H2D/D2H inside). */
int ocldec_b200_decompile(const char *listing, size_t len, const ocldec_b200_options *opts,
                          ocldec_b200_result **out);
void ocldec_b200_free(ocldec_b200_result *res);
/* decompile_listing sharded across devices: the listing is
 * cut into ndevices byte-balanced runs of whole kernel sections (at
 * ".kernel" lines); one host thread per shard drives its device's session;
 * the shards' {out_bytes, lines, split error, kernels} tuples give each
 * shard's offset in combined_source, its listing-global line base and the
 * global split error (decompiler.cpp:105-125); each thread then copies its
 * text straight into the result at its offset.  The result is identical to
 * ocldec_b200_decompile's.  A device may be listed more than once (several
 * sessions on one device).  opts->device is ignored. */
int ocldec_b200_decompile_multi(const char *listing, size_t len, const ocldec_b200_options *opts,
                                const int *devices, int ndevices, ocldec_b200_result **out);
/* parse_abi_overrides (abi_model.cpp:109-153) alone, on the host: writes its
 * diagnostics as "<severity> <line> <message>\n" lines into buf (capacity
 * cap, NUL-terminated); returns the number of errors, or -2 when buf is too
 * small. */
int ocldec_b200_abi_map_check(const char *text, size_t len, char *buf, size_t cap);
const char *ocldec_b200_last_error(void);
int ocldec_b200_version(void);

/* ---------------------------------------------------------------- batch
 * Session API for HBM-resident corpora (bench and multi-GPU shards).  A
 * session owns device buffers on one device and one stream; calls on one
 * session are serialized by the caller. */
typedef struct ocldec_b200_session ocldec_b200_session;

ocldec_b200_session *ocldec_b200_session_create(int device, size_t arena_bytes);
void ocldec_b200_session_destroy(ocldec_b200_session *s);
/* The stream all session work is issued on (a cudaStream_t). */
void *ocldec_b200_session_stream(ocldec_b200_session *s);

/* Decompiles a device-resident listing d_listing[0, len) whose kernel sections
 * start at the byte offsets chunk_starts[0..nchunks) (each a ".kernel" line;
 * chunk_starts[0] == 0).  Output stays on the device: *d_out / *out_len.
 * Asynchronous on the session stream unless sync != 0.  Per-call counters
 * are returned through ocldec_b200_session_stats. */
int ocldec_b200_session_run(ocldec_b200_session *s, const void *d_listing, size_t len,
                            const uint64_t *chunk_starts, size_t nchunks, int fold_local_size,
                            int sync);
/* Host-buffer batch call on a session (the e2e path): H2D of the listing,
 * the device pipeline, D2H of combined_source into host_out (capacity
 * out_cap).  *out_len always receives the output size; returns -2 when
 * host_out is too small.  Pinned host buffers make both copies DMA. */
int ocldec_b200_session_run_host(ocldec_b200_session *s, const char *listing, size_t len,
                                 int fold_local_size, char *host_out, uint64_t out_cap,
                                 uint64_t *out_len);
typedef struct ocldec_b200_stats {
    uint64_t kernels, instructions, lines, in_bytes, out_bytes, failed, goto_form, fallbacks;
    uint64_t retried; /* kernels re-run with a larger arena */
    uint64_t decompile_launches, total_launches;
    double ms_parse, ms_decompile, ms_emit; /* last run, per pass (events); emit = combined_source gather */
    uint64_t prof_cycles[16]; /* OCLDEC_B200_PROF=1: SM cycles per decompile phase (cumulative) */
    double ms_front, ms_lower, ms_render; /* decompile pass split by launch (k_front/k_lower/k_emit) */
    double ms_fold;                       /* k_fold (fold_expr over the statements) */
} ocldec_b200_stats;
int ocldec_b200_session_stats(ocldec_b200_session *s, ocldec_b200_stats *st);
/* Device pointer + length of the last run's combined output. */
int ocldec_b200_session_output(ocldec_b200_session *s, const void **d_out, uint64_t *len);
/* Copies per-kernel (source offset, length, flags) of the last run to host arrays
 * of size >= kernels: off/len in the combined output, flags bit0 failed,
 * bit1 structured; fallbacks per kernel. */
int ocldec_b200_session_kernels(ocldec_b200_session *s, uint64_t *off, uint64_t *len,
                                uint32_t *flags, uint32_t *fallbacks);

/* Kernel names of the last run: name k is the caller's listing bytes
 * [off[k], off[k] + len[k]) (off[k] == UINT64_MAX when the .kernel line held
 * a stripped comment and the name is not one span of the listing). */
int ocldec_b200_session_names(ocldec_b200_session *s, uint64_t *off, uint32_t *len);
/* DecompileResult::diagnostics of the last run, in sink order, as
 * "<severity> <line> <message>\n" lines (NUL-terminated) in buf; returns the
 * count, or -2 when cap < *need. */
int ocldec_b200_session_diagnostics(ocldec_b200_session *s, char *buf, uint64_t cap, uint64_t *need);

/* Whether session runs keep per-kernel host records (default 1): kernel
 * names, source spans, flags and diagnostics for session_kernels /
 * session_names / session_diagnostics.  With 0 the per-kernel results stay
 * on the device and a run only gathers its totals (session_stats) and
 * combined_source: no per-kernel device-to-host traffic or host loops. */
int ocldec_b200_session_set_records(ocldec_b200_session *s, int keep);

/* Whether session runs (session_run / run_host / run_generated) also run the
 * batched semantic check (options.semantic_check for
 * the one-shot calls) with this environment seed, and how many kernels of
 * the last run ended in each ocldec_b200_semcheck status 0..5 (device
 * counters; no per-kernel transfer). */
int ocldec_b200_session_set_semantic(ocldec_b200_session *s, int on, uint64_t seed);
int ocldec_b200_session_semantic_counts(ocldec_b200_session *s, uint64_t counts[6]);

/* cudaMemcpy(dst, src, n, cudaMemcpyDefault): host<->device staging helper
 * for callers without their own CUDA runtime binding. */
int ocldec_b200_copy(void *dst, const void *src, uint64_t n);

/* ------------------------------------------------------ synthetic corpora
 * Counter-based generator; kernel k is a pure function of
 * (shape, stress, seed, k), identical on host and device. */
/* Host: writes kernels [k0, k0+count) into buf (cap bytes); offsets gets
 * count+1 byte offsets; returns bytes written or a negative error
 * (-2 = buffer too small; *needed gets the size). */
int64_t ocldec_b200_gen_host(int shape, int stress, uint64_t seed, uint64_t k0, uint64_t count,
                             char *buf, uint64_t cap, uint64_t *offsets, uint64_t *instructions,
                             uint64_t *needed);
/* Device: generates kernels [k0, k0+count) into a session-owned device buffer;
 * returns its pointer, length, and per-kernel offsets (device). */
int ocldec_b200_gen_device(ocldec_b200_session *s, int shape, int stress, uint64_t seed,
                           uint64_t k0, uint64_t count, const void **d_buf, uint64_t *len,
                           const uint64_t **d_offsets, uint64_t *instructions);

/* Streaming run of a generated corpus (~320 GB of listing
 * for 1M kernels, more than HBM): kernels [k0, k0+count) are sized on the
 * device, cut into chunks of at most chunk_bytes (0 = default) at kernel
 * boundaries, and each chunk is generated into the session's text buffer and
 * decompiled before the next one is generated; no whole-corpus buffer.  Each
 * chunk's combined output replaces the previous one on the device.  With
 * sample_stride > 0, kernel k with k % sample_stride == 0 gets the FNV-1a
 * hash and length of its source at index k / sample_stride - ceil(k0 /
 * sample_stride) of sample_hash / sample_len (either may be NULL). */
typedef struct ocldec_b200_stream_stats {
    uint64_t kernels, instructions, in_bytes, out_bytes, chunks, failed, goto_form, fallbacks;
    double ms_decompile; /* device time of the decompile passes (parse + decompile + gather), all chunks */
    double ms_generate;  /* device time of the generator (sizing + per-chunk text) */
    double ms_wall;      /* device time of the whole call */
} ocldec_b200_stream_stats;
int ocldec_b200_session_run_generated(ocldec_b200_session *s, int shape, int stress, uint64_t seed,
                                      uint64_t k0, uint64_t count, uint64_t chunk_bytes, int fold_local_size,
                                      uint64_t sample_stride, uint64_t *sample_hash, uint64_t *sample_len,
                                      ocldec_b200_stream_stats *out);

#ifdef __cplusplus
}
#endif

#endif /* OCLDEC_B200_H */
