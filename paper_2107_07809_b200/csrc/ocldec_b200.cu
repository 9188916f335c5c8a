// ocldec-b200: device passes, host orchestration and the C ABI
// (include/ocldec_b200.h).  sm_100a only.
//
// Pass plan per chunk of the listing:
//   P1a k_nl_count/k_nl_write  16-byte vector loads, block scan of newline
//                              flags -> newline positions
//   P1b k_classify             thread per line: comment strip, trim, first word,
//                              operand / label bounds for the decode pools
//   P1c section scan           (kernel count, last directive) pair scan -> line roles
//   P1d k_decode               thread per text line: labels, perfect-hash
//                              mnemonic, operands (pool offsets scanned from
//                              the bounds)
//   P2-P4a k_front/k_lower/k_fold/k_emit  thread per .kernel section, size-sorted waves with
//                              exact per-kernel arenas: config/ABI, CFG,
//                              exec-mask normalization, region reduction,
//                              liveness, lowering, emission
//   P4b k_gather               scan of output lengths, warp-per-kernel scatter
//                              into the combined_source buffer
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ocldec_b200.h"
#include "od_device.cuh"
#include "od_oracle.cuh"
#include "od_scan.cuh"

using namespace od;

namespace {

thread_local std::string g_err;

#define CK(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess) {                                                                   \
            g_err = std::string(#x) + ": " + cudaGetErrorString(e_);                               \
            return -3;                                                                             \
        }                                                                                          \
    } while (0)

constexpr u32 kTileThreads = 256;
constexpr u32 kTileVecs = 4;                                  // uint4 per thread per tile
constexpr u32 kTileBytes = kTileThreads * kTileVecs * 16;     // 16 KiB

// ------------------------------------------------------------------ P1a
// Newline count per 16 KiB tile.  The chunk may start unaligned: the tile
// grid covers [base - mis, base + len) and masks bytes outside.
__global__ void k_nl_count(const u8 *__restrict__ base, u64 len, u32 mis, u32 *tile_cnt) {
    const u8 *p0 = base - mis;
    const u64 tile0 = (u64)blockIdx.x * kTileBytes;
    u32 c = 0;
#pragma unroll
    for (u32 j = 0; j < kTileVecs; ++j) {
        u64 o = tile0 + ((u64)j * kTileThreads + threadIdx.x) * 16;
        if (o >= len + mis)
            continue;
        uint4 v = *reinterpret_cast<const uint4 *>(p0 + o);
        u32 w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                u64 pos = o + q * 4 + b;
                u8 ch = (u8)(w[q] >> (8 * b));
                if (ch == '\n' && pos >= mis && pos < len + mis)
                    ++c;
            }
        }
    }
    // block reduce
    c = __reduce_add_sync(0xffffffffu, c);
    __shared__ u32 sm[kTileThreads / 32];
    if ((threadIdx.x & 31) == 0)
        sm[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        u32 v = threadIdx.x < kTileThreads / 32 ? sm[threadIdx.x] : 0;
        v = __reduce_add_sync(0xffffffffu, v);
        if (threadIdx.x == 0)
            tile_cnt[blockIdx.x] = v;
    }
}

// Writes the chunk-relative position of every newline, in order.
__global__ void k_nl_write(const u8 *__restrict__ base, u64 len, u32 mis, const u32 *tile_off,
                           u32 *nlpos) {
    const u8 *p0 = base - mis;
    const u64 tile0 = (u64)blockIdx.x * kTileBytes;
    __shared__ SU32 sm[32];
    u32 run = tile_off[blockIdx.x];
    for (u32 j = 0; j < kTileVecs; ++j) {
        u64 o = tile0 + ((u64)j * kTileThreads + threadIdx.x) * 16;
        u32 bits = 0; // newline bitmap of my 16 bytes
        if (o < len + mis) {
            uint4 v = *reinterpret_cast<const uint4 *>(p0 + o);
            u32 w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    u64 pos = o + q * 4 + b;
                    u8 ch = (u8)(w[q] >> (8 * b));
                    if (ch == '\n' && pos >= mis && pos < len + mis)
                        bits |= 1u << (q * 4 + b);
                }
        }
        SU32 agg;
        SU32 ex = block_exclusive(SU32{(u32)__popc(bits)}, SU32{0}, AddU32{}, sm, &agg);
        u32 k = run + ex.v;
        while (bits) {
            u32 b = __ffs(bits) - 1;
            bits &= bits - 1;
            nlpos[k++] = (u32)(o + b - mis);
        }
        run += agg.v;
    }
}

// ------------------------------------------------------------------ P1b
// Thread per line: comment strip + rtrim + first-word kind.
// Also sizes the decode pools: an upper bound of the line's operands (one
// more than its runs of ',' / isspace bytes, the decoder's own separator
// predicate c_space: every token after the first follows such a run) and of
// its labels (its ':' count), over the raw line, which contains whatever the
// comment strip keeps.
// k_decode's staging: the block's 256 lines are one contiguous span of the
// listing, staged in shared memory with 16-byte loads of its aligned interior
// (bytewise for the first block of a misaligned chunk).  Returns false when
// the span is larger than the stage (the lines then read the listing in
// HBM).  [ab, se) is staged at stage[0]; [sb, se) is the block's raw span.
constexpr u32 kLineStage = 16384;

__device__ __forceinline__ bool stage_lines(const u8 *__restrict__ t, u64 len, const u32 *__restrict__ nlpos,
                                            u32 nlf, u32 nlines, u8 *stage, u64 *sb_out, u64 *ab_out,
                                            u64 *se_out) {
    const u32 l0 = blockIdx.x * blockDim.x;
    const u32 l1 = min(l0 + blockDim.x, nlines);
    const u64 sb = l0 == 0 ? 0 : (u64)nlpos[l0 - 1] + 1;
    const u64 se = l1 - 1 < nlf ? (u64)nlpos[l1 - 1] : len;
    const u32 lead = (u32)((uintptr_t)(t + sb) & 15);
    const bool vec = sb >= lead;
    const u64 ab = vec ? sb - lead : sb;
    const bool staged = se - ab <= kLineStage;
    if (staged) {
        u64 done = ab;
        if (vec) {
            const u64 nv = (se - ab) / 16;
            const uint4 *src = reinterpret_cast<const uint4 *>(t + ab);
            for (u64 q = threadIdx.x; q < nv; q += blockDim.x)
                reinterpret_cast<uint4 *>(stage)[q] = src[q];
            done = ab + 16 * nv;
        }
        for (u64 o = done + threadIdx.x; o < se; o += blockDim.x)
            stage[o - ab] = t[o];
    }
    *sb_out = sb;
    *ab_out = ab;
    *se_out = se;
    return staged;
}

__global__ void k_classify(const u8 *__restrict__ t, u64 len, const u32 *__restrict__ nlpos,
                           u32 nlf, u32 nlines, LineRec *lines, u32 *complex_bytes, u32 *ops_ub,
                           u32 *labs_ub) {
    u32 l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= nlines)
        return;
    u32 b = l == 0 ? 0 : nlpos[l - 1] + 1;
    u32 e = l < nlf ? nlpos[l] : (u32)len;
    // (staging the block's span in shared memory first, as k_decode does,
    // measured slower: parse 245 -> 263 ms per C4 step)
    const u8 *tb = t;
    // one pass over the raw line: the pool bounds (separator runs, ':'
    // count) and strip_comments' cut; a "/*" leaves the cut to strip_scan
    bool cx = false;
    u32 cut = e - b, runs = 0, colons = 0;
    {
        bool prev = false, inq = false, found = false, slow = false;
        for (u32 i = b; i < e; ++i) {
            const u8 c = tb[i];
            const bool sep = c == ',' || c_space(c);
            runs += sep && !prev;
            prev = sep;
            colons += c == ':';
            if (found)
                continue;
            if (c == '"')
                inq = !inq;
            if (!inq) {
                if (c == '#' || c == ';') {
                    cut = i - b;
                    found = true;
                } else if (c == '/' && i + 1 < e && tb[i + 1] == '*') {
                    found = slow = true;
                }
            }
        }
        if (slow)
            cut = strip_scan(tb + b, e - b, &cx);
    }
    LineRec r;
    r.off = b;
    r.complex = cx;
    r.role = LR_NONE;
    r.pad = 0;
    r.aux = 0;
    if (!cx) {
        r.len = rtrim_len(tb + b, cut);
        r.kind = classify_content(tb, Span{r.off, r.len});
    } else {
        r.len = e - b; // raw span, materialized later
        r.kind = LK_BLANK;
        atomicAdd(complex_bytes, e - b);
    }
    lines[l] = r;
    const bool content = cx || r.len;
    ops_ub[l] = content ? runs + 1 : 0;
    labs_ub[l] = content ? colons : 0;
}

// Complex lines (with a terminated /* */ mid-line) are materialized into the
// aux area after the chunk, then classified.
__global__ void k_materialize(u8 *t, u32 aux_base, u32 nlines, LineRec *lines, u32 *aux_top) {
    u32 l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= nlines || !lines[l].complex)
        return;
    LineRec r = lines[l];
    u32 n = strip_materialize(t + r.off, r.len, nullptr);
    u32 dst = aux_base + atomicAdd(aux_top, n);
    strip_materialize(t + r.off, r.len, t + dst);
    r.off = dst;
    r.len = rtrim_len(t + dst, n);
    r.kind = classify_content(t, Span{r.off, r.len});
    lines[l] = r;
}

// ------------------------------------------------------------------ P1c
struct SecLoad {
    const LineRec *lines;
    __device__ SecVal operator()(u64 i) const {
        u8 k = lines[i].kind;
        SecVal v;
        v.cnt = k == LK_KERNEL ? 1 : 0;
        v.last = (k == LK_KERNEL || k == LK_DIR_CONFIG || k == LK_DIR_TEXT) ? (i32)i : -1;
        return v;
    }
};
struct SecStore {
    LineRec *lines;
    u32 *kstart;
    u32 *err; // min error line (0xffffffff none) and kind
    __device__ void operator()(u64 i, SecVal ex, SecVal v) const {
        LineRec &L = lines[i];
        u8 k = L.kind;
        if (k == LK_KERNEL) {
            kstart[ex.cnt] = (u32)i;
            return;
        }
        if (k == LK_KERNEL_NONAME) {
            atomicMin(err, (u32)i);
            return;
        }
        if (k == LK_DIR_CONFIG || k == LK_DIR_TEXT) {
            if (ex.cnt == 0)
                atomicMin(err, (u32)i);
            return;
        }
        if (k != LK_OTHER || ex.cnt == 0)
            return;
        u8 mode_kind = lines[ex.last].kind; // last directive before (>= the .kernel line)
        L.role = mode_kind == LK_DIR_TEXT ? LR_TEXT : LR_CONFIG;
    }
};

// ------------------------------------------------------------------ P1d
__device__ RootTable d_roots;

__global__ void k_init_roots() {
    if (threadIdx.x == 0 && blockIdx.x == 0)
        build_root_table(&d_roots);
}

// One pass per text line into the operand / label pools at the offsets
// scanned from k_classify's bounds.  The block's 256 lines are one contiguous span of the listing: it is staged
// in shared memory (16-byte vector loads for the aligned interior) and every
// thread decodes its line from there.  Lines whose content lives in the aux
// area (comment-stripped copies) and oversized spans read the listing in HBM.
// Shape key of the decode order: operand bound (0..7) x length class.
#ifndef OD_DECODE_LEN_CLASSES
#define OD_DECODE_LEN_CLASSES 2
#endif
#ifndef OD_DECODE_LEN_STEP
#define OD_DECODE_LEN_STEP 6
#endif

// 6 blocks per SM (40 registers, 16 bytes of spills) over the register-
// limited 5: parse 263 -> 245 ms per C4 step (8 blocks: 254 ms)
#ifndef OD_DECODE_MINB
#define OD_DECODE_MINB 6
#endif
__global__ void __launch_bounds__(256, OD_DECODE_MINB) k_decode(const u8 *__restrict__ t, u64 len, const u32 *__restrict__ nlpos,
                                                u32 nlf, u32 nlines, const LineRec *__restrict__ lines,
                                                LineIns *lins, const u32 *ops_off, const u32 *labs_off,
                                                Opnd *ops, Label *labs, u32 ops_total, u32 *overflow,
                                                const u32 *__restrict__ ops_ub) {
    __shared__ RootTable rt;
    __shared__ __align__(16) u8 stage[kLineStage];
    for (u32 i = threadIdx.x; i < sizeof(RootTable) / 4; i += blockDim.x)
        reinterpret_cast<u32 *>(&rt)[i] = reinterpret_cast<const u32 *>(&d_roots)[i];
    u64 sb, ab, se;
    const bool staged = stage_lines(t, len, nlpos, nlf, nlines, stage, &sb, &ab, &se);
    const u32 l0 = blockIdx.x * blockDim.x;
    // Lines of one shape take the same decode paths: the block's lines are
    // reordered by a shape key (operand bound from k_classify, long or
    // short) with a counting sort in shared memory, so each warp decodes
    // lines of similar shape (each line's decode is independent).
    constexpr u32 kNB = 8 * OD_DECODE_LEN_CLASSES + 1; // last bucket: not a text line
    __shared__ u32 bucket[kNB];
    __shared__ u16 order[256];
    if (threadIdx.x < kNB)
        bucket[threadIdx.x] = 0;
    __syncthreads();
    u32 key = kNB - 1; // past the end, or not a text line
    {
        const u32 lk = l0 + threadIdx.x;
        if (lk < nlines) {
            const LineRec Lk = lines[lk];
            if (Lk.role == LR_TEXT) {
#if OD_DECODE_LEN_CLASSES == 2
                const u32 lc = Lk.len >= 36 ? 1u : 0u;
#else
                const u32 lc = min(Lk.len / OD_DECODE_LEN_STEP, (u32)OD_DECODE_LEN_CLASSES - 1);
#endif
                key = min(ops_ub[lk], 7u) * OD_DECODE_LEN_CLASSES + lc;
            }
        }
    }
    const u32 rank = atomicAdd(&bucket[key], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
        u32 acc = 0;
        for (u32 b = 0; b < kNB; ++b) {
            const u32 c = bucket[b];
            bucket[b] = acc;
            acc += c;
        }
    }
    __syncthreads();
    order[bucket[key] + rank] = (u16)threadIdx.x;
    __syncthreads();
    const u32 l = l0 + order[threadIdx.x];
    if (l >= nlines)
        return;
    const LineRec L = lines[l];
    if (L.role != LR_TEXT)
        return;
    // the decoder addresses the listing by chunk offsets: tb[off] == t[off]
    const bool in_stage = staged && !L.complex && L.off >= sb && (u64)L.off + L.len <= se;
    const u8 *tb = in_stage ? stage - ab : t;
    LineIns li;
    const u32 oo = ops_off[l], lo = labs_off[l];
    const u32 cap = (l + 1 < nlines ? ops_off[l + 1] : ops_total) - oo;
    decode_line(tb, Span{L.off, L.len}, &rt, &li, ops + oo, cap, labs + lo);
    if (li.nops > cap) { // k_classify's bound is exact-or-above by construction
        atomicOr(overflow, 1u);
        li.nops = (u16)cap;
    }
    li.op_start = oo;
    li.lab_start = lo;
    lins[l] = li;
}

// Per-kernel sizes (a pass over the kernel's decoded lines), size key and
// arena budget.
// One warp per kernel: kernel_size's sums (od_kernel.cuh) over a lane-strided
// walk of the kernel's lines (coalesced record reads), reduced across the warp.
__global__ void k_ksize(const u32 *kstart, u32 nk, u32 nlines, const LineRec *lines, const LineIns *lins,
                        const Opnd *ops, KSize *sizes, u32 *key, u64 *budget, u32 group, u32 novr) {
    const u32 k = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const u32 lane = threadIdx.x & 31;
    if (k >= nk) // whole warps: nk is warp-uniform
        return;
    const u32 b = kstart[k], e = k + 1 < nk ? kstart[k + 1] : nlines;
    u32 ncfg = 0, nins = 0, nlab = 0, labelled = 0, enders = 0, xops = 0;
    for (u32 l = b + 1 + lane; l < e; l += 32) {
        const u8 role = lines[l].role;
        if (role == LR_CONFIG) {
            ++ncfg;
            continue;
        }
        if (role != LR_TEXT)
            continue;
        const LineIns &L = lins[l];
        nlab += L.nlabels;
        labelled += L.nlabels ? 1 : 0;
        if (!(L.flags & IF_HAS_INS))
            continue;
        ++nins;
        if (L.prefix == PX_S && (L.root == R_BRANCH || L.root == R_ENDPGM || (L.rflags & RF_CBRANCH)))
            ++enders;
        u32 m;
        if (L.prefix == PX_S && exec_kind_of(L.root, L.prefix, L.flags, L.nops, ops + L.op_start, &m) != XK_NONE)
            ++xops;
    }
    const u32 full = 0xffffffffu;
    ncfg = __reduce_add_sync(full, ncfg);
    nins = __reduce_add_sync(full, nins);
    nlab = __reduce_add_sync(full, nlab);
    const u32 nbx = __reduce_add_sync(full, labelled + enders + xops);
    if (lane)
        return;
    KSize z;
    z.n = e - b;
    z.ncfg = ncfg;
    z.nins = nins;
    z.nlab = nlab;
    z.nb = 3 + nbx;
    z.novr = novr;
    sizes[k] = z;
    // sort key: lines, optionally grouped by class (straight-line kernels
    // first) so an SM's resident kernels share their hot code
    const u32 n15 = z.n < 0x3fffu ? z.n : 0x3fffu;
    u32 cls = 0;
    if (group == 1)
        cls = z.nb > 4 ? 0u : 2u;                           // straight-line first, then branching
    else if (group == 2)
        cls = z.nb <= 4 ? 3u : (z.nb <= 24 ? 2u : (z.nb <= 96 ? 1u : 0u)); // by block-count class
    key[k] = group ? (cls << 14) | n15 : z.n;
    budget[k] = kernel_budget(z, 1);
}

// Counting sort by descending size: histogram, scan, scatter.
constexpr u32 kSizeBuckets = 1u << 16;
__device__ __forceinline__ u32 size_bucket(u32 n) {
    return kSizeBuckets - 1 - (n < kSizeBuckets - 1 ? n : kSizeBuckets - 1);
}
__global__ void k_hist(const u32 *key, u32 nk, u32 *hist) {
    u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nk)
        atomicAdd(&hist[size_bucket(key[k])], 1u);
}
__global__ void k_scatter(const u32 *key, u32 nk, u32 *cursor, u32 *order, const u64 *budget, u64 *sbudget) {
    u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nk)
        return;
    u32 pos = atomicAdd(&cursor[size_bucket(key[k])], 1u);
    order[pos] = k;
    sbudget[pos] = budget[k];
}

// Interleaves the size-sorted order (even positions first, then odd), so
// contiguous waves get the same mix of kernel sizes.
__global__ void k_interleave(const u32 *order, const u64 *sb, u32 n, u32 *order_out, u64 *sb_out) {
    u32 i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const u32 p = (i & 1) ? (n + 1) / 2 + i / 2 : i / 2;
    order_out[p] = order[i];
    sb_out[p] = sb[i];
}

// Class of a kernel after k_front (the code the next launches run): 0 done
// (failed / skipped), 1 straight-line, 2 structured with ifs, 3 goto form.
struct Cnt4 {
    u32 c[4];
    __device__ static Cnt4 shfl_up(Cnt4 x, int d) {
        Cnt4 r;
        for (int q = 0; q < 4; ++q)
            r.c[q] = __shfl_up_sync(0xffffffffu, x.c[q], d);
        return r;
    }
};
struct AddCnt4 {
    __device__ Cnt4 operator()(Cnt4 a, Cnt4 b) const {
        Cnt4 r;
        for (int q = 0; q < 4; ++q)
            r.c[q] = a.c[q] + b.c[q];
        return r;
    }
};
__device__ __forceinline__ u32 lower_class(const KState *g) {
    if (g->done)
        return 0;
    if (!g->K.reduced)
        return 3;
    return g->K.nif ? 2 : 1;
}
struct ClsLoad {
    const u8 *arena;
    const u64 *boff;
    u64 boff0;
    __device__ Cnt4 operator()(u64 i) const {
        const u32 c = lower_class(reinterpret_cast<const KState *>(arena + (boff[i] - boff0)));
        Cnt4 v;
        for (int q = 0; q < 4; ++q)
            v.c[q] = q == (int)c ? 1u : 0u;
        return v;
    }
};
struct ClsStore {
    u32 *perm;
    const Cnt4 *total;
    __device__ void operator()(u64 i, Cnt4 ex, Cnt4 v) const {
        u32 base = 0;
        for (int q = 0; q < 4; ++q) {
            if (v.c[q]) {
                perm[base + ex.c[q]] = (u32)i;
                return;
            }
            base += total->c[q];
        }
    }
};

// ------------------------------------------------------------------ P4b
struct U64Val {
    u64 v;
    __device__ static U64Val shfl_up(U64Val x, int d) { return U64Val{__shfl_up_sync(0xffffffffu, x.v, d)}; }
};
struct AddU64 {
    __device__ U64Val operator()(U64Val a, U64Val b) const { return U64Val{a.v + b.v}; }
};
// Output lengths (+1 for the separator) scanned in u64: a chunk's combined
// output may pass 4 GiB (inline-asm fallback lines expand 2-4x).
struct OutLenLoad {
    const KRes *res;
    __device__ U64Val operator()(u64 i) const {
        u64 n = res[i].status == KS_OK ? res[i].out_len : 0;
        return U64Val{n ? n + 1 : 0};
    }
};
struct OutOffStore {
    u64 *off;
    __device__ void operator()(u64 i, U64Val ex, U64Val) const { off[i] = ex.v; }
};

// Warp per kernel: staging -> combined output (+ the "\n" separator that
// combined_source puts between non-empty sources).  The staged text is
// 16-byte aligned, its destination is not: the head up to the destination's
// next 16-byte boundary and the tail go bytewise; the body is written as
// aligned 16-byte stores, each assembled from two aligned 16-byte source
// loads with byte permutes (the source misalignment is the head length).
__global__ void k_gather(const KRes *__restrict__ res, const u64 *__restrict__ off, u32 nk,
                         const u8 *__restrict__ stage, u8 *out, u64 out_base, u64 total) {
    const u64 warp = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u32 lane = threadIdx.x & 31;
    if (warp >= nk)
        return;
    const KRes r = res[warp];
    if (r.status != KS_OK || !r.out_len)
        return;
    const u8 *s = stage + r.stage_off;
    u8 *d = out + out_base + off[warp];
    const u32 n = r.out_len;
    const u32 h = min((u32)((16 - ((uintptr_t)d & 15)) & 15), n);
    if (lane < h)
        d[lane] = s[lane];
    const u32 nv = (n - h) / 16;
    const uint4 *s4 = reinterpret_cast<const uint4 *>(s); // s + h + 16q spans s4[q], s4[q + 1] when h > 0
    uint4 *d4 = reinterpret_cast<uint4 *>(d + h);
    const u32 sh = h & 3, wo = h >> 2; // byte and word offset of the body in the source
    for (u32 q = lane; q < nv; q += 32) {
        if (!h) {
            d4[q] = s4[q];
            continue;
        }
        const uint4 a = s4[q], b = s4[q + 1];
        const u32 w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        u32 o[4];
        for (u32 k = 0; k < 4; ++k) {
            const u32 lo = w[wo + k], hi = w[wo + k + 1 < 8 ? wo + k + 1 : 7];
            o[k] = sh ? __byte_perm(lo, hi, 0x3210 + 0x1111 * sh) : lo;
        }
        d4[q] = make_uint4(o[0], o[1], o[2], o[3]);
    }
    for (u32 i = h + 16 * nv + lane; i < n; i += 32)
        d[i] = s[i];
    if (lane == 0 && out_base + off[warp] + n < total)
        d[n] = '\n';
}

struct U64Load {
    const u64 *p;
    __device__ U64Val operator()(u64 i) const { return U64Val{p[i]}; }
};
struct U64Store {
    u64 *p;
    __device__ void operator()(u64 i, U64Val ex, U64Val) const { p[i] = ex.v; }
};
struct U32Load {
    const u32 *p;
    __device__ SU32 operator()(u64 i) const { return SU32{p[i]}; }
};
struct U32Store {
    u32 *p;
    __device__ void operator()(u64 i, SU32 ex, SU32) const { p[i] = ex.v; }
};
struct U32SumLoad64 {
    const u32 *p;
    __device__ U64Val operator()(u64 i) const { return U64Val{p[i]}; }
};

// Per-chunk totals of the kernel results (the session path without
// per-kernel host records): instructions, failed, goto form, fallbacks.
__global__ void k_res_stats(const KRes *__restrict__ res, u32 nk, unsigned long long *tot) {
    const u32 k = blockIdx.x * blockDim.x + threadIdx.x;
    u64 ni = 0;
    u32 f = 0, g = 0, fb = 0;
    if (k < nk) {
        const KRes r = res[k];
        ni = r.ninstr;
        f = r.status == KS_FAILED;
        g = r.status == KS_OK && !r.structured;
        fb = r.fallbacks;
    }
    const u32 full = 0xffffffffu;
    for (u32 d = 16; d; d >>= 1) {
        ni += __shfl_down_sync(full, ni, d);
        f += __shfl_down_sync(full, f, d);
        g += __shfl_down_sync(full, g, d);
        fb += __shfl_down_sync(full, fb, d);
    }
    if ((threadIdx.x & 31) == 0 && (ni | f | g | fb)) {
        atomicAdd(&tot[0], (unsigned long long)ni);
        atomicAdd(&tot[1], (unsigned long long)f);
        atomicAdd(&tot[2], (unsigned long long)g);
        atomicAdd(&tot[3], (unsigned long long)fb);
    }
}

// Diagnostic spans of a chunk packed into one buffer (one D2H instead of a
// copy per span): warp per span, spans[i] = {src offset, length, dst offset}.
__global__ void k_span_gather(const u8 *__restrict__ t, const uint4 *__restrict__ spans, u32 n, u8 *out) {
    const u64 w = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (w >= n)
        return;
    const uint4 sp = spans[w];
    const u64 dst = (u64)sp.z | ((u64)sp.w << 32);
    for (u32 i = threadIdx.x & 31; i < sp.y; i += 32)
        out[dst + i] = t[(u64)sp.x + i];
}

// ================================================================== host side
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
};

int ensure(DevBuf &b, size_t bytes) {
    if (bytes <= b.cap && b.p)
        return 0;
    if (b.p) {
        cudaDeviceSynchronize(); // copies on the copy stream may still read it
        cudaFree(b.p);
    }
    size_t want = std::max(bytes + 256, b.cap + b.cap / 2);
    b.p = nullptr;
    b.cap = 0;
    CK(cudaMalloc(&b.p, want));
    b.cap = want;
    return 0;
}

// Grows b to at least bytes, preserving the first keep bytes.
int ensure_keep(DevBuf &b, size_t bytes, size_t keep, cudaStream_t st) {
    if (bytes <= b.cap && b.p)
        return 0;
    size_t want = std::max(bytes + 256, b.cap + b.cap / 2);
    void *np = nullptr;
    CK(cudaMalloc(&np, want));
    if (b.p && keep) {
        CK(cudaMemcpyAsync(np, b.p, std::min(keep, b.cap), cudaMemcpyDeviceToDevice, st));
        CK(cudaStreamSynchronize(st));
    }
    if (b.p) {
        cudaDeviceSynchronize(); // copies on the copy stream may still read it
        cudaFree(b.p);
    }
    b.p = np;
    b.cap = want;
    return 0;
}

template <class T> T *P(DevBuf &b) { return reinterpret_cast<T *>(b.p); }

// A kernel diagnostic with its listing spans copied out (the device text
// buffer is reused by the next chunk).
struct HostDiag {
    u32 line;
    u16 code, c;
    std::string a, b;
};

// ABI overrides parsed on the host (parse_abi_overrides, abi_model.cpp:109-153)
// and resolved as far as they do not depend on the kernel (abi_model.cpp:196-243).
struct HostOvr {
    AbiOvr dev;
    std::string tail, target; // for the messages
};

std::string trim_ovr(const std::string &s) { // trim_view  abi_model.cpp:72-78
    size_t b = 0, e = s.size();
    while (b < e && (s[b] == ' ' || s[b] == '\t'))
        ++b;
    while (e > b && (s[e - 1] == ' ' || s[e - 1] == '\t' || s[e - 1] == '\r'))
        --e;
    return s.substr(b, e - b);
}

bool parse_u32_ovr(std::string s, u32 *out) { // parse_u32  abi_model.cpp:59-70
    int base = 10;
    if (s.size() > 2 && s[0] == '0' && (s[1] == 'x' || s[1] == 'X')) {
        base = 16;
        s = s.substr(2);
    }
    if (s.empty())
        return false;
    u64 v = 0;
    for (char c : s) {
        int d;
        if (c >= '0' && c <= '9')
            d = c - '0';
        else if (base == 16 && c >= 'a' && c <= 'f')
            d = c - 'a' + 10;
        else if (base == 16 && c >= 'A' && c <= 'F')
            d = c - 'A' + 10;
        else
            return false;
        if (d >= base)
            return false;
        v = v * base + d;
        if (v > 0xffffffffull)
            return false;
    }
    *out = (u32)v;
    return true;
}

struct OvrDiag {
    int sev, line;
    std::string msg;
};

std::vector<HostOvr> parse_overrides(const std::string &text, std::vector<OvrDiag> *diags) {
    std::vector<HostOvr> out;
    size_t pos = 0;
    int line_no = 0;
    while (pos < text.size()) { // std::getline
        size_t nl = text.find('\n', pos);
        std::string raw = text.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
        pos = nl == std::string::npos ? text.size() : nl + 1;
        ++line_no;
        std::string line = trim_ovr(raw);
        if (line.empty() || line[0] == '#')
            continue;
        size_t eq = line.find('=');
        if (eq == std::string::npos) {
            diags->push_back({2, line_no, "override line is not key=value"});
            continue;
        }
        std::string key = trim_ovr(line.substr(0, eq)), value = trim_ovr(line.substr(eq + 1));
        HostOvr o;
        memset(&o.dev, 0, sizeof(o.dev));
        size_t colon = key.find(':');
        u32 offset;
        if (!parse_u32_ovr(trim_ovr(colon == std::string::npos ? key : key.substr(0, colon)), &offset)) {
            diags->push_back({2, line_no, "bad offset in override key"});
            continue;
        }
        o.dev.offset = offset;
        o.dev.dwords = 1;
        if (colon != std::string::npos) {
            u32 w;
            if (!parse_u32_ovr(trim_ovr(key.substr(colon + 1)), &w) || (w != 1 && w != 2)) {
                diags->push_back({2, line_no, "override width must be 1 or 2 dwords"});
                continue;
            }
            o.dev.dwords = (u8)w;
        }
        if (value.empty()) {
            diags->push_back({2, line_no, "override has an empty target"});
            continue;
        }
        o.target = value;
        size_t tc = value.find(':');
        std::string head = tc == std::string::npos ? value : value.substr(0, tc);
        o.tail = tc == std::string::npos ? std::string() : value.substr(tc + 1);
        if (head == "arg") {
            o.dev.kind = OV_ARG;
        } else {
            int fn = head == "global_offset" ? F_GLOBAL_OFFSET
                     : head == "global_size" ? F_GLOBAL_SIZE
                     : head == "work_dim"    ? F_WORK_DIM
                     : head == "local_size"  ? F_LOCAL_SIZE
                     : head == "num_groups"  ? F_NUM_GROUPS
                                             : -1;
            u32 dim = 0;
            if (fn < 0)
                o.dev.kind = OV_BAD_TARGET;
            else if (!o.tail.empty() && (!parse_u32_ovr(o.tail, &dim) || dim > 2))
                o.dev.kind = OV_BAD_DIM;
            else {
                o.dev.kind = OV_BUILTIN;
                o.dev.fn = (u8)fn;
                o.dev.dim = (u8)dim;
            }
        }
        out.push_back(std::move(o));
    }
    return out;
}

int diag_severity(u16 code) {
    switch (code) {
    case DG_UNREACHABLE: return 0;
    case DG_ARG_TYPE: case DG_OPERAND: case DG_MASK_MULTI: case DG_MASK_NONE: case DG_MASK_EXECZ_INV:
    case DG_MASK_NO_RESTORE: case DG_MASK_EXECZ_RST: case DG_SLOAD_UNMAPPED: case DG_ADDC: case DG_GOTO:
    case DG_EXEC_BRANCH:
        return 1;
    default: return 2;
    }
}

bool is_type_suffix(const std::string &tok) { // parse_type_suffix  type_recovery.cpp:50-73
    if (tok.size() < 2 || tok.size() > 3 || !strchr("iufb", tok[0]))
        return false;
    std::string w = tok.substr(1);
    return w == "8" || w == "16" || w == "24" || w == "32" || w == "64";
}

// decompose_mnemonic's root (asm_frontend.cpp:375-423) of an s_ mnemonic.
std::string mnemonic_root(const std::string &m) {
    std::string rest = m.size() > 2 ? m.substr(2) : std::string();
    std::vector<std::string> toks;
    size_t p = 0;
    for (;;) {
        size_t q = rest.find('_', p);
        toks.push_back(rest.substr(p, q == std::string::npos ? std::string::npos : q - p));
        if (q == std::string::npos)
            break;
        p = q + 1;
    }
    size_t end = toks.size(), peeled = 0;
    while (end > 1 && peeled < 2 && is_type_suffix(toks[end - 1])) {
        --end;
        ++peeled;
    }
    std::string root;
    for (size_t i = 0; i < end; ++i) {
        if (i)
            root += '_';
        root += toks[i];
    }
    return root;
}

// The reference's message text for a diagnostic.
std::string diag_message(const HostDiag &d, const std::vector<HostOvr> *ovr = nullptr) {
    switch (d.code) {
    case DG_DIMS: return "bad .dims axes '" + d.a + "'";
    case DG_CWS_COUNT: return "cws expects 1 to 3 sizes";
    case DG_CWS_VALUE: return "bad cws value '" + d.a + "'";
    case DG_SGPRS: return "bad sgprsnum value";
    case DG_VGPRS: return "bad vgprsnum value";
    case DG_ARG_FIELDS: return "arg directive needs name, type string and type";
    case DG_ARG_TYPE: return "unrecognized argument type '" + d.a + "' for '" + d.b + "'";
    case DG_OPERAND: {
        std::string m;
        switch (d.c) {
        case 1: m = "unbalanced bracket in register operand '" + d.a + "'"; break;
        case 2: m = "register range without ':' in '" + d.a + "'"; break;
        case 3: m = "bad register range '" + d.a + "'"; break;
        case 4: m = "negative register index in '" + d.a + "'"; break;
        default: {
            const bool scalar = !d.a.empty() && d.a[0] == 's';
            m = "register '" + d.a + "' exceeds the " + (scalar ? "SGPR" : "VGPR") + " file (max " +
                (scalar ? "103" : "255") + ")";
        }
        }
        return m + "; keeping the line as inline assembly";
    }
    case DG_BR_NOLABEL: return "branch without a label operand";
    case DG_BR_UNDEF: return "branch to undefined label '" + d.a + "'";
    case DG_CBR_UNSUP: return "unsupported conditional branch s_" + mnemonic_root(d.a);
    case DG_CBR_END: return "conditional branch at end of kernel";
    case DG_UNREACHABLE: return "unreachable code";
    case DG_MASK_MULTI:
        return "exec mask saved in s[" + std::to_string(d.c) + ":" + std::to_string(d.c + 1) +
               "] has multiple join points";
    case DG_MASK_NONE: return "exec mask save without inversion or restore";
    case DG_MASK_EXECZ_INV: return "execz branch does not meet the mask inversion";
    case DG_MASK_NO_RESTORE: return "mask inversion without a matching restore";
    case DG_MASK_EXECZ_RST: return "execz branch does not meet the mask restore";
    case DG_SLOAD_UNMAPPED: return "scalar load from unmapped settings offset";
    case DG_ADDC: return "v_addc_u32 outside the 64-bit add idiom; carry treated as zero";
    case DG_GOTO: return "control flow not fully structured; emitting labeled blocks";
    case DG_EXEC_BRANCH: return "exec-dependent branch kept as inline asm";
    case DG_OVR_ARG: return "override names unknown argument '" + (ovr && d.c < ovr->size() ? (*ovr)[d.c].tail : "") + "'";
    case DG_OVR_TARGET: return "unknown override target '" + (ovr && d.c < ovr->size() ? (*ovr)[d.c].target : "") + "'";
    case DG_OVR_DIM: return "override dimension must be 0..2";
    default: return "diagnostic " + std::to_string(d.code);
    }
}

} // namespace

struct ocldec_b200_session {
    int device = 0;
    int nsm = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t stream2 = nullptr; // second decompile-wave stream
    u32 two_mode = 2;               // OCLDEC_B200_TWO_STREAMS: 0 off, 1 on, 2 (default) long-kernel chunks
    cudaStream_t cstream = nullptr; // host<->device copies overlapped with the chunks
    cudaEvent_t cev[3];             // [0..1] text buffer loaded, [2] chunk output ready
    DevBuf text2;                   // second chunk text buffer (double buffering)
    size_t arena_bytes = 0;
    DevBuf text, tiles, tiles_off, nlpos, lines, lins, ops_cnt, labs_cnt, ops_off, labs_off, ops,
        labs, kstart, scan_tmp, scan_tot, counters, arena, stage, res, outoff, out, only, retry,
        gen_len, gen_ninstr, gen_buf, gen_off, kmeta, order, budget, sbudget, boff, hist, prof, ksizes, perm, cnt4;
    u64 pool_bytes = 0;  // arena pool per decompile wave
    bool prof_on = false;
    u32 lanes_front = 32, lanes_lower = 32, lanes_emit = 32; // 32 / kernels per warp, per phase
    u32 smem_front = 0, smem_lower = 0, smem_emit = 0;        // occupancy limiters (dynamic smem)
    u32 group_class = 0;                                      // wave order grouped by kernel class
    u64 out_len = 0;
    u64 nk_total = 0;
    u32 only_len = 0;
    bool only_set = false;
    ocldec_b200_stats stats{};
    cudaEvent_t ev[8];
    std::vector<KRes> host_res;      // last run, all chunks
    std::vector<u64> host_kernel_off;
    std::vector<u32> host_name_line; // chunk-relative .kernel line (host path names)
    std::vector<u64> host_name_off;  // listing offset of each kernel's name (~0: not a listing span)
    u64 chunk_base = 0;              // listing offset of the chunk run_chunk is working on
    std::vector<cudaEvent_t> pev;    // phase-launch events (pool)
    DevBuf dpool, dtop;              // device diagnostic records of a chunk
    std::vector<HostDiag> host_diag; // materialized diagnostics, all chunks
    std::vector<HostOvr> ovr_host;   // ABI overrides of the current call
    u32 dump_flags = 0;              // DOT dumps of the current call (DumpFlags)
    DevBuf xtext, xrec, xtop, xcfg;  // device dump pool (DumpCfg)
    std::vector<std::vector<std::pair<int32_t, std::string>>> host_dumps; // per host_res kernel
    std::vector<OvrDiag> ovr_diags;  // their parse diagnostics
    DevBuf dovr, dovr_text;
    DevBuf sgen;                     // streamed generation: the current group of chunks
    DevBuf rstat;                    // per-chunk result totals (k_res_stats)
    bool keep_records = true;        // per-kernel host records (names, spans, flags, diagnostics)
    // Small readbacks (counters, totals) go through mapped pinned memory
    // written by a one-warp kernel, not a D2H copy: on the host-buffer path
    // the copy engine is busy with the previous chunk's output, and a small
    // cudaMemcpy queued behind it stalled the next chunk's parse (measured:
    // parse 382 vs 245 ms per C4 step).
    u8 *peek_h = nullptr, *peek_d = nullptr;
    bool wide_lower = false;         // OCLDEC_B200_WIDE_LOWER: k_lower_wide for long-kernel chunks
    bool sem_on = false;             // the batched semantic check of the current call
    u64 sem_seed = 0;
    bool sem_session = false;        // session_set_semantic: every session run checks
    u64 sem_session_seed = 0;
    u64 sem_kbase = 0;               // listing ordinal of the run's first kernel (a shard's offset)
    long sem_budget = 1 << 14;       // in-wave steps per environment before a kernel is deferred
                                     // (OCLDEC_B200_SEM_BUDGET; 0: never)
    const u64 *sem_kmap = nullptr;   // deferred re-check: listing ordinal per kernel (device)
    DevBuf semkmap, semdef, semspan, semdefbuf;
    std::string def_text;            // the run's deferred kernels' sections ...
    std::vector<u64> def_ord;        // ... and their listing ordinals
    int def_fold = 0;
    u64 def_kb_left = kSemDeferRunKB; // the run's remaining deferral allowance
    ocldec_b200_session *aux = nullptr; // re-checks the deferred kernels at the run's end
    std::string ovr_src;             // the ABI override text of the current run (set_overrides)
    DevBuf semres, semscratch;       // per chunk kernel: SemResult; the check's lane scratch
    DevBuf semcnt;                   // kernels per SemStatus since the run began (u64[8])
    bool sem_counted = false;        // the last run ran the check (semcnt is its count)
    std::vector<ocldec_b200_semcheck> host_sem; // per host_res kernel
    u32 novr = 0;
    std::vector<u64> host_kdiag;     // per kernel: first host_diag index (count in host_res[k].ndiag)
    size_t pev_used = 0;
};

namespace {

// Events bracketing each phase launch of a chunk (timed after the chunk syncs).
int phase_event(ocldec_b200_session *s, cudaEvent_t *e) {
    if (s->pev_used == s->pev.size()) {
        cudaEvent_t n;
        CK(cudaEventCreate(&n));
        s->pev.push_back(n);
    }
    *e = s->pev[s->pev_used++];
    return 0;
}

void sum_phase_events(ocldec_b200_session *s) {
    for (size_t i = 0; i + 4 < s->pev_used; i += 5) {
        float ms = 0;
        cudaEventElapsedTime(&ms, s->pev[i], s->pev[i + 1]);
        s->stats.ms_front += ms;
        cudaEventElapsedTime(&ms, s->pev[i + 1], s->pev[i + 2]);
        s->stats.ms_lower += ms;
        cudaEventElapsedTime(&ms, s->pev[i + 2], s->pev[i + 3]);
        s->stats.ms_fold += ms;
        cudaEventElapsedTime(&ms, s->pev[i + 3], s->pev[i + 4]);
        s->stats.ms_render += ms;
    }
    s->pev_used = 0;
}

// Generic exclusive scan launcher.
template <class T, class Op, class Load, class Store>
int scan_exclusive(ocldec_b200_session *s, u64 n, T ident, Op op, Load load, Store store, T *d_total) {
    if (n == 0)
        return 0;
    u64 per = (u64)kScanThreads * kScanItems;
    u64 nb = (n + per - 1) / per;
    if (ensure(s->scan_tmp, nb * sizeof(T)))
        return -3;
    T *agg = P<T>(s->scan_tmp);
    k_scan_reduce<<<(u32)nb, kScanThreads, 0, s->stream>>>(n, ident, op, load, agg);
    k_scan_blocks<<<1, kScanThreads, 0, s->stream>>>(nb, ident, op, agg, d_total);
    k_scan_apply<<<(u32)nb, kScanThreads, 0, s->stream>>>(n, ident, op, load, store, agg);
    s->stats.total_launches += 3;
    CK(cudaGetLastError());
    return 0;
}

constexpr size_t kPeekBytes = 4096;

__global__ void k_peek(u8 *dst, const u8 *src, u32 n) {
    for (u32 i = threadIdx.x; i < n; i += blockDim.x)
        dst[i] = src[i];
}

int d2h_sync(ocldec_b200_session *s, void *h, const void *d, size_t n) {
    if (s->peek_d && n <= kPeekBytes) {
        k_peek<<<1, 128, 0, s->stream>>>(s->peek_d, static_cast<const u8 *>(d), (u32)n);
        s->stats.total_launches++;
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(s->stream));
        memcpy(h, s->peek_h, n);
        return 0;
    }
    CK(cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    return 0;
}

struct ChunkOut {
    u32 nk;
    u32 nlines;
    u32 err_line; // 0xffffffff none (chunk-relative)
    u32 err_kind;
    u64 out_bytes;
};

// Runs P1-P4 on one chunk t[0, len) (device).  can_extend: t is the
// session's text buffer with room for the aux area.  Outputs are appended to
// s->out at out_base; per-kernel results are appended to s->host_res.
int collect_deferred(ocldec_b200_session *s, const u8 *t, u64 len, u32 nlf, const DecompArgs &a, u64 kb0,
                     int fold_local_size);
int finish_deferred(ocldec_b200_session *s);

int run_chunk(ocldec_b200_session *s, const u8 *t, u64 len, bool can_extend, u32 line_base,
              int fold_local_size, u64 out_base, bool prev_nonempty, ChunkOut *co) {
    cudaStream_t st = s->stream;
    co->nk = 0;
    co->nlines = 0;
    co->err_line = 0xffffffffu;
    co->err_kind = 0;
    co->out_bytes = 0;
    if (len == 0)
        return 0;
    if (len >= 0xf0000000ull) {
        g_err = "chunk larger than 3.75 GiB";
        return -5; // the host path retries with smaller chunks
    }
    const u32 mis = (u32)((uintptr_t)t & 15);
    const u64 span = len + mis;
    const u32 ntiles = (u32)((span + kTileBytes - 1) / kTileBytes);
    if (ensure(s->tiles, (ntiles + 1) * 4ull) || ensure(s->tiles_off, (ntiles + 1) * 4ull) ||
        ensure(s->counters, 64))
        return -3;
    u32 *cnt = P<u32>(s->counters);
    CK(cudaMemsetAsync(cnt, 0, 64, st));
    CK(cudaEventRecord(s->ev[0], st));
    k_nl_count<<<ntiles, kTileThreads, 0, st>>>(t, len, mis, P<u32>(s->tiles));
    if (scan_exclusive(s, ntiles, SU32{0}, AddU32{}, U32Load{P<u32>(s->tiles)},
                       U32Store{P<u32>(s->tiles_off)}, reinterpret_cast<SU32 *>(cnt)))
        return -3;
    u32 nlf = 0;
    if (d2h_sync(s, &nlf, cnt, 4))
        return -3;
    // last character: a final line without '\n' still counts
    u8 last = 0;
    if (d2h_sync(s, &last, t + len - 1, 1))
        return -3;
    const u32 nlines = nlf + (last != '\n' ? 1 : 0);
    co->nlines = nlines;
    if (ensure(s->nlpos, (nlf + 1) * 4ull) || ensure(s->lines, (u64)(nlines + 1) * sizeof(LineRec)))
        return -3;
    k_nl_write<<<ntiles, kTileThreads, 0, st>>>(t, len, mis, P<u32>(s->tiles_off), P<u32>(s->nlpos));
    const u32 lb = 256, lg = (nlines + lb - 1) / lb;
    if (ensure(s->ops_cnt, (nlines + 1) * 4ull) || ensure(s->labs_cnt, (nlines + 1) * 4ull))
        return -3;
    k_classify<<<lg, lb, 0, st>>>(t, len, P<u32>(s->nlpos), nlf, nlines, P<LineRec>(s->lines), cnt + 1,
                                  P<u32>(s->ops_cnt), P<u32>(s->labs_cnt));
    s->stats.total_launches += 3;
    CK(cudaGetLastError());
    u32 cbytes = 0;
    if (d2h_sync(s, &cbytes, cnt + 1, 4))
        return -3;
    if (cbytes) {
        if (len + (u64)cbytes >= 0xffff0000ull) {
            g_err = "chunk plus comment-stripped lines exceed 4 GiB";
            return -5; // the host path retries with smaller chunks
        }
        if (!can_extend) {
            // copy the chunk into the session buffer (with aux room) and redo
            if (ensure(s->text, len + cbytes + 64))
                return -3;
            CK(cudaMemcpyAsync(s->text.p, t, len, cudaMemcpyDeviceToDevice, st));
            return run_chunk(s, P<u8>(s->text), len, true, line_base, fold_local_size, out_base,
                             prev_nonempty, co);
        }
        k_materialize<<<lg, lb, 0, st>>>(const_cast<u8 *>(t), (u32)len, nlines, P<LineRec>(s->lines),
                                         cnt + 2);
        s->stats.total_launches++;
    }
    // P1c section scan
    if (ensure(s->kstart, (nlines + 1) * 4ull))
        return -3;
    CK(cudaMemsetAsync(cnt + 4, 0xff, 4, st));
    if (scan_exclusive(s, nlines, SecVal{0, -1}, SecOp{}, SecLoad{P<LineRec>(s->lines)},
                       SecStore{P<LineRec>(s->lines), P<u32>(s->kstart), cnt + 4},
                       reinterpret_cast<SecVal *>(cnt + 6)))
        return -3;
    u32 sec[4];
    if (d2h_sync(s, sec, cnt + 4, 16))
        return -3;
    const u32 err = sec[0];
    const u32 nk = sec[2];
    if (err != 0xffffffffu) {
        co->err_line = err;
        LineRec lr;
        if (d2h_sync(s, &lr, P<LineRec>(s->lines) + err, sizeof lr))
            return -3;
        co->err_kind = lr.kind == LK_KERNEL_NONAME ? 1 : lr.kind == LK_DIR_CONFIG ? 2 : 3;
        return 0;
    }
    co->nk = nk;
    if (nk == 0)
        return 0;
    CK(cudaEventRecord(s->ev[1], st));
    // P1d decode: pool offsets from k_classify's bounds, then the fill
    if (ensure(s->lins, (u64)(nlines + 1) * sizeof(LineIns)) || ensure(s->ops_off, (nlines + 1) * 4ull) ||
        ensure(s->labs_off, (nlines + 1) * 4ull))
        return -3;
    if (scan_exclusive(s, nlines, SU32{0}, AddU32{}, U32Load{P<u32>(s->ops_cnt)},
                       U32Store{P<u32>(s->ops_off)}, reinterpret_cast<SU32 *>(cnt + 8)) ||
        scan_exclusive(s, nlines, SU32{0}, AddU32{}, U32Load{P<u32>(s->labs_cnt)},
                       U32Store{P<u32>(s->labs_off)}, reinterpret_cast<SU32 *>(cnt + 9)))
        return -3;
    u32 pools[2];
    if (d2h_sync(s, pools, cnt + 8, 8))
        return -3;
    if (ensure(s->ops, (pools[0] + 1ull) * sizeof(Opnd)) || ensure(s->labs, (pools[1] + 1ull) * sizeof(Label)))
        return -3;
    k_decode<<<lg, lb, 0, st>>>(t, len, P<u32>(s->nlpos), nlf, nlines, P<LineRec>(s->lines), P<LineIns>(s->lins),
                                P<u32>(s->ops_off), P<u32>(s->labs_off), P<Opnd>(s->ops), P<Label>(s->labs),
                                pools[0], cnt + 3, P<u32>(s->ops_cnt));
    s->stats.total_launches++;
    CK(cudaGetLastError());
    CK(cudaEventRecord(s->ev[2], st));

    // P2-P4a decompile: size-sorted waves, exact per-kernel arenas, retries
    if (ensure(s->res, (u64)nk * sizeof(KRes)) || ensure(s->outoff, (u64)(nk + 1) * 8) ||
        ensure(s->kmeta, (u64)nk * 4 + 16) || ensure(s->order, (u64)nk * 4 + 16) ||
        ensure(s->budget, (u64)(nk + 1) * 8) || ensure(s->sbudget, (u64)(nk + 1) * 8) ||
        ensure(s->boff, (u64)(nk + 2) * 8) || ensure(s->hist, (u64)kSizeBuckets * 4))
        return -3;
    u64 stage_cap = std::max<u64>(len + (64ull << 20), 2 * len);
    if (ensure(s->stage, stage_cap))
        return -3;
    CK(cudaMemsetAsync(cnt + 14, 0, 8, st));
    DecompArgs a;
    a.t = t;
    a.lines = P<LineRec>(s->lines);
    a.lins = P<LineIns>(s->lins);
    a.ops = P<Opnd>(s->ops);
    a.labs = P<Label>(s->labs);
    a.kstart = P<u32>(s->kstart);
    a.nk = nk;
    a.nlines = nlines;
    a.line_base = line_base;
    a.fold_local_size = (u32)fold_local_size;
    a.stage = P<u8>(s->stage);
    a.stage_cap = s->stage.cap;
    a.stage_top = reinterpret_cast<unsigned long long *>(cnt + 14);
    if (ensure(s->dpool, std::max<u64>(1ull << 16, (u64)nk * 2) * sizeof(Diag)) || ensure(s->dtop, 16))
        return -3;
    CK(cudaMemsetAsync(s->dtop.p, 0, 8, st));
    a.dpool = P<Diag>(s->dpool);
    a.dcap = s->dpool.cap / sizeof(Diag);
    a.dtop = P<unsigned long long>(s->dtop);
    a.ovr = s->novr ? P<AbiOvr>(s->dovr) : nullptr;
    a.novr = s->novr;
    a.ovr_text = s->novr ? P<u8>(s->dovr_text) : nullptr;
    a.dump = nullptr;
    DumpCfg dc{};
    if (s->dump_flags) {
        if (ensure(s->xtext, std::max<u64>(16ull << 20, std::min<u64>((u64)len * 2, 1ull << 30))) ||
            ensure(s->xrec, std::max<u64>(1ull << 16, (u64)nk * 8) * sizeof(DumpRec)) ||
            ensure(s->xtop, 16) || ensure(s->xcfg, sizeof(DumpCfg)))
            return -3;
        CK(cudaMemsetAsync(s->xtop.p, 0, 16, st));
        dc.text = P<u8>(s->xtext);
        dc.cap = s->xtext.cap;
        dc.rec = P<DumpRec>(s->xrec);
        dc.rcap = s->xrec.cap / sizeof(DumpRec);
        dc.top = P<unsigned long long>(s->xtop);
        dc.flags = s->dump_flags;
        CK(cudaMemcpyAsync(s->xcfg.p, &dc, sizeof(dc), cudaMemcpyHostToDevice, st));
        a.dump = P<DumpCfg>(s->xcfg);
    }
    a.res = P<KRes>(s->res);
    a.only = s->only_set ? P<u8>(s->only) : nullptr;
    a.only_len = s->only_len;
    a.prof = s->prof_on ? P<u64>(s->prof) : nullptr;
    a.retry_cnt = cnt + 12;
    if (s->sem_on && (ensure(s->semres, (u64)nk * sizeof(SemResult) + 16) ||
                      ensure(s->semscratch, 2ull * kSemBatch * kSemEnvs * kSemLaneBytes) || !s->semcnt.p ||
                      ensure(s->semdef, 4ull * (kSemDeferCap + 2))))
        return -3;
    if (s->sem_on)
        CK(cudaMemsetAsync(s->semdef.p, 0, 8, st));
    const u64 sem_kb0 = s->stats.kernels; // kernels of the run before this chunk
    // OCLDEC_B200_WIDE_LOWER=1: in chunks of long kernels (C5: ~340 KB of
    // listing, hundreds of if-joins each) kernels with >= kWideJoins joins are
    // lowered by the whole warp (k_lower_wide, lane-parallel merge_join /
    // collect_delta).  Off by default: measured no gain on C5 (the 32 active
    // lanes widen the rest of the lowering's local-memory traffic) and a
    // loss on C4.
    a.wide_joins = s->wide_lower && s->lanes_lower == 32 && !OD_LOCAL_LOWER && len / nk >= (64u << 10)
                       ? kWideJoins : ~0u;
    CK(cudaMemsetAsync(cnt + 12, 0, 4, st));
    const u32 kb = 256, kg = (nk + kb - 1) / kb;
    u32 *key = P<u32>(s->kmeta);
    if (ensure(s->ksizes, (u64)nk * sizeof(KSize) + 16))
        return -3;
    a.sizes = P<KSize>(s->ksizes);
    k_ksize<<<(u32)(((u64)nk * 32 + kb - 1) / kb), kb, 0, st>>>(P<u32>(s->kstart), nk, nlines, P<LineRec>(s->lines), P<LineIns>(s->lins),
                               P<Opnd>(s->ops), P<KSize>(s->ksizes), key, P<u64>(s->budget), s->group_class,
                               s->novr);
    CK(cudaMemsetAsync(s->hist.p, 0, kSizeBuckets * 4ull, st));
    k_hist<<<kg, kb, 0, st>>>(key, nk, P<u32>(s->hist));
    if (scan_exclusive(s, kSizeBuckets, SU32{0}, AddU32{}, U32Load{P<u32>(s->hist)},
                       U32Store{P<u32>(s->hist)}, reinterpret_cast<SU32 *>(cnt + 11)))
        return -3;
    k_scatter<<<kg, kb, 0, st>>>(key, nk, P<u32>(s->hist), P<u32>(s->order), P<u64>(s->budget),
                                 P<u64>(s->sbudget));
    // two wave streams for this chunk (see session_init)
    const bool two_streams =
        s->stream2 && (s->two_mode == 1 || (s->two_mode == 2 && len / std::max<u64>(nk, 1) >= (64u << 10)));
    if (nk >= 1024 && two_streams) {
        k_interleave<<<kg, kb, 0, st>>>(P<u32>(s->order), P<u64>(s->sbudget), nk, key, P<u64>(s->budget));
        CK(cudaMemcpyAsync(s->order.p, key, (u64)nk * 4, cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(s->sbudget.p, s->budget.p, (u64)nk * 8, cudaMemcpyDeviceToDevice, st));
        s->stats.total_launches++;
    }
    CK(cudaMemsetAsync(P<u64>(s->sbudget) + nk, 0, 8, st));
    if (scan_exclusive(s, nk + 1, U64Val{0}, AddU64{}, U64Load{P<u64>(s->sbudget)},
                       U64Store{P<u64>(s->boff)}, reinterpret_cast<U64Val *>(P<u64>(s->budget) + nk)))
        return -3;
    s->stats.total_launches += 4;
    std::vector<u64> boff(nk + 1);
    if (d2h_sync(s, boff.data(), s->boff.p, (u64)(nk + 1) * 8))
        return -3;
    // waves: as many size-sorted kernels as the arena pool holds
    // Waves of size-sorted kernels, each as many as its arena region holds.
    // Large launches alternate between two streams (each with half of the
    // arena), so one wave's phase tails overlap the other wave's bulk.
    auto launch_waves = [&](const u64 *h_boff, const u32 *d_order, const u64 *d_boff, u32 count,
                            u32 scale) -> int {
        if (!count)
            return 0;
        const u64 total = h_boff[count] - h_boff[0];
        u64 maxneed = 0;
        for (u32 i = 0; i < count; ++i)
            maxneed = std::max<u64>(maxneed, h_boff[i + 1] - h_boff[i]);
        const bool two = count >= 1024 && two_streams;
        if (ensure(s->arena, std::max<u64>(two ? 2 * maxneed + 512 : maxneed, std::min<u64>(s->pool_bytes, total))))
            return -3;
        const u64 half = (s->arena.cap / 2) & ~255ull;
        u64 cap = s->arena.cap;
        if (two)
            cap = std::min<u64>(half, std::max<u64>(maxneed, (total + 1) / 2 + maxneed / 2));
        if (two) {
            CK(cudaEventRecord(s->ev[7], st));
            CK(cudaStreamWaitEvent(s->stream2, s->ev[7], 0));
        }
        u32 w0 = 0, wi = 0;
        while (w0 < count) {
            // largest w1 with boff[w1] - boff[w0] <= cap
            u32 lo = w0 + 1, hi = count;
            while (lo < hi) {
                u32 mid = lo + (hi - lo + 1) / 2;
                if (h_boff[mid] - h_boff[w0] <= cap)
                    lo = mid;
                else
                    hi = mid - 1;
            }
            const u32 w1 = lo;
            const bool second = two && (wi & 1);
            cudaStream_t ws = second ? s->stream2 : st;
            a.order = d_order + w0;
            a.boff = d_boff + w0;
            a.boff0 = h_boff[w0];
            a.count = w1 - w0;
            a.scale = scale;
            a.arena = P<u8>(s->arena) + (second ? half : 0);
            auto grid = [&](u32 lp) { return (u32)(((u64)a.count * lp + OD_BLOCK - 1) / OD_BLOCK); };
            cudaEvent_t pe[5];
            for (auto &e : pe)
                if (phase_event(s, &e))
                    return -3;
            CK(cudaEventRecord(pe[0], ws));
            a.lanes_per = s->lanes_front;
            a.perm = nullptr;
            k_front<<<grid(a.lanes_per), OD_BLOCK, s->smem_front, ws>>>(a);
            if (!two && a.count >= 256 && s->group_class) {
                // regroup the wave by what k_front found (straight / if-joins /
                // goto form) so the later phases' resident kernels share code
                if (ensure(s->perm, (u64)a.count * 4 + 16) || ensure(s->cnt4, 64))
                    return -3;
                if (scan_exclusive(s, a.count, Cnt4{{0, 0, 0, 0}}, AddCnt4{},
                                   ClsLoad{a.arena, a.boff, a.boff0},
                                   ClsStore{P<u32>(s->perm), P<Cnt4>(s->cnt4)}, P<Cnt4>(s->cnt4)))
                    return -3;
                a.perm = P<u32>(s->perm);
            }
            CK(cudaEventRecord(pe[1], ws));
            a.lanes_per = s->lanes_lower;
            k_lower<<<grid(a.lanes_per), OD_BLOCK, s->smem_lower, ws>>>(a);
            if (a.wide_joins != ~0u) {
                k_lower_wide<<<grid(a.lanes_per), OD_BLOCK, s->smem_lower, ws>>>(a);
                s->stats.total_launches++;
            }
            CK(cudaEventRecord(pe[2], ws));
            k_fold<<<grid(a.lanes_per), OD_BLOCK, s->smem_lower, ws>>>(a);
            CK(cudaEventRecord(pe[3], ws));
            a.lanes_per = s->lanes_emit;
            k_emit<<<grid(a.lanes_per), OD_BLOCK, s->smem_emit, ws>>>(a);
            if (s->dump_flags & DUMP_BODY) {
                k_export<<<grid(a.lanes_per), OD_BLOCK, 0, ws>>>(a);
                s->stats.total_launches++;
            }
            if (s->sem_on) { // the batched semantic check: one persistent launch per wave
                // each wave stream has its own slot counter and scratch half
                u32 *next = reinterpret_cast<u32 *>(P<u64>(s->semcnt) + (second ? 6 : 7));
                CK(cudaMemsetAsync(next, 0, sizeof(u32), ws));
                const u32 warps = std::min<u32>(kSemBatch, a.count);
                u8 *scr = P<u8>(s->semscratch) + (second ? (u64)kSemBatch * kSemEnvs * kSemLaneBytes : 0);
                SemArgs sa{a.count, next, scr, P<SemResult>(s->semres), s->sem_seed,
                           s->sem_kbase + s->stats.kernels, P<u64>(s->semcnt), s->sem_kmap,
                           s->sem_budget, P<u32>(s->semdef), kSemDeferCap,
                           (u32)std::min<u64>(kSemDeferKB, s->def_kb_left)};
                k_semcheck<<<(warps * 32 + 127) / 128, 128, 0, ws>>>(a, sa);
                s->stats.total_launches++;
            }
            CK(cudaEventRecord(pe[4], ws));
            s->stats.decompile_launches += 4;
            s->stats.total_launches += 4;
            CK(cudaGetLastError());
            w0 = w1;
            ++wi;
        }
        if (two) {
            CK(cudaEventRecord(s->ev[7], s->stream2));
            CK(cudaStreamWaitEvent(st, s->ev[7], 0));
        }
        return 0;
    };
    if (launch_waves(boff.data(), P<u32>(s->order), P<u64>(s->boff), nk, 1))
        return -3;
    // retries: kernels that outgrew their pools (or the staging buffer)
    std::vector<KRes> hr(nk);
    u32 scale = 1;
    std::vector<KSize> zs;
    for (int attempt = 0;; ++attempt) {
        u32 nretry = 0; // counted by k_emit: the results are copied only when some kernel must re-run
        if (d2h_sync(s, &nretry, cnt + 12, 4))
            return -3;
        if (!nretry)
            break;
        CK(cudaMemsetAsync(cnt + 12, 0, 4, st));
        if (d2h_sync(s, hr.data(), a.res, (u64)nk * sizeof(KRes)))
            return -3;
        std::vector<u32> redo;
        bool stage_full = false;
        for (u32 k = 0; k < nk; ++k)
            if (hr[k].status == KS_OOM || hr[k].status == KS_STAGE_FULL) {
                redo.push_back(k);
                stage_full |= hr[k].status == KS_STAGE_FULL;
            }
        if (redo.empty())
            break;
        if (attempt == 8) { // arenas 4^8 x the sized budget: never silently drop a kernel
            g_err = "internal error: " + std::to_string(redo.size()) + " kernels outgrew every arena retry";
            return -3;
        }
        s->stats.retried += redo.size();
        if (stage_full) {
            u64 top = 0;
            if (d2h_sync(s, &top, a.stage_top, 8))
                return -3;
            DevBuf nb;
            u64 want = std::max<u64>(top * 2, s->stage.cap * 2);
            CK(cudaMalloc(&nb.p, want));
            nb.cap = want;
            CK(cudaMemcpyAsync(nb.p, s->stage.p, std::min<u64>(top, s->stage.cap), cudaMemcpyDeviceToDevice, st));
            CK(cudaStreamSynchronize(st));
            cudaFree(s->stage.p);
            s->stage = nb;
            a.stage = P<u8>(s->stage);
            a.stage_cap = s->stage.cap;
            u64 dt = 0;
            if (d2h_sync(s, &dt, s->dtop.p, 8))
                return -3;
            if (s->dump_flags) { // dump pool full: grow it, keep what was written
                u64 xt[2];
                if (d2h_sync(s, xt, s->xtop.p, 16))
                    return -3;
                if (xt[0] > dc.cap || xt[1] > dc.rcap) {
                    const u64 tkeep = std::min<u64>(xt[0], dc.cap), rkeep = std::min<u64>(xt[1], dc.rcap);
                    if (ensure_keep(s->xtext, std::max<u64>(xt[0], dc.cap) * 2, tkeep, st) ||
                        ensure_keep(s->xrec, std::max<u64>(xt[1], dc.rcap) * 2 * sizeof(DumpRec),
                                    rkeep * sizeof(DumpRec), st))
                        return -3;
                    dc.text = P<u8>(s->xtext);
                    dc.cap = s->xtext.cap;
                    dc.rec = P<DumpRec>(s->xrec);
                    dc.rcap = s->xrec.cap / sizeof(DumpRec);
                    const u64 nt[2] = {tkeep, rkeep};
                    CK(cudaMemcpyAsync(s->xtop.p, nt, 16, cudaMemcpyHostToDevice, st));
                    CK(cudaMemcpyAsync(s->xcfg.p, &dc, sizeof(dc), cudaMemcpyHostToDevice, st));
                    CK(cudaStreamSynchronize(st));
                }
            }
            if (dt > a.dcap) { // diagnostic pool full: grow it, keep the records written so far
                const u64 old_cap = a.dcap;
                if (ensure_keep(s->dpool, dt * 2 * sizeof(Diag), old_cap * sizeof(Diag), st))
                    return -3;
                a.dpool = P<Diag>(s->dpool);
                a.dcap = s->dpool.cap / sizeof(Diag);
                CK(cudaMemcpyAsync(s->dtop.p, &old_cap, 8, cudaMemcpyHostToDevice, st));
                CK(cudaStreamSynchronize(st));
            }
        }
        bool oom = false;
        for (u32 k : redo)
            oom |= hr[k].status == KS_OOM;
        if (oom)
            scale *= 4;
        if (zs.empty()) {
            zs.resize(nk);
            if (d2h_sync(s, zs.data(), a.sizes, (u64)nk * sizeof(KSize)))
                return -3;
        }
        std::vector<u64> rb(redo.size() + 1, 0);
        for (size_t i = 0; i < redo.size(); ++i)
            rb[i + 1] = rb[i] + kernel_budget(zs[redo[i]], scale);
        CK(cudaMemcpyAsync(P<u32>(s->order), redo.data(), redo.size() * 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(P<u64>(s->boff), rb.data(), rb.size() * 8, cudaMemcpyHostToDevice, st));
        if (launch_waves(rb.data(), P<u32>(s->order), P<u64>(s->boff), (u32)redo.size(), scale))
            return -3;
        CK(cudaStreamSynchronize(st));
    }
    CK(cudaEventRecord(s->ev[3], st));
    // P4b offsets + gather
    if (scan_exclusive(s, nk, U64Val{0}, AddU64{}, OutLenLoad{a.res}, OutOffStore{P<u64>(s->outoff)},
                       reinterpret_cast<U64Val *>(cnt + 10)))
        return -3;
    u32 cblk[16]; // the chunk's counters: [3] decode overflow, [10..11] output total (u64)
    if (d2h_sync(s, cblk, cnt, sizeof cblk))
        return -3;
    if (cblk[3]) {
        g_err = "internal error: an operand pool bound was exceeded";
        return -3;
    }
    if (s->sem_on && s->sem_budget != 0 && collect_deferred(s, t, len, nlf, a, sem_kb0, fold_local_size))
        return -3;
    u64 tot = 0;
    memcpy(&tot, cblk + 10, 8);
    // tot = sum(len + 1) over non-empty; the last separator is dropped
    u64 chunk_bytes = tot ? tot - 1 : 0;
    u64 base = out_base;
    if (tot && prev_nonempty) {
        // separator between the previous chunk's last source and ours
        if (ensure_keep(s->out, out_base + 1 + chunk_bytes + 16, out_base, st))
            return -3;
        CK(cudaMemsetAsync(P<u8>(s->out) + out_base, '\n', 1, st));
        base += 1;
    }
    if (ensure_keep(s->out, base + chunk_bytes + 16, base, st))
        return -3;
    k_gather<<<(u32)(((u64)nk * 32 + 255) / 256), 256, 0, st>>>(a.res, P<u64>(s->outoff), nk, P<u8>(s->stage),
                                                     P<u8>(s->out), base, base + chunk_bytes);
    s->stats.total_launches++;
    CK(cudaGetLastError());
    CK(cudaEventRecord(s->ev[4], st));
    co->out_bytes = (base - out_base) + chunk_bytes;
    if (!s->keep_records) {
        // totals only: the per-kernel results stay on the device
        if (ensure(s->rstat, 64))
            return -3;
        CK(cudaMemsetAsync(s->rstat.p, 0, 32, st));
        k_res_stats<<<(nk + 255) / 256, 256, 0, st>>>(a.res, nk, P<unsigned long long>(s->rstat));
        s->stats.total_launches++;
        CK(cudaGetLastError());
        u64 tot[4];
        if (d2h_sync(s, tot, s->rstat.p, 32))
            return -3;
        s->stats.instructions += tot[0];
        s->stats.failed += tot[1];
        s->stats.goto_form += tot[2];
        s->stats.fallbacks += tot[3];
        float ms2 = 0;
        cudaEventElapsedTime(&ms2, s->ev[0], s->ev[2]);
        s->stats.ms_parse += ms2;
        cudaEventElapsedTime(&ms2, s->ev[2], s->ev[3]);
        s->stats.ms_decompile += ms2;
        cudaEventElapsedTime(&ms2, s->ev[3], s->ev[4]);
        s->stats.ms_emit += ms2;
        sum_phase_events(s);
        return 0;
    }
    // keep per-kernel results for the host API
    if (d2h_sync(s, hr.data(), a.res, (u64)nk * sizeof(KRes)))
        return -3;
    std::vector<u64> offs(nk);
    if (d2h_sync(s, offs.data(), s->outoff.p, (u64)nk * 8))
        return -3;
    std::vector<u32> ks(nk);
    if (d2h_sync(s, ks.data(), s->kstart.p, (u64)nk * 4))
        return -3;
    // diagnostics: the records of the kept results, spans copied out
    std::vector<Diag> dv;
    {
        u64 dt = 0;
        if (d2h_sync(s, &dt, s->dtop.p, 8))
            return -3;
        dt = std::min<u64>(dt, a.dcap);
        if (dt) {
            dv.resize(dt);
            if (d2h_sync(s, dv.data(), s->dpool.p, dt * sizeof(Diag)))
                return -3;
        }
    }
    // the kept records' listing spans, packed on the device, one D2H
    std::vector<uint4> spans;
    u64 span_bytes = 0;
    auto add_span = [&](u32 off, u32 n) {
        if (n) {
            spans.push_back(make_uint4(off, n, (u32)span_bytes, (u32)(span_bytes >> 32)));
            span_bytes += n;
        }
    };
    for (u32 k = 0; k < nk; ++k)
        if (hr[k].status == KS_OK || hr[k].status == KS_FAILED)
            for (u32 q = 0; q < hr[k].ndiag && hr[k].diag_off + q < dv.size(); ++q) {
                const Diag &d = dv[hr[k].diag_off + q];
                add_span(d.a_off, d.a_len);
                add_span(d.b_off, d.b_len);
            }
    std::string span_text(span_bytes, '\0');
    if (!spans.empty()) {
        DevBuf &sb = s->scan_tmp; // free between scans
        const u64 sl = spans.size() * sizeof(uint4);
        if (ensure(sb, sl + span_bytes + 16))
            return -3;
        CK(cudaMemcpyAsync(sb.p, spans.data(), sl, cudaMemcpyHostToDevice, st));
        k_span_gather<<<(u32)((spans.size() * 32 + 255) / 256), 256, 0, st>>>(t, P<uint4>(sb), (u32)spans.size(),
                                                                           P<u8>(sb) + sl);
        s->stats.total_launches++;
        CK(cudaGetLastError());
        if (d2h_sync(s, &span_text[0], P<u8>(sb) + sl, span_bytes))
            return -3;
    }
    u64 span_pos = 0;
    auto take_span = [&](u32 n, std::string *out) {
        out->assign(span_text, span_pos, n);
        span_pos += n;
    };
    for (u32 k = 0; k < nk; ++k) {
        s->host_kdiag.push_back(s->host_diag.size());
        if (hr[k].status == KS_OK || hr[k].status == KS_FAILED) {
            for (u32 q = 0; q < hr[k].ndiag && hr[k].diag_off + q < dv.size(); ++q) {
                const Diag &d = dv[hr[k].diag_off + q];
                HostDiag h;
                h.line = d.line;
                h.code = d.code;
                h.c = d.c;
                take_span(d.a_len, &h.a);
                take_span(d.b_len, &h.b);
                s->host_diag.push_back(std::move(h));
            }
        } else {
            hr[k].ndiag = 0;
        }
    }
    if (s->dump_flags) {
        // DOT dumps: one record per (kernel, step); a retried kernel wrote
        // its dumps again (identical), so the last record of a key wins
        u64 xt[2];
        if (d2h_sync(s, xt, s->xtop.p, 16))
            return -3;
        const u64 nr = std::min<u64>(xt[1], dc.rcap), nt = std::min<u64>(xt[0], dc.cap);
        std::vector<DumpRec> rv(nr);
        std::string tx(nt, '\0');
        if ((nr && d2h_sync(s, rv.data(), s->xrec.p, nr * sizeof(DumpRec))) ||
            (nt && d2h_sync(s, &tx[0], s->xtext.p, nt)))
            return -3;
        std::vector<std::map<int32_t, std::string>> per(nk);
        for (const DumpRec &d : rv)
            if (d.k < nk && d.off + d.len <= nt)
                per[d.k][d.step] = tx.substr(d.off, d.len);
        for (u32 k = 0; k < nk; ++k) {
            std::vector<std::pair<int32_t, std::string>> v;
            if (hr[k].status == KS_OK || hr[k].status == KS_FAILED)
                for (auto &e : per[k])
                    v.emplace_back(e.first, std::move(e.second));
            s->host_dumps.push_back(std::move(v));
        }
    }
    if (s->sem_on) {
        std::vector<SemResult> sv(nk);
        if (d2h_sync(s, sv.data(), s->semres.p, (u64)nk * sizeof(SemResult)))
            return -3;
        for (u32 k = 0; k < nk; ++k)
            s->host_sem.push_back(ocldec_b200_semcheck{sv[k].status, sv[k].envs, sv[k].hash_asm, sv[k].hash_body});
    }
    for (u32 k = 0; k < nk; ++k) {
        s->host_res.push_back(hr[k]);
        s->host_kernel_off.push_back(base + offs[k]);
        s->host_name_line.push_back(ks[k]);
        s->host_name_off.push_back((u64)hr[k].name_off + hr[k].name_len <= len ? s->chunk_base + hr[k].name_off
                                                                              : ~0ull);
        s->stats.instructions += hr[k].ninstr;
        s->stats.failed += hr[k].status == KS_FAILED;
        s->stats.goto_form += hr[k].status == KS_OK && !hr[k].structured;
        s->stats.fallbacks += hr[k].fallbacks;
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, s->ev[0], s->ev[2]);
    s->stats.ms_parse += ms;
    cudaEventElapsedTime(&ms, s->ev[2], s->ev[3]);
    s->stats.ms_decompile += ms;
    cudaEventElapsedTime(&ms, s->ev[3], s->ev[4]);
    s->stats.ms_emit += ms;
    sum_phase_events(s);
    return 0;
}

int session_init(ocldec_b200_session *s, int device, size_t arena_bytes) {
    s->device = device;
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    s->nsm = prop.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    {
        // Overlapping waves on two streams mixes phase code on the SMs: on
        // chunks of short kernels (C4) that costs more instruction-cache
        // misses than it hides tails; on chunks of long kernels (C5: ~340 KB
        // of listing each, long phase tails) it gains 21 % (measured, C5 100k
        // sample: 74.2 -> 89.9 M instr/s).  Default: long-kernel chunks only.
        const char *ts = getenv("OCLDEC_B200_TWO_STREAMS");
        s->two_mode = ts && *ts == '0' ? 0u : ts && *ts == '1' ? 1u : 2u;
        if (s->two_mode)
            CK(cudaStreamCreateWithFlags(&s->stream2, cudaStreamNonBlocking));
    }
    for (auto &e : s->ev)
        CK(cudaEventCreate(&e));
    CK(cudaStreamCreateWithFlags(&s->cstream, cudaStreamNonBlocking));
    for (auto &e : s->cev)
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    if (!getenv("OCLDEC_B200_NO_PEEK")) {
        CK(cudaHostAlloc(reinterpret_cast<void **>(&s->peek_h), kPeekBytes, cudaHostAllocMapped));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void **>(&s->peek_d), s->peek_h, 0));
    }
    // arena pool for one decompile wave (per-kernel slices sized by arena_budget)
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    s->pool_bytes = arena_bytes ? arena_bytes : std::min<size_t>(free_b * 2 / 5, (size_t)64 << 30);
    s->arena_bytes = s->pool_bytes;
    {
        const char *sb = getenv("OCLDEC_B200_SEM_BUDGET");
        if (sb && *sb)
            s->sem_budget = strtol(sb, nullptr, 0);
        const char *wl = getenv("OCLDEC_B200_WIDE_LOWER");
        s->wide_lower = wl && *wl == '1';
    }
    const char *pe = getenv("OCLDEC_B200_PROF");
    s->prof_on = pe && *pe && *pe != '0';
    // kernels per warp per phase (1, 2, 4, 8, 16 or 32); OCLDEC_B200_KPW sets all
    auto kpw_env = [](const char *name, u32 dflt) {
        const char *kp = getenv(name);
        u32 k = kp && *kp ? (u32)atoi(kp) : dflt;
        return (k == 1 || k == 2 || k == 4 || k == 8 || k == 16 || k == 32) ? k : dflt;
    };
    const u32 kall = kpw_env("OCLDEC_B200_KPW", 1);
    s->lanes_front = 32 / kpw_env("OCLDEC_B200_KPW_FRONT", kall);
    s->lanes_lower = 32 / kpw_env("OCLDEC_B200_KPW_LOWER", kall);
    s->lanes_emit = 32 / kpw_env("OCLDEC_B200_KPW_EMIT", kall);
    // OCLDEC_B200_OCC_{FRONT,LOWER,EMIT}=blocks per SM: caps occupancy with
    // dynamic shared memory (tuning experiments; 0 = no cap)
    auto occ_smem = [](const char *name) -> u32 {
        const char *e = getenv(name);
        u32 occ = e && *e ? (u32)atoi(e) : 0;
        return occ ? (u32)((200u * 1024u) / occ) & ~1023u : 0u;
    };
    {
        const char *g = getenv("OCLDEC_B200_GROUP"); // 0 size only, 1 straight/branching (default), 2 block classes
        s->group_class = g && *g ? (u32)(*g - '0') : 2u;
    }
    s->smem_front = occ_smem("OCLDEC_B200_OCC_FRONT");
    s->smem_lower = occ_smem("OCLDEC_B200_OCC_LOWER");
    s->smem_emit = occ_smem("OCLDEC_B200_OCC_EMIT");
    CK(cudaFuncSetAttribute(k_front, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_lower, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_lower_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    CK(cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    if (ensure(s->prof, 16 * 8))
        return -3;
    CK(cudaMemset(s->prof.p, 0, 16 * 8));
    CK(cudaFuncSetAttribute(k_front, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    CK(cudaFuncSetAttribute(k_lower, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    CK(cudaFuncSetAttribute(k_lower_wide, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    CK(cudaFuncSetAttribute(k_emit, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    CK(cudaFuncSetAttribute(k_fold, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    CK(cudaFuncSetAttribute(k_fold, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    // the stack holds the per-thread pipeline context
    CK(cudaDeviceSetLimit(cudaLimitStackSize, 16 * 1024));
    k_init_roots<<<1, 1, 0, s->stream>>>();
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s->stream));
    return 0;
}

void reset_stats(ocldec_b200_session *s) {
    s->stats = ocldec_b200_stats{};
    s->pev_used = 0;
    if (s->prof_on && s->prof.p)
        cudaMemsetAsync(s->prof.p, 0, 16 * 8, s->stream);
    s->host_res.clear();
    s->host_kernel_off.clear();
    s->host_name_line.clear();
    s->host_name_off.clear();
    s->host_diag.clear();
    s->host_kdiag.clear();
    s->host_dumps.clear();
    s->host_sem.clear();
    s->def_text.clear();
    s->def_ord.clear();
    s->def_kb_left = kSemDeferRunKB;
    s->sem_counted = s->sem_on;
    if (s->sem_on && !ensure(s->semcnt, 8 * sizeof(u64)))
        cudaMemsetAsync(s->semcnt.p, 0, 8 * sizeof(u64), s->stream);
    s->out_len = 0;
}

// Splits a host listing into chunks at ".kernel" line starts.
// As few chunks of at most `target` bytes as fit, of about equal size (every
// phase launch ends in a tail); with first > 0 the first chunk is `first`
// bytes and the rest is balanced.
// Whether the line at p[ls..] has ".kernel" as its first word (the cut
// points of host_chunks).
bool kernel_line(const char *p, size_t len, size_t ls) {
    size_t j = ls;
    while (j < len && (p[j] == ' ' || p[j] == '\t'))
        ++j;
    return j + 7 <= len && memcmp(p + j, ".kernel", 7) == 0 &&
           (j + 7 == len || p[j + 7] == ' ' || p[j + 7] == '\t' || p[j + 7] == '\n' || p[j + 7] == '\r');
}

// ".kernel" lines in p[0, len): a shard's kernel offset.
u64 count_kernel_lines(const char *p, size_t len) {
    u64 n = 0;
    for (size_t ls = 0; ls < len;) {
        n += kernel_line(p, len, ls) ? 1 : 0;
        const void *nlp = memchr(p + ls, '\n', len - ls);
        if (!nlp)
            break;
        ls = (size_t)((const char *)nlp - p) + 1;
    }
    return n;
}

// Chunk plan of the host-buffer path.  The first chunk's load and the last
// chunk's output read-back are the only copies the pipeline cannot hide, so
// with three or more chunks the first and last are made smaller and the
// middle ones larger (up to 1.2 x target, under the 3.75 GiB chunk limit),
// keeping the chunk count (each chunk costs its phase tails).  C4 1M:
// 3.2 GB equal chunks -> 1.9 GB first, 3.9 GB middle, ~1.8 GB last.
// OCLDEC_B200_TAPER=0 keeps equal chunks; `first` (OCLDEC_B200_FIRST_CHUNK)
// fixes the first chunk and splits the rest equally.
std::vector<u64> host_chunks(const char *p, size_t len, size_t target, size_t first) {
    std::vector<u64> starts{0};
    size_t mid = 0;
    if (!first) {
        const size_t nch = len ? (len + target - 1) / target : 1;
        const size_t avg = (len + nch - 1) / nch;
        first = mid = avg;
        const char *tp = getenv("OCLDEC_B200_TAPER");
        if (nch >= 3 && !(tp && *tp == '0')) {
            // 3.625 GiB: room under the 3.75 GiB chunk limit for the
            // boundary's overshoot to the next .kernel line
            const size_t cap = std::min<size_t>(target / 5 * 6, (size_t)0xe8000000ull);
            size_t small = len > (nch - 2) * cap ? (len - (nch - 2) * cap) / 2 : 0;
            small = std::min(std::max(small, avg / 3), avg);
            first = small;
            mid = (len - 2 * small + (nch - 3)) / (nch - 2);
        }
    } else if (len > first) {
        const size_t rem = len - first;
        const size_t nch = (rem + target - 1) / target;
        mid = (rem + nch - 1) / nch;
    }
    size_t next = first;
    while (next < len) {
        // find a line whose first word is exactly ".kernel"
        size_t i = next;
        bool found = false;
        while (i < len) {
            const void *nlp = memchr(p + i, '\n', len - i);
            if (!nlp)
                break;
            size_t ls = (const char *)nlp - p + 1;
            if (kernel_line(p, len, ls)) {
                starts.push_back(ls);
                found = true;
                break;
            }
            i = ls;
        }
        if (!found)
            break;
        next = starts.back() + mid;
    }
    return starts;
}


struct HostRun {
    u64 out_bytes = 0;
    int32_t split_error_line = 0, split_error_kind = 0;
    double device_ms = 0;
    bool want_names = true; // kernel names for the result (not needed by session_run_host)
    std::vector<std::string> names;
};

std::mutex g_cache_mu;
std::map<std::pair<int, size_t>, ocldec_b200_session *> g_cache;

size_t chunk_target() {
    const char *e = getenv("OCLDEC_B200_CHUNK_BYTES");
    if (e && *e) {
        size_t v = strtoull(e, nullptr, 0);
        if (v >= 1)
            return v;
    }
    // 3 GiB: few chunks (each phase launch ends in a tail); a chunk whose
    // comment-stripped copies would push it past 4 GiB is retried smaller.
    // On this host-buffer path 6 tapered chunks (C4 1M) beat 5 near-equal
    // chunks of 3.6 GiB end to end, 134.0 vs 133.5 M instr/s: the larger
    // first load and last read-back cost more than the saved chunk (the
    // device-resident bench passes its own 3.6 GiB chunk starts).
    return (size_t)3 << 30;
}

// Parses an ABI override file (or clears the overrides) and uploads the
// resolved list for build_abi.
int set_overrides(ocldec_b200_session *s, const char *text, size_t len) {
    s->ovr_src.clear();
    s->ovr_host.clear();
    s->ovr_diags.clear();
    s->novr = 0;
    if (!text)
        return 0;
    s->ovr_src.assign(text, len);
    s->ovr_host = parse_overrides(std::string(text, len), &s->ovr_diags);
    if (s->ovr_host.empty())
        return 0;
    if (s->ovr_host.size() > 65535) {
        g_err = "more than 65535 ABI overrides";
        return -1;
    }
    std::vector<AbiOvr> dv;
    std::string blob;
    for (HostOvr &o : s->ovr_host) {
        if (o.dev.kind == OV_ARG) {
            o.dev.name_off = (u32)blob.size();
            o.dev.name_len = (u32)o.tail.size();
            blob += o.tail;
        }
        dv.push_back(o.dev);
    }
    if (ensure(s->dovr, dv.size() * sizeof(AbiOvr)) || ensure(s->dovr_text, blob.size() + 16))
        return -3;
    CK(cudaMemcpy(s->dovr.p, dv.data(), dv.size() * sizeof(AbiOvr), cudaMemcpyHostToDevice));
    if (!blob.empty())
        CK(cudaMemcpy(s->dovr_text.p, blob.data(), blob.size(), cudaMemcpyHostToDevice));
    s->novr = (u32)dv.size();
    return 0;
}

// decompile_listing over a host buffer: chunking at .kernel lines, H2D of
// each chunk, the device pipeline, names back to the host.  Output stays in
// s->out[0, out_bytes).
// With host_out, each chunk's output is copied back into host_out on the copy
// stream while the next chunk runs (host_out must hold out_cap bytes; output
// beyond it is not copied).  The next chunk's text is loaded the same way
// into the other of two text buffers, so the PCIe traffic hides behind the
// decompiler except for the first load and the last store.
int run_host_listing_at(ocldec_b200_session *s, const char *listing, size_t len, int fold_local_size,
                        const char *only_kernel, HostRun *hr, char *host_out, u64 out_cap, size_t target);

int run_host_listing(ocldec_b200_session *s, const char *listing, size_t len, int fold_local_size,
                     const char *only_kernel, HostRun *hr, char *host_out, u64 out_cap) {
    size_t target = chunk_target();
    for (;;) {
        const bool names = hr->want_names;
        *hr = HostRun{};
        hr->want_names = names;
        int rc = run_host_listing_at(s, listing, len, fold_local_size, only_kernel, hr, host_out, out_cap, target);
        if (rc != -5 || target <= (64u << 20))
            return rc == -5 ? -1 : rc;
        target /= 2; // chunk + comment-stripped copies past the u32 range
    }
}

// The semantic check's deferred kernels of one chunk (k_semcheck listed
// them: still running after sem_budget steps): their sections' bytes join
// the run's deferred listing, with their listing ordinals.
int collect_deferred(ocldec_b200_session *s, const u8 *t, u64 len, u32 nlf, const DecompArgs &a, u64 kb0,
                     int fold_local_size) {
    cudaStream_t st = s->stream;
    u32 nd = 0;
    if (d2h_sync(s, &nd, s->semdef.p, 4))
        return -3;
    nd = std::min<u32>(nd, kSemDeferCap);
    if (!nd)
        return 0;
    std::vector<u32> lk(nd + 2);
    if (d2h_sync(s, lk.data(), s->semdef.p, 4ull * (nd + 2)) || ensure(s->semspan, 24ull * nd + 16))
        return -3;
    s->def_kb_left -= std::min<u64>(s->def_kb_left, std::min<u64>(lk[1], kSemDeferKB));
    u64 *span = P<u64>(s->semspan);
    k_def_spans<<<(nd + 127) / 128, 128, 0, st>>>(P<u32>(s->semdef), nd, P<u32>(s->nlpos), nlf, a.kstart, a.nk, len,
                                                   span);
    std::vector<u64> sp(2ull * nd);
    if (d2h_sync(s, sp.data(), span, 16ull * nd))
        return -3;
    std::vector<u64> dst(nd);
    u64 tot = 0;
    for (u32 j = 0; j < nd; ++j) {
        dst[j] = tot;
        tot += sp[2 * j + 1];
    }
    if (ensure(s->semdefbuf, tot + 16))
        return -3;
    CK(cudaMemcpyAsync(span + 2ull * nd, dst.data(), 8ull * nd, cudaMemcpyHostToDevice, st));
    k_def_pack<<<(nd * 32 + 127) / 128, 128, 0, st>>>(t, span, span + 2ull * nd, nd, P<u8>(s->semdefbuf));
    std::string bytes(tot, '\0');
    if (d2h_sync(s, bytes.data(), s->semdefbuf.p, tot))
        return -3;
    for (u32 j = 0; j < nd; ++j) {
        s->def_text.append(bytes, dst[j], sp[2 * j + 1]);
        if (s->def_text.empty() || s->def_text.back() != '\n')
            s->def_text += '\n';
        s->def_ord.push_back(s->sem_kbase + kb0 + lk[2 + j]);
    }
    s->def_fold = fold_local_size;
    return 0;
}

// The run's deferred kernels, re-checked together without a step budget on
// an auxiliary session (same device, seed, fold and ABI options; each kernel
// keyed by its ordinal in this run's listing, so its environments are the
// ones the in-wave check would have used).  The verdicts replace the
// deferred placeholders: per kernel (host records) and in the status counts.
int finish_deferred(ocldec_b200_session *s) {
    if (s->def_ord.empty())
        return 0;
    if (!s->aux) {
        s->aux = ocldec_b200_session_create(s->device, 1ull << 30);
        if (!s->aux)
            return -3;
    }
    ocldec_b200_session *x = s->aux;
    const size_t n = s->def_ord.size();
    if (ensure(x->semkmap, 8ull * n + 8))
        return -3;
    CK(cudaMemcpy(x->semkmap.p, s->def_ord.data(), 8ull * n, cudaMemcpyHostToDevice));
    x->keep_records = true;
    x->sem_on = true;
    x->sem_seed = s->sem_seed;
    x->sem_budget = 0;
    x->sem_kbase = 0;
    x->sem_kmap = P<u64>(x->semkmap);
    int rc = set_overrides(x, s->ovr_src.empty() ? nullptr : s->ovr_src.data(), s->ovr_src.size());
    HostRun hr;
    if (!rc)
        rc = run_host_listing(x, s->def_text.data(), s->def_text.size(), s->def_fold, nullptr, &hr, nullptr, 0);
    x->sem_kmap = nullptr;
    x->sem_on = false;
    if (rc) {
        g_err = "semantic re-check of deferred kernels: " + g_err;
        return rc;
    }
    if (x->host_sem.size() != n) {
        g_err = "internal error: deferred semantic re-check lost kernels";
        return -3;
    }
    u64 cnt[8];
    CK(cudaMemcpyAsync(cnt, s->semcnt.p, sizeof cnt, cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    for (size_t i = 0; i < n; ++i) {
        const ocldec_b200_semcheck &r = x->host_sem[i];
        if (r.status < 6)
            ++cnt[r.status];
        const u64 idx = s->def_ord[i] - s->sem_kbase;
        if (idx < s->host_sem.size())
            s->host_sem[idx] = r;
    }
    CK(cudaMemcpyAsync(s->semcnt.p, cnt, 6 * sizeof(u64), cudaMemcpyHostToDevice, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    s->def_text.clear();
    s->def_ord.clear();
    return 0;
}

int run_host_listing_at(ocldec_b200_session *s, const char *listing, size_t len, int fold_local_size,
                        const char *only_kernel, HostRun *hr, char *host_out, u64 out_cap, size_t target) {
    reset_stats(s);
    s->stats.in_bytes = len;
    s->only_len = 0;
    if (only_kernel) {
        u32 ol = (u32)strlen(only_kernel);
        if (ensure(s->only, ol + 8))
            return -3;
        CK(cudaMemcpy(s->only.p, only_kernel, ol, cudaMemcpyHostToDevice));
        s->only_len = ol;
        s->only_set = true;
    } else {
        s->only_set = false;
    }
    // equal chunks (0); OCLDEC_B200_FIRST_CHUNK=bytes makes the first one
    // that size instead (a smaller first load, one more chunk: measured slower)
    size_t first = 0;
    if (const char *e = getenv("OCLDEC_B200_FIRST_CHUNK"))
        first = strtoull(e, nullptr, 0);
    std::vector<u64> starts = host_chunks(listing, len, target, first);
    const size_t nch = starts.size();
    auto cb = [&](size_t c) { return starts[c]; };
    auto ce = [&](size_t c) { return c + 1 < nch ? starts[c + 1] : (u64)len; };
    u64 maxn = 0;
    for (size_t c = 0; c < nch; ++c)
        maxn = std::max<u64>(maxn, ce(c) - cb(c));
    DevBuf *tb[2] = {&s->text, &s->text2};
    if (ensure(s->text, 2 * maxn + 4096) || (nch > 1 && ensure(s->text2, 2 * maxn + 4096)))
        return -3;
    auto load = [&](size_t c) -> int {
        const u64 n = ce(c) - cb(c);
        if (n)
            CK(cudaMemcpyAsync(tb[c & 1]->p, listing + cb(c), n, cudaMemcpyHostToDevice, s->cstream));
        CK(cudaEventRecord(s->cev[c & 1], s->cstream));
        return 0;
    };
    u64 out_pos = 0;
    u32 line_base = 0;
    bool nonempty = false;
    cudaEvent_t e0 = s->ev[5], e1 = s->ev[6];
    CK(cudaEventRecord(e0, s->stream));
    if (nch && load(0))
        return -3;
    for (size_t c = 0; c < nch; ++c) {
        u64 b = cb(c);
        u64 n = ce(c) - b;
        // the other buffer's chunk (c - 1) is finished: run_chunk returns synchronized
        if (c + 1 < nch && load(c + 1))
            return -3;
        CK(cudaStreamWaitEvent(s->stream, s->cev[c & 1], 0));
        u8 *tc = P<u8>(*tb[c & 1]);
        ChunkOut co;
        size_t before = s->host_res.size();
        s->chunk_base = b;
        int rc = run_chunk(s, tc, n, true, line_base, fold_local_size, out_pos, nonempty, &co);
        if (rc) {
            cudaStreamSynchronize(s->cstream);
            return rc;
        }
        if (host_out && co.err_line == 0xffffffffu && co.out_bytes && out_pos + co.out_bytes <= out_cap) {
            CK(cudaEventRecord(s->cev[2], s->stream));
            CK(cudaStreamWaitEvent(s->cstream, s->cev[2], 0));
            CK(cudaMemcpyAsync(host_out + out_pos, P<u8>(s->out) + out_pos, co.out_bytes, cudaMemcpyDeviceToHost,
                               s->cstream));
        }
        if (co.err_line != 0xffffffffu) {
            hr->split_error_line = (int32_t)(line_base + co.err_line + 1);
            hr->split_error_kind = (int32_t)co.err_kind;
            s->host_res.clear();
            s->host_kernel_off.clear();
            s->host_diag.clear();
            s->host_kdiag.clear();
            s->host_dumps.clear();
            hr->names.clear();
            out_pos = 0;
            break;
        }
        for (size_t k = before; hr->want_names && k < s->host_res.size(); ++k) {
            const KRes &r = s->host_res[k];
            std::string nm;
            if (r.name_off + (u64)r.name_len <= n) {
                nm.assign(listing + b + r.name_off, r.name_len);
            } else {
                nm.resize(r.name_len);
                if (r.name_len)
                    CK(cudaMemcpy(&nm[0], tc + r.name_off, r.name_len, cudaMemcpyDeviceToHost));
            }
            hr->names.push_back(nm);
        }
        out_pos += co.out_bytes;
        nonempty = nonempty || co.out_bytes > 0;
        line_base += co.nlines;
        s->stats.lines += co.nlines;
        s->stats.kernels += co.nk;
    }
    CK(cudaEventRecord(e1, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaStreamSynchronize(s->cstream));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    hr->device_ms = ms;
    hr->out_bytes = out_pos;
    s->out_len = out_pos;
    s->stats.out_bytes = out_pos;
    return finish_deferred(s);
}

} // namespace

// ================================================================== C ABI
extern "C" {

const char *ocldec_b200_last_error(void) { return g_err.c_str(); }
int ocldec_b200_version(void) { return OCLDEC_B200_ABI_VERSION; }

ocldec_b200_session *ocldec_b200_session_create(int device, size_t arena_bytes) {
    auto *s = new ocldec_b200_session();
    if (session_init(s, device, arena_bytes)) {
        delete s;
        return nullptr;
    }
    return s;
}

void ocldec_b200_session_destroy(ocldec_b200_session *s) {
    if (!s)
        return;
    if (s->aux)
        ocldec_b200_session_destroy(s->aux);
    cudaSetDevice(s->device);
    DevBuf *bufs[] = {&s->text, &s->text2, &s->tiles, &s->tiles_off, &s->nlpos, &s->lines, &s->lins, &s->ops_cnt,
                      &s->labs_cnt, &s->ops_off, &s->labs_off, &s->ops, &s->labs, &s->kstart,
                      &s->scan_tmp, &s->scan_tot, &s->counters, &s->arena, &s->stage, &s->res,
                      &s->outoff, &s->out, &s->only, &s->retry, &s->gen_len, &s->gen_ninstr,
                      &s->gen_buf, &s->gen_off, &s->kmeta, &s->order, &s->budget, &s->sbudget,
                      &s->boff, &s->hist, &s->prof, &s->ksizes, &s->dpool, &s->dtop, &s->perm, &s->cnt4,
                      &s->dovr, &s->dovr_text, &s->xtext, &s->xrec, &s->xtop, &s->xcfg, &s->sgen, &s->rstat, &s->semres, &s->semscratch, &s->semcnt, &s->semkmap, &s->semdef, &s->semspan, &s->semdefbuf};
    for (DevBuf *b : bufs)
        if (b->p)
            cudaFree(b->p);
    for (auto &e : s->ev)
        cudaEventDestroy(e);
    for (auto &e : s->pev)
        cudaEventDestroy(e);
    if (s->stream)
        cudaStreamDestroy(s->stream);
    if (s->stream2)
        cudaStreamDestroy(s->stream2);
    if (s->cstream)
        cudaStreamDestroy(s->cstream);
    if (s->peek_h)
        cudaFreeHost(s->peek_h);
    for (auto &e : s->cev)
        cudaEventDestroy(e);
    delete s;
}

void *ocldec_b200_session_stream(ocldec_b200_session *s) { return s ? (void *)s->stream : nullptr; }

int ocldec_b200_session_run(ocldec_b200_session *s, const void *d_listing, size_t len,
                            const uint64_t *chunk_starts, size_t nchunks, int fold_local_size, int sync) {
    if (!s || (!d_listing && len)) {
        g_err = "bad arguments";
        return -1;
    }
    CK(cudaSetDevice(s->device));
    reset_stats(s);
    s->only_set = false;
    set_overrides(s, nullptr, 0);
    s->stats.in_bytes = len;
    u64 out_pos = 0;
    u32 line_base = 0;
    bool nonempty = false;
    const u8 *base = static_cast<const u8 *>(d_listing);
    if (nchunks == 0) {
        static const uint64_t zero = 0;
        chunk_starts = &zero;
        nchunks = 1;
    }
    for (size_t c = 0; c < nchunks; ++c) {
        u64 b = chunk_starts[c];
        u64 e = c + 1 < nchunks ? chunk_starts[c + 1] : len;
        ChunkOut co;
        s->chunk_base = b;
        int rc = run_chunk(s, base + b, e - b, false, line_base, fold_local_size, out_pos, nonempty, &co);
        if (rc)
            return rc == -5 ? -1 : rc; // (chunk + comment-stripped copies: the caller picks smaller chunks)
        if (co.err_line != 0xffffffffu) {
            g_err = "split_kernels error";
            s->stats.lines += co.nlines;
            return -4;
        }
        out_pos += co.out_bytes;
        nonempty = nonempty || co.out_bytes > 0;
        // next chunk's first line number: lines so far (chunk ends right after a '\n')
        line_base += co.nlines;
        s->stats.lines += co.nlines;
        s->stats.kernels += co.nk;
    }
    s->out_len = out_pos;
    s->stats.out_bytes = out_pos;
    if (int rc = finish_deferred(s))
        return rc;
    if (sync)
        CK(cudaStreamSynchronize(s->stream));
    return 0;
}

int ocldec_b200_session_set_records(ocldec_b200_session *s, int keep) {
    if (!s)
        return -1;
    s->keep_records = keep != 0;
    return 0;
}

int ocldec_b200_session_set_semantic(ocldec_b200_session *s, int on, uint64_t seed) {
    if (!s)
        return -1;
    s->sem_session = s->sem_on = on != 0;
    s->sem_session_seed = s->sem_seed = seed;
    return 0;
}

int ocldec_b200_session_semantic_counts(ocldec_b200_session *s, uint64_t counts[6]) {
    if (!s || !counts)
        return -1;
    u64 c[8] = {};
    if (s->sem_counted && s->semcnt.p) {
        CK(cudaSetDevice(s->device));
        CK(cudaMemcpyAsync(c, s->semcnt.p, sizeof c, cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
    }
    for (int i = 0; i < 6; ++i)
        counts[i] = c[i];
    return 0;
}

int ocldec_b200_copy(void *dst, const void *src, uint64_t n) {
    CK(cudaMemcpy(dst, src, n, cudaMemcpyDefault));
    return 0;
}

int ocldec_b200_session_stats(ocldec_b200_session *s, ocldec_b200_stats *st) {
    if (!s || !st)
        return -1;
    if (s->prof_on)
        CK(cudaMemcpy(s->stats.prof_cycles, s->prof.p, sizeof(s->stats.prof_cycles), cudaMemcpyDeviceToHost));
    *st = s->stats;
    return 0;
}

int ocldec_b200_session_output(ocldec_b200_session *s, const void **d_out, uint64_t *len) {
    if (!s)
        return -1;
    *d_out = s->out.p;
    *len = s->out_len;
    return 0;
}

int ocldec_b200_session_kernels(ocldec_b200_session *s, uint64_t *off, uint64_t *len, uint32_t *flags,
                                uint32_t *fallbacks) {
    if (!s)
        return -1;
    for (size_t k = 0; k < s->host_res.size(); ++k) {
        const KRes &r = s->host_res[k];
        if (off)
            off[k] = s->host_kernel_off[k];
        if (len)
            len[k] = r.status == KS_OK ? r.out_len : 0;
        if (flags)
            flags[k] = (r.status == KS_FAILED ? 1u : 0u) | (r.structured ? 2u : 0u) |
                       (r.status == KS_SKIP ? 4u : 0u);
        if (fallbacks)
            fallbacks[k] = r.fallbacks;
    }
    return 0;
}

int ocldec_b200_session_names(ocldec_b200_session *s, uint64_t *off, uint32_t *len) {
    if (!s)
        return -1;
    for (size_t k = 0; k < s->host_res.size(); ++k) {
        if (off)
            off[k] = s->host_name_off[k];
        if (len)
            len[k] = s->host_res[k].name_len;
    }
    return 0;
}

int ocldec_b200_session_diagnostics(ocldec_b200_session *s, char *buf, uint64_t cap, uint64_t *need) {
    if (!s || (!buf && cap))
        return -1;
    std::string out;
    int n = 0;
    for (size_t k = 0; k < s->host_res.size() && k < s->host_kdiag.size(); ++k) {
        const KRes &r = s->host_res[k];
        if (r.status == KS_SKIP)
            continue;
        for (u32 q = 0; q < r.ndiag; ++q) {
            const HostDiag &h = s->host_diag[s->host_kdiag[k] + q];
            out += std::to_string(diag_severity(h.code)) + " " + std::to_string(h.line) + " " +
                   diag_message(h, &s->ovr_host) + "\n";
            ++n;
        }
    }
    if (need)
        *need = out.size() + 1;
    if (out.size() + 1 > cap) {
        g_err = "diagnostics buffer too small";
        return -2;
    }
    memcpy(buf, out.data(), out.size());
    buf[out.size()] = 0;
    return n;
}

} // extern "C"

namespace {

// One shard of a decompile call: a contiguous run of kernel sections of the
// caller's listing, decompiled on one session (one device).  SURVEY §8(e):
// the only cross-shard coupling is the placement computed from each shard's
// {out_bytes, lines, split error, kernels} tuple.
struct Shard {
    ocldec_b200_session *s = nullptr;
    const char *p = nullptr;
    size_t len = 0;
    HostRun hr;
    int rc = 0;
    std::string err;       // g_err of the shard's thread
    u64 lines = 0;         // listing lines in the shard
    u64 line_base = 0;     // lines before the shard
    u64 out_off = 0;       // where its text goes in combined_source
    bool lead_nl = false;  // a "\n" separator precedes it
    u64 kbase = 0;         // .kernel sections before the shard (semantic-check environment keys)
};

void run_shard(Shard &sh, const ocldec_b200_options &o) {
    ocldec_b200_session *s = sh.s;
    sh.rc = 0;
    if (cudaSetDevice(s->device) != cudaSuccess) {
        sh.rc = -3;
        sh.err = "cudaSetDevice failed";
        return;
    }
    if (int rc0 = set_overrides(s, o.abi_map, o.abi_map ? o.abi_map_len : 0)) {
        sh.rc = rc0;
        sh.err = g_err;
        return;
    }
    s->dump_flags = (o.dump_cfg ? DUMP_CFG : 0u) | (o.dump_regions ? DUMP_REGIONS : 0u) |
                    (o.record_reduction ? DUMP_MERGES : 0u) | (o.export_body ? DUMP_BODY : 0u);
    s->sem_on = o.semantic_check != 0;
    s->sem_seed = o.semantic_seed;
    s->sem_kbase = sh.kbase;
    sh.rc = run_host_listing(s, sh.p, sh.len, o.fold_local_size, o.only_kernel, &sh.hr, nullptr, 0);
    s->sem_kbase = 0;
    s->dump_flags = 0;
    s->sem_on = s->sem_session;
    s->sem_seed = s->sem_session_seed;
    sh.lines = s->stats.lines;
    if (sh.rc)
        sh.err = g_err;
}

// The shard's combined output into the result buffer at its placement.
void copy_shard_out(Shard &sh, char *combined) {
    if (!sh.hr.out_bytes)
        return;
    if (cudaSetDevice(sh.s->device) != cudaSuccess ||
        cudaMemcpyAsync(combined + sh.out_off, sh.s->out.p, sh.hr.out_bytes, cudaMemcpyDeviceToHost,
                        sh.s->stream) != cudaSuccess ||
        cudaStreamSynchronize(sh.s->stream) != cudaSuccess) {
        sh.rc = -3;
        sh.err = "device to host copy of the combined output failed";
        return;
    }
    if (sh.lead_nl)
        combined[sh.out_off - 1] = '\n';
}

// Runs fn(i) for every shard, one host thread per shard when there are
// several (one per device: each thread drives its own session's stream).
template <class Fn> void for_shards(std::vector<Shard> &sh, Fn fn) {
    if (sh.size() == 1) {
        fn(0);
        return;
    }
    std::vector<std::thread> th;
    for (size_t i = 0; i < sh.size(); ++i)
        th.emplace_back([&, i] { fn(i); });
    for (auto &t : th)
        t.join();
}

// A shard's step -4 flow-graph record with its terminator lines (field 8 of
// each "B" line, od_kernel.cuh cfg_text) moved to listing lines.
std::string shift_cfg_lines(const std::string &t, u64 base) {
    std::string o;
    o.reserve(t.size() + 64);
    size_t i = 0;
    while (i < t.size()) {
        size_t e = t.find('\n', i);
        if (e == std::string::npos)
            e = t.size();
        if (t.compare(i, 2, "B ") == 0) {
            size_t f = i; // start of field 8 (the line)
            for (int w = 0; w < 7 && f < e; ++w)
                f = t.find(' ', f) + 1;
            size_t g = t.find(' ', f);
            if (f > i && g != std::string::npos && g < e) {
                const u64 line = strtoull(t.c_str() + f, nullptr, 10);
                o.append(t, i, f - i);
                o += std::to_string(line ? line + base : 0);
                o.append(t, g, e - g);
            } else {
                o.append(t, i, e - i);
            }
        } else {
            o.append(t, i, e - i);
        }
        if (e < t.size())
            o += '\n';
        i = e + 1;
    }
    return o;
}

// decompile_listing over shards: run, place, copy out, and assemble the
// DecompileResult (decompiler.cpp:117-133 / combined_source :105-115).
int decompile_shards(std::vector<Shard> &sh, const ocldec_b200_options &o, ocldec_b200_result **out) {
    for_shards(sh, [&](size_t i) { run_shard(sh[i], o); });
    for (Shard &x : sh)
        if (x.rc) {
            g_err = x.err;
            return x.rc;
        }
    // placement: the one exchange step (here within the process)
    int32_t err_line = 0, err_kind = 0;
    u64 lines = 0, pos = 0;
    bool any = false;
    double dev_ms = 0;
    for (Shard &x : sh) {
        x.line_base = lines;
        if (!err_line && x.hr.split_error_line > 0) {
            err_line = (int32_t)(lines + x.hr.split_error_line);
            err_kind = x.hr.split_error_kind;
        }
        lines += x.lines;
        dev_ms = std::max(dev_ms, x.hr.device_ms);
        if (x.hr.out_bytes) {
            x.lead_nl = any;
            pos += any ? 1 : 0;
            x.out_off = pos;
            pos += x.hr.out_bytes;
            any = true;
        }
    }
    const u64 out_len = err_line ? 0 : pos;
    auto *res = static_cast<ocldec_b200_result *>(calloc(1, sizeof(ocldec_b200_result)));
    res->split_error_line = err_line;
    res->split_error_kind = err_kind;
    res->device_ms = dev_ms;
    res->combined = static_cast<char *>(malloc(out_len + 1));
    res->combined[out_len] = 0;
    res->combined_len = out_len;
    if (!err_line) {
        for_shards(sh, [&](size_t i) { copy_shard_out(sh[i], res->combined); });
        for (Shard &x : sh)
            if (x.rc) {
                g_err = x.err;
                ocldec_b200_free(res);
                return x.rc;
            }
    }
    u64 nk_all = 0;
    for (Shard &x : sh)
        nk_all += err_line ? 0 : x.s->host_res.size();
    res->kernels = static_cast<ocldec_b200_kernel *>(calloc(nk_all + 1, sizeof(ocldec_b200_kernel)));
    if (o.semantic_check)
        res->sem = static_cast<ocldec_b200_semcheck *>(calloc(nk_all + 1, sizeof(ocldec_b200_semcheck)));
    std::string nm;
    u64 nkept = 0;
    std::vector<ocldec_b200_dump> dv;
    std::string dtx;
    std::vector<ocldec_b200_diag> dl;
    std::string dt;
    auto add = [&](int sev, int line, const std::string &msg) {
        ocldec_b200_diag d;
        d.severity = sev;
        d.line = line;
        d.msg_off = dt.size();
        d.msg_len = msg.size();
        dt += msg;
        dl.push_back(d);
    };
    if (err_line) {
        static const char *kSplit[] = {"parse error", ".kernel directive without a name",
                                       ".config outside of a .kernel section", ".text outside of a .kernel section"};
        add(2, err_line, kSplit[err_kind >= 1 && err_kind <= 3 ? err_kind : 0]);
    } else {
        for (Shard &x : sh) {
            ocldec_b200_session *s = x.s;
            const size_t nk = s->host_res.size();
            for (size_t k = 0; k < nk; ++k) {
                const KRes &r = s->host_res[k];
                if (r.status == KS_SKIP)
                    continue;
                ocldec_b200_kernel &K = res->kernels[nkept];
                K.name_off = nm.size();
                K.name_len = x.hr.names[k].size();
                nm += x.hr.names[k];
                K.src_off = x.out_off + s->host_kernel_off[k];
                K.src_len = r.status == KS_OK ? r.out_len : 0;
                K.failed = r.status == KS_FAILED;
                K.structured = r.structured;
                K.fallback_count = (int32_t)r.fallbacks;
                K.instructions = r.ninstr;
                res->instructions += r.ninstr;
                if (res->sem && k < s->host_sem.size())
                    res->sem[nkept] = s->host_sem[k];
                // DecompiledKernel::cfg_dot and ReduceResult::dumps
                if (k < s->host_dumps.size())
                    for (const auto &e : s->host_dumps[k]) {
                        ocldec_b200_dump d{};
                        d.kernel = nkept;
                        d.step = e.first;
                        d.off = dtx.size();
                        if (e.first == -4 && x.line_base)
                            dtx += shift_cfg_lines(e.second, x.line_base);
                        else
                            dtx += e.second;
                        d.len = dtx.size() - d.off;
                        dv.push_back(d);
                    }
                // DecompileResult::diagnostics in sink order (line 0: override
                // errors, not listing lines)
                for (u32 q = 0; q < r.ndiag; ++q) {
                    const HostDiag &h = s->host_diag[s->host_kdiag[k] + q];
                    add(diag_severity(h.code), h.line ? (int)(h.line + x.line_base) : 0,
                        diag_message(h, &s->ovr_host));
                }
                ++nkept;
            }
        }
    }
    res->nkernels = nkept;
    res->ndumps = dv.size();
    res->dumps = static_cast<ocldec_b200_dump *>(malloc((dv.size() + 1) * sizeof(ocldec_b200_dump)));
    if (!dv.empty())
        memcpy(res->dumps, dv.data(), dv.size() * sizeof(ocldec_b200_dump));
    res->dump_text = static_cast<char *>(malloc(dtx.size() + 1));
    memcpy(res->dump_text, dtx.data(), dtx.size());
    res->dump_text[dtx.size()] = 0;
    res->names = static_cast<char *>(malloc(nm.size() + 1));
    memcpy(res->names, nm.data(), nm.size());
    res->names[nm.size()] = 0;
    const size_t nk_diags = dl.size();
    for (const OvrDiag &d : sh[0].s->ovr_diags)
        add(d.sev, d.line, d.msg);
    res->ndiags = nk_diags;
    res->nabi_diags = dl.size() - nk_diags;
    res->diags = static_cast<ocldec_b200_diag *>(malloc((dl.size() + 1) * sizeof(ocldec_b200_diag)));
    if (!dl.empty())
        memcpy(res->diags, dl.data(), dl.size() * sizeof(ocldec_b200_diag));
    res->abi_diags = res->diags + nk_diags;
    res->diag_text = static_cast<char *>(malloc(dt.size() + 1));
    memcpy(res->diag_text, dt.data(), dt.size());
    res->diag_text[dt.size()] = 0;
    *out = res;
    return 0;
}

// The cached session for (device, arena, slot): slot > 0 when one call puts
// several shards on the same device.
ocldec_b200_session *cached_session(int device, size_t arena, int slot) {
    ocldec_b200_session *&s = g_cache[{device, arena + (size_t)slot * 0x100000000000000ull}];
    if (!s)
        s = ocldec_b200_session_create(device, arena);
    return s;
}

} // namespace

extern "C" {

int ocldec_b200_decompile(const char *listing, size_t len, const ocldec_b200_options *opts,
                          ocldec_b200_result **out) {
    if (!out || (!listing && len)) {
        g_err = "bad arguments";
        return -1;
    }
    *out = nullptr;
    ocldec_b200_options o{};
    if (opts)
        o = *opts;
    std::lock_guard<std::mutex> lock(g_cache_mu);
    std::vector<Shard> sh(1);
    sh[0].s = cached_session(o.device, o.arena_bytes, 0);
    if (!sh[0].s)
        return -3;
    sh[0].p = listing;
    sh[0].len = len;
    return decompile_shards(sh, o, out);
}

int ocldec_b200_decompile_multi(const char *listing, size_t len, const ocldec_b200_options *opts,
                                const int *devices, int ndevices, ocldec_b200_result **out) {
    if (!out || (!listing && len) || !devices || ndevices < 1) {
        g_err = "bad arguments";
        return -1;
    }
    *out = nullptr;
    ocldec_b200_options o{};
    if (opts)
        o = *opts;
    std::lock_guard<std::mutex> lock(g_cache_mu);
    // byte-balanced shards cut at ".kernel" lines (fewer when the listing has
    // fewer sections than devices)
    const size_t target = std::max<size_t>(1, (len + ndevices - 1) / (size_t)ndevices);
    std::vector<u64> starts = host_chunks(listing, len, target, 0);
    if (starts.size() > (size_t)ndevices)
        starts.resize((size_t)ndevices);
    std::vector<Shard> sh(starts.size());
    for (size_t i = 0; i < sh.size(); ++i) {
        int slot = 0;
        for (size_t j = 0; j < i; ++j)
            slot += devices[j] == devices[i];
        sh[i].s = cached_session(devices[i], o.arena_bytes, slot);
        if (!sh[i].s)
            return -3;
        sh[i].p = listing + starts[i];
        sh[i].len = (i + 1 < sh.size() ? starts[i + 1] : (u64)len) - starts[i];
        if (o.semantic_check && i > 0)
            sh[i].kbase = sh[i - 1].kbase + count_kernel_lines(sh[i - 1].p, sh[i - 1].len);
    }
    return decompile_shards(sh, o, out);
}

int ocldec_b200_session_run_host(ocldec_b200_session *s, const char *listing, size_t len,
                                 int fold_local_size, char *host_out, uint64_t out_cap,
                                 uint64_t *out_len) {
    if (!s || (!listing && len) || !out_len) {
        g_err = "bad arguments";
        return -1;
    }
    CK(cudaSetDevice(s->device));
    HostRun hr;
    set_overrides(s, nullptr, 0);
    hr.want_names = false;
    int rc = run_host_listing(s, listing, len, fold_local_size, nullptr, &hr, host_out, host_out ? out_cap : 0);
    if (rc)
        return rc;
    *out_len = hr.out_bytes;
    if (hr.out_bytes > out_cap || !host_out) {
        g_err = "output buffer too small";
        return -2;
    }
    return 0;
}

int ocldec_b200_abi_map_check(const char *text, size_t len, char *buf, size_t cap) {
    if ((!text && len) || (!buf && cap)) {
        g_err = "bad arguments";
        return -1;
    }
    std::vector<OvrDiag> d;
    parse_overrides(std::string(text ? text : "", len), &d);
    std::string out;
    int errors = 0;
    for (const OvrDiag &x : d) {
        out += std::to_string(x.sev) + " " + std::to_string(x.line) + " " + x.msg + "\n";
        errors += x.sev == 2;
    }
    if (out.size() + 1 > cap)
        return -2;
    memcpy(buf, out.data(), out.size());
    buf[out.size()] = 0;
    return errors;
}

void ocldec_b200_free(ocldec_b200_result *res) {
    if (!res)
        return;
    free(res->kernels);
    free(res->names);
    free(res->combined);
    free(res->dumps);
    free(res->dump_text);
    free(res->sem);
    free(res->diags); // abi_diags points into the same array
    free(res->diag_text);
    free(res);
}

int64_t ocldec_b200_gen_host(int shape, int stress, uint64_t seed, uint64_t k0, uint64_t count, char *buf,
                             uint64_t cap, uint64_t *offsets, uint64_t *instructions, uint64_t *needed) {
    GenCfg g{(u32)shape, (u32)stress, seed};
    u64 total = 0, ni = 0;
    for (u64 i = 0; i < count; ++i) {
        Writer w{nullptr, 0, 0, false};
        ni += gen_kernel(g, k0 + i, &w);
        if (offsets)
            offsets[i] = total;
        total += w.n;
    }
    if (offsets)
        offsets[count] = total;
    if (needed)
        *needed = total;
    if (instructions)
        *instructions = ni;
    if (!buf)
        return (int64_t)total;
    if (total > cap)
        return -2;
    for (u64 i = 0; i < count; ++i) {
        u64 off = offsets ? offsets[i] : 0;
        Writer w{reinterpret_cast<u8 *>(buf) + off, 0, 0xffffffffu, false};
        gen_kernel(g, k0 + i, &w);
    }
    return (int64_t)total;
}

int ocldec_b200_gen_device(ocldec_b200_session *s, int shape, int stress, uint64_t seed, uint64_t k0,
                           uint64_t count, const void **d_buf, uint64_t *len, const uint64_t **d_offsets,
                           uint64_t *instructions) {
    if (!s)
        return -1;
    CK(cudaSetDevice(s->device));
    if (ensure(s->gen_len, (count + 1) * 8) || ensure(s->gen_ninstr, (count + 1) * 4) ||
        ensure(s->gen_off, (count + 1) * 8) || ensure(s->counters, 64))
        return -3;
    GenArgs a;
    a.cfg = GenCfg{(u32)shape, (u32)stress, seed};
    a.k0 = k0;
    a.count = count;
    a.len = P<u64>(s->gen_len);
    a.ninstr = P<u32>(s->gen_ninstr);
    a.buf = nullptr;
    a.base = 0;
    CK(cudaMemsetAsync(a.len + count, 0, 8, s->stream));
    k_gen<<<(u32)((count + 127) / 128), 128, 0, s->stream>>>(a, 0);
    CK(cudaGetLastError());
    // offsets = exclusive scan of lengths (count + 1 entries, last = total)
    if (scan_exclusive(s, count + 1, U64Val{0}, AddU64{}, U64Load{a.len}, U64Store{P<u64>(s->gen_off)},
                       reinterpret_cast<U64Val *>(P<u32>(s->counters) + 8)))
        return -3;
    u64 total = 0;
    if (d2h_sync(s, &total, P<u64>(s->gen_off) + count, 8))
        return -3;
    // instruction total
    if (scan_exclusive(s, count, U64Val{0}, AddU64{}, U32SumLoad64{a.ninstr}, U64Store{a.len},
                       reinterpret_cast<U64Val *>(P<u32>(s->counters) + 12)))
        return -3;
    u64 ni = 0;
    if (d2h_sync(s, &ni, P<u32>(s->counters) + 12, 8))
        return -3;
    if (ensure(s->gen_buf, total + 64))
        return -3;
    a.len = P<u64>(s->gen_off);
    a.buf = P<u8>(s->gen_buf);
    k_gen<<<(u32)((count + 127) / 128), 128, 0, s->stream>>>(a, 1);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s->stream));
    *d_buf = s->gen_buf.p;
    *len = total;
    *d_offsets = P<u64>(s->gen_off);
    if (instructions)
        *instructions = ni;
    return 0;
}

// Streams a generated corpus through the pipeline: kernels [k0, k0+count)
// of (shape, stress, seed) are sized on the device, cut into chunks of at
// most chunk_bytes at kernel boundaries, and each chunk is generated into
// the session's text buffer and decompiled before the next is generated, so
// no whole-corpus buffer exists (C5: ~320 GB of listing for 1M kernels).
// Each chunk's output replaces the previous one in the session's output
// buffer.  Every sample_stride-th kernel (k % sample_stride == 0, 0 = none)
// gets the FNV-1a hash and length of its source in sample_hash/sample_len
// (indexed k / sample_stride), for comparison with the reference.
int ocldec_b200_session_run_generated(ocldec_b200_session *s, int shape, int stress, uint64_t seed,
                                      uint64_t k0, uint64_t count, uint64_t chunk_bytes, int fold_local_size,
                                      uint64_t sample_stride, uint64_t *sample_hash, uint64_t *sample_len,
                                      ocldec_b200_stream_stats *out) {
    if (!s || !out) {
        g_err = "bad arguments";
        return -1;
    }
    CK(cudaSetDevice(s->device));
    *out = ocldec_b200_stream_stats{};
    reset_stats(s);
    s->only_set = false;
    set_overrides(s, nullptr, 0);
    if (!chunk_bytes)
        chunk_bytes = chunk_target();
    chunk_bytes = std::min<u64>(chunk_bytes, 0xe0000000ull);
    cudaStream_t st = s->stream;
    cudaEvent_t e0, e1, g0e, g1e;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&g0e));
    CK(cudaEventCreate(&g1e));
    CK(cudaEventRecord(e0, st));
    // sizing pass over the whole range: per-kernel bytes and instructions
    if (ensure(s->gen_len, (count + 1) * 8) || ensure(s->gen_ninstr, (count + 1) * 4) ||
        ensure(s->gen_off, (count + 1) * 8) || ensure(s->counters, 64))
        return -3;
    GenArgs a;
    a.cfg = GenCfg{(u32)shape, (u32)stress, seed};
    a.k0 = k0;
    a.count = count;
    a.len = P<u64>(s->gen_len);
    a.ninstr = P<u32>(s->gen_ninstr);
    a.buf = nullptr;
    a.base = 0;
    CK(cudaMemsetAsync(a.len + count, 0, 8, st));
    k_gen<<<(u32)((count + 127) / 128), 128, 0, st>>>(a, 0);
    CK(cudaGetLastError());
    if (scan_exclusive(s, count + 1, U64Val{0}, AddU64{}, U64Load{a.len}, U64Store{P<u64>(s->gen_off)},
                       reinterpret_cast<U64Val *>(P<u32>(s->counters) + 8)))
        return -3;
    std::vector<u64> offs(count + 1);
    if (d2h_sync(s, offs.data(), s->gen_off.p, (count + 1) * 8))
        return -3;
    float ms = 0;
    {
        cudaEvent_t t;
        CK(cudaEventCreate(&t));
        CK(cudaEventRecord(t, st));
        CK(cudaEventSynchronize(t));
        CK(cudaEventElapsedTime(&ms, e0, t));
        cudaEventDestroy(t);
    }
    out->ms_generate += ms;
    // chunks: as few as fit under chunk_bytes, about equal
    const u64 total = offs[count];
    const u64 nch = std::max<u64>(1, (total + chunk_bytes - 1) / chunk_bytes);
    const u64 tgt = (total + nch - 1) / nch;
    std::vector<u64> kb{0};
    for (u64 k = 0; k < count;) {
        u64 e = std::upper_bound(offs.begin() + k + 1, offs.begin() + count + 1, offs[kb.back()] + tgt) -
                offs.begin() - 1;
        if (e <= k)
            e = k + 1;
        kb.push_back(e);
        k = e;
    }
    u64 maxn = 0;
    for (size_t c = 0; c + 1 < kb.size(); ++c)
        maxn = std::max<u64>(maxn, offs[kb[c + 1]] - offs[kb[c]]);
    if (maxn >= 0xf0000000ull) {
        g_err = "a single generated kernel exceeds the chunk size limit";
        return -1;
    }
    // Chunks are generated G at a time (one k_gen launch over G chunks'
    // kernels: the generator is one thread per kernel, so a lone chunk keeps
    // only a few warps per SM busy), then decompiled one after the other
    // from the group buffer.
    size_t G = 8;
    if (const char *e = getenv("OCLDEC_B200_GEN_GROUP"))
        G = std::max<size_t>(1, strtoull(e, nullptr, 0));
    const size_t nchunks = kb.size() - 1;
    u32 line_base = 0;
    size_t g0 = 0, g1 = 0;
    for (size_t c = 0; c < nchunks; ++c) {
        const u64 ka = kb[c], kz = kb[c + 1], n = offs[kz] - offs[ka];
        if (c == g1) { // generate the next group
            g0 = c;
            g1 = std::min(nchunks, c + G);
            const u64 gb = offs[kb[g1]] - offs[kb[g0]];
            if (ensure(s->sgen, gb + 64))
                return -3;
            GenArgs g = a;
            g.k0 = k0 + kb[g0];
            g.count = kb[g1] - kb[g0];
            g.len = P<u64>(s->gen_off) + kb[g0];
            g.buf = P<u8>(s->sgen);
            g.base = offs[kb[g0]];
            CK(cudaEventRecord(g0e, st));
            k_gen<<<(u32)((g.count + 127) / 128), 128, 0, st>>>(g, 1);
            CK(cudaGetLastError());
            CK(cudaEventRecord(g1e, st));
            CK(cudaEventSynchronize(g1e));
            CK(cudaEventElapsedTime(&ms, g0e, g1e));
            out->ms_generate += ms;
        }
        const size_t before = s->host_res.size();
        ChunkOut co;
        s->chunk_base = 0;
        int rc = run_chunk(s, P<u8>(s->sgen) + (offs[ka] - offs[kb[g0]]), n, false, line_base, fold_local_size,
                           0, false, &co);
        if (rc)
            return rc;
        if (co.err_line != 0xffffffffu) {
            g_err = "split_kernels error in a generated chunk";
            return -4;
        }
        // sampled kernels: source hash (FNV-1a, as the oracle's batch driver)
        for (size_t q = before; sample_stride && q < s->host_res.size(); ++q) {
            const u64 k = ka + (q - before);
            if ((k0 + k) % sample_stride)
                continue;
            const KRes &r = s->host_res[q];
            std::string src(r.status == KS_OK ? r.out_len : 0, '\0');
            if (!src.empty())
                CK(cudaMemcpy(&src[0], P<u8>(s->out) + s->host_kernel_off[q], src.size(), cudaMemcpyDeviceToHost));
            u64 h = 1469598103934665603ull;
            for (unsigned char ch : src) {
                h ^= ch;
                h *= 1099511628211ull;
            }
            const u64 si = (k0 + k) / sample_stride - (k0 + sample_stride - 1) / sample_stride;
            if (sample_hash)
                sample_hash[si] = h;
            if (sample_len)
                sample_len[si] = src.size();
        }
        line_base += co.nlines;
        s->stats.lines += co.nlines;
        s->stats.kernels += co.nk;
        out->in_bytes += n;
        out->out_bytes += co.out_bytes;
        out->chunks++;
        // per-kernel host records are not kept across chunks
        s->host_res.clear();
        s->host_kernel_off.clear();
        s->host_name_line.clear();
        s->host_name_off.clear();
        s->host_diag.clear();
        s->host_kdiag.clear();
        s->host_dumps.clear();
    }
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    out->ms_wall = ms;
    out->ms_decompile = s->stats.ms_parse + s->stats.ms_decompile + s->stats.ms_emit;
    out->kernels = s->stats.kernels;
    out->instructions = s->stats.instructions;
    out->failed = s->stats.failed;
    out->goto_form = s->stats.goto_form;
    out->fallbacks = s->stats.fallbacks;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(g0e);
    cudaEventDestroy(g1e);
    return finish_deferred(s);
}

} // extern "C"
