// ocldec-b200: declarations shared by the translation units of the device
// library (ocldec_b200.cu: host + parse kernels; od_front.cu: k_front;
// od_phases.cu: k_lower/k_fold/k_emit; od_genk.cu: the corpus generator).
// Separate units let each phase get its own ptxas options (Makefile).
#pragma once

#include <cuda_runtime.h>

#include "od_gen.cuh"
#include "od_kernel.cuh"

namespace od {

// ------------------------------------------------------------------ P2-P4a (decompile phases)
struct KRes {
    u32 status;     // KStatus, KS_SKIP = 4 for only_kernel filtering, 5 = staging full
    u32 structured;
    u32 fallbacks;
    u32 ninstr;
    u64 stage_off;
    u32 out_len;
    u32 name_off;   // kernel name span (chunk-relative; >= chunk len: aux area)
    u32 name_len;
    u32 ndiag;      // diagnostics of the kernel, at diag_off in the diagnostic pool
    u64 diag_off;
};


struct DecompArgs {
    const u8 *t;
    const LineRec *lines;
    const LineIns *lins;
    const Opnd *ops;
    const Label *labs;
    const u32 *kstart;
    u32 nk, nlines, line_base, fold_local_size;
    const u32 *order;   // kernels of this wave (size-sorted)
    const u64 *boff;    // arena offsets (exclusive scan of budgets, per order slot)
    u64 boff0;          // boff of the first slot of the wave
    u32 count;          // kernels in the wave
    u32 scale;
    u8 *arena;
    u8 *stage;
    u64 stage_cap;
    unsigned long long *stage_top;
    KRes *res;
    const u8 *only;  // only_kernel name (device) or null
    u32 only_len;
    u64 *prof;
    u32 lanes_per; // lanes per kernel: 32 / kernels-per-warp
    const u32 *perm; // wave slot permutation for the launches after k_front (null: identity)
    const AbiOvr *ovr; // ABI overrides of the run (novr)
    u32 novr;
    const u8 *ovr_text;
    const DumpCfg *dump; // DOT dumps (null: none)
    Diag *dpool;   // diagnostic records of finished kernels
    u64 dcap;
    unsigned long long *dtop;
    const KSize *sizes; // per kernel (k_ksize)
    u32 *retry_cnt;     // kernels that ended out of arena or staging room (k_emit counts them)
    u32 wide_joins;     // if-joins from which k_lower_wide lowers a kernel (~0u: k_lower takes all)
};

// Three launches per wave, one per pipeline phase (od_lower.cuh dk_front /
// dk_lower / dk_emit): every warp on an SM runs the same phase's code.  kpw
// kernels per warp (lane 0 of each 32/kpw-lane group works), kernels
// size-sorted (largest first) so the block scheduler starts big kernels
// first; each kernel gets an exact arena slice sized by kernel_budget(lines),
// whose base holds its KState between the launches.
struct Slot0 {
    u32 k;
    u32 i;     // wave slot
    u8 *base;
};
__device__ __forceinline__ bool dk_slot(const DecompArgs &a, Slot0 *o) {
    const u32 g = blockIdx.x * blockDim.x + threadIdx.x;
    if ((threadIdx.x & 31) % a.lanes_per)
        return false;
    u32 i = g / a.lanes_per;
    if (i >= a.count)
        return false;
    if (a.perm) // lower / fold / emit: slots grouped by the class k_front found
        i = a.perm[i];
    o->i = i;
    o->k = a.order[i];
    o->base = a.arena + (a.boff[i] - a.boff0);
    return true;
}

// 1: a phase kernel runs on a local-memory copy of the KState; 0: in place in
// HBM (measured per phase: lowering is faster in place, the others on the copy;
// local memory interleaves words across the 32 lanes, so a lone active lane
// spreads its state over 32x the L1 lines).
#ifndef OD_LOCAL_STATE
#define OD_LOCAL_STATE 1
#endif
#ifndef OD_LOCAL_LOWER
#define OD_LOCAL_LOWER 0
#endif
#ifndef OD_LOCAL_FOLD
#define OD_LOCAL_FOLD OD_LOCAL_STATE
#endif

// Threads per block of the phase kernels (one kernel per warp).
#ifndef OD_BLOCK
#define OD_BLOCK 128
#endif

// Minimum resident blocks per SM for the phase kernels (register caps), in
// 128-thread blocks.
#ifndef OD_MINB_FRONT
#define OD_MINB_FRONT 16
#endif
#ifndef OD_MINB_LOWER
#define OD_MINB_LOWER 16
#endif
#ifndef OD_MINB_FOLD
#define OD_MINB_FOLD 10
#endif
#ifndef OD_MINB_EMIT
#define OD_MINB_EMIT 16
#endif

// The phase kernels run on a local (stack) copy of the KState: its hot
// counters (arena tops, writer position, stack tops) then live in L1
// write-back local memory instead of write-through global memory.  Copies
// are word loops (an aggregate copy here was miscompiled by nvcc 12.9).
__device__ __forceinline__ void kstate_load(KState &S, const KState *g) {
    static_assert(sizeof(KState) % 8 == 0, "KState is copied in u64 words");
    const u64 *src = reinterpret_cast<const u64 *>(g);
    u64 *dst = reinterpret_cast<u64 *>(&S);
    for (u32 q = 0; q < sizeof(KState) / 8; ++q)
        dst[q] = src[q];
    kstate_fix(S);
}
__device__ __forceinline__ void kstate_store(KState *g, const KState &S) {
    const u64 *src = reinterpret_cast<const u64 *>(&S);
    u64 *dst = reinterpret_cast<u64 *>(g);
    for (u32 q = 0; q < sizeof(KState) / 8; ++q)
        dst[q] = src[q];
}


__global__ void __launch_bounds__(OD_BLOCK, OD_MINB_FRONT * 128 / OD_BLOCK) k_front(DecompArgs a);
__global__ void __launch_bounds__(OD_BLOCK, OD_MINB_LOWER * 128 / OD_BLOCK) k_lower(DecompArgs a);
__global__ void __launch_bounds__(OD_BLOCK, OD_MINB_LOWER * 128 / OD_BLOCK) k_lower_wide(DecompArgs a);
constexpr u32 kWideJoins = 64; // if-joins from which a kernel is lowered by the whole warp (long-kernel chunks)
__global__ void __launch_bounds__(OD_BLOCK, OD_MINB_FOLD * 128 / OD_BLOCK) k_fold(DecompArgs a);
__global__ void __launch_bounds__(OD_BLOCK, OD_MINB_EMIT * 128 / OD_BLOCK) k_emit(DecompArgs a);
__global__ void __launch_bounds__(OD_BLOCK) k_export(DecompArgs a);
struct SemResult;
struct SemArgs;
__global__ void __launch_bounds__(128) k_semcheck(DecompArgs a, SemArgs sa);
__global__ void k_def_spans(const u32 *dlist, u32 n, const u32 *nlpos, u32 nlf, const u32 *kstart, u32 nk,
                            u64 len, u64 *span);
__global__ void k_def_pack(const u8 *t, const u64 *span, const u64 *dst_off, u32 n, u8 *dst);

// ------------------------------------------------------------------ generator
struct GenArgs {
    GenCfg cfg;
    u64 k0, count;
    u64 *len;   // per kernel length (sizing) -> offsets after scan
    u32 *ninstr;
    u8 *buf;
    u64 base;   // write pass: kernel i goes to buf + len[i] - base
};

__global__ void k_gen(GenArgs a, int mode);


} // namespace od
