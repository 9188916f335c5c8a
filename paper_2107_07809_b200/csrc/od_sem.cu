// ocldec-b200: k_semcheck, the batched semantic check (od_oracle.cuh,
// SURVEY §8(f) rank 4), in its own translation unit so that the phase
// kernels' code layout (od_phases.cu, instruction-fetch bound) does not move
// with the interpreter's.
#include <cstdio>
#include "od_device.cuh"
#include "od_oracle.cuh"

namespace od {

// The batched semantic check (od_oracle.cuh) of wave slot i: environment
// `lane` on lanes 0..kSemEnvs-1 of the calling warp, in the warp's scratch.
// With a step budget, a kernel whose environments are still running after
// `budget` steps (typically a loop that will run the 2^20-step fuel out) is
// listed as deferred instead of holding the wave: the host re-checks the
// deferred kernels of the whole run together at its end.
__device__ __noinline__ void sem_one(const DecompArgs &a, const SemArgs &sa, u32 i, u32 lane, u8 *wscratch) {
    const u32 k = a.order[i];
    const u32 lanes = kSemEnvs;
    const u32 m = (1u << lanes) - 1;
    SemResult *out = sa.out;
    u64 *counts = sa.counts;
    if (a.res[k].status != KS_OK) {
        if (lane == 0) {
            out[k] = SemResult{SEM_NOT_RUN, 0, 0, 0};
            // arena / pool retries re-run the kernel (and this check): counted then
            if (a.res[k].status != KS_OOM && a.res[k].status != KS_STAGE_FULL)
                atomicAdd(reinterpret_cast<unsigned long long *>(counts + SEM_NOT_RUN), 1ull);
        }
        return;
    }
    const u64 ord = sa.kmap ? sa.kmap[sa.kbase + k] : sa.kbase + k;
    // The kernel's state is read in place (one L1-cached copy per warp, not a
    // 2.5 KB local copy per lane): its four self-pointers are fixed once.
    KState *g = reinterpret_cast<KState *>(a.arena + (a.boff[i] - a.boff0));
    if (lane == 0)
        kstate_fix(*g);
    __syncwarp(m);
    const KState &S = *g;
    SemCtx c;
    c.K = &S.K;
    c.unsupported = false;
    c.nan_choice = false;
    SemRng r = sem_stream(sa.seed, ord, lane);
    sem_env(r, lane, S.K.cfg.dims, S.K.cfg.cws, &c.env);
    sem_args(c, r);
    u8 *base = wscratch + (u64)lane * kSemLaneBytes;
    SemMem ma, mb;
    ma.init(base, c.env.mem_seed);
    mb.init(base, c.env.mem_seed);
    u64 *vk = reinterpret_cast<u64 *>(base), *vv = vk + kSemVarCap;
    for (u32 q = 0; q < kSemVarCap; ++q)
        vk[q] = 0;
    base += kSemVarCap * 16;
    SemMachine mach{c, ma};
    mach.wm = m;
    mach.init();
    if (sa.budget != 0) {
        // a straight pass over a long kernel is not a loop: at least 8 steps per
        // instruction (a negative budget is an exact limit, for tests)
        mach.run(sa.budget > 0 ? max((long)sa.budget, 8l * (long)S.K.nins) : -sa.budget);
        if (__ballot_sync(m, mach.held)) {
            // the deferred sections travel to the host: at most kSemDeferKB of listing per chunk
            const u32 kb = (u32)(((u64)S.K.nins * 64 + 1023) >> 10);
            u32 slot = ~0u;
            if (lane == 0 && atomicAdd(sa.dlist + 1, kb) + kb <= sa.dkb)
                slot = atomicAdd(sa.dlist, 1u);
            slot = __shfl_sync(m, slot, 0);
            if (slot < sa.dcap) {
                if (lane == 0) {
                    sa.dlist[2 + slot] = k;
                    out[k] = SemResult{SEM_DEFERRED, 0, 0, 0};
                }
                return;
            }
            // the deferral list or its byte budget is full: finish here
        }
    }
    mach.run();
    SemEval ev{c, mb, SemVars{vk, vv, false}, reinterpret_cast<u64 *>(base), false, false};
    ev.run(S.hoist, S.body);
#ifdef OD_SEM_DEBUG
    if (ord == OD_SEM_DEBUG) {
        printf("S %u %u asm bad=%d n=%u [", (u32)ord, lane, (int)mach.bad, ma.count);
        for (u32 q = 0; q < ma.n; ++q)
            printf(" %llx:%x", (unsigned long long)ma.addr[q], ma.val[q]);
        printf(" ] body bad=%d full=%d n=%u [", (int)ev.bad, (int)ev.full, mb.count);
        for (u32 q = 0; q < mb.n; ++q)
            printf(" %llx:%x", (unsigned long long)mb.addr[q], mb.val[q]);
        printf(" ]\n");
    }
#endif
    const bool bad = mach.bad || ev.bad;
    const bool full = ma.full || mb.full || ev.full || ev.vars.full;
    const bool same = ma.hash == mb.hash && ma.count == mb.count;
    const u32 any_bad = __ballot_sync(m, bad), any_full = __ballot_sync(m, full), any_diff = __ballot_sync(m, !same);
    const u32 any_nan = __ballot_sync(m, c.nan_choice);
    u64 ha = sem_env_mix(ma.hash, ma.count, lane), hb = sem_env_mix(mb.hash, mb.count, lane);
    for (u32 d = lanes / 2; d; d >>= 1) {
        ha += __shfl_down_sync(m, ha, d);
        hb += __shfl_down_sync(m, hb, d);
    }
    if (lane == 0) {
        const u32 st = any_bad    ? SEM_UNSUPPORTED
                       : any_full ? SEM_CAPACITY
                       : any_nan  ? SEM_INDETERMINATE
                       : any_diff ? SEM_MISMATCH
                                  : SEM_EQUAL;
        out[k] = SemResult{st, lanes, ha, hb};
        atomicAdd(reinterpret_cast<unsigned long long *>(counts + st), 1ull);
    }
}

// Persistent over the wave: each warp takes the next unchecked slot from
// the wave's counter, so a kernel that runs long overlaps the rest of the
// wave instead of holding a whole batch launch.  Warps <= kSemBatch (the
// scratch's slots).
__global__ void __launch_bounds__(128) k_semcheck(DecompArgs a, SemArgs sa) {
    const u32 wl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (lane >= kSemEnvs)
        return;
    u8 *ws = sa.scratch + (u64)wl * kSemEnvs * kSemLaneBytes;
    for (;;) {
        u32 i = 0;
        if (lane == 0)
            i = atomicAdd(sa.next, 1u);
        i = __shfl_sync((1u << kSemEnvs) - 1, i, 0);
        if (i >= sa.n)
            return;
        sem_one(a, sa, i, lane, ws);
    }
}

// Byte spans of the listed kernels in the chunk text (their .kernel line to
// the next kernel's, or the chunk end): the deferred kernels' sections.
__global__ void k_def_spans(const u32 *dlist, u32 n, const u32 *nlpos, u32 nlf, const u32 *kstart, u32 nk,
                            u64 len, u64 *span) {
    const u32 j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n)
        return;
    const u32 k = dlist[2 + j];
    auto line_start = [&](u32 l) -> u64 { return l == 0 ? 0 : l - 1 < nlf ? (u64)nlpos[l - 1] + 1 : len; };
    const u64 b = line_start(kstart[k]);
    const u64 e = k + 1 < nk ? line_start(kstart[k + 1]) : len;
    span[2 * j] = b;
    span[2 * j + 1] = e > b ? e - b : 0;
}

// Packs the spans' bytes at their offsets in dst (warp per span).
__global__ void k_def_pack(const u8 *t, const u64 *span, const u64 *dst_off, u32 n, u8 *dst) {
    const u32 w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n)
        return;
    const u64 b = span[2 * w], l = span[2 * w + 1], o = dst_off[w];
    for (u64 q = lane; q < l; q += 32)
        dst[o + q] = t[b + q];
}

} // namespace od
