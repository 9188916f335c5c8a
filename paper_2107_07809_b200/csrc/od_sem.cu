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
__device__ __noinline__ void sem_one(const DecompArgs &a, u32 i, u32 lane, u8 *wscratch, SemResult *out, u64 seed,
                                     u64 kbase, u64 *counts) {
    const u32 k = a.order[i];
    const u32 lanes = kSemEnvs;
    const u32 m = (1u << lanes) - 1;
    if (a.res[k].status != KS_OK) {
        if (lane == 0) {
            out[k] = SemResult{SEM_NOT_RUN, 0, 0, 0};
            // arena / pool retries re-run the kernel (and this check): counted then
            if (a.res[k].status != KS_OOM && a.res[k].status != KS_STAGE_FULL)
                atomicAdd(reinterpret_cast<unsigned long long *>(counts + SEM_NOT_RUN), 1ull);
        }
        return;
    }
    KState S;
    kstate_load(S, reinterpret_cast<const KState *>(a.arena + (a.boff[i] - a.boff0)));
    SemCtx c;
    c.K = &S.K;
    c.unsupported = false;
    c.nan_choice = false;
    SemRng r = sem_stream(seed, kbase + k, lane);
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
    mach.run();
    SemEval ev{c, mb, SemVars{vk, vv, false}, reinterpret_cast<u64 *>(base), false, false};
    ev.run(S.hoist, S.body);
#ifdef OD_SEM_DEBUG
    if (kbase + k == OD_SEM_DEBUG) {
        printf("S %u %u asm bad=%d n=%u [", (u32)(kbase + k), lane, (int)mach.bad, ma.count);
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
// the wave's counter, so a kernel that runs its environments to the fuel
// limit (2^20 interpreted steps) overlaps the rest of the wave instead of
// holding a whole batch launch.  Warps <= kSemBatch (the scratch's slots).
__global__ void __launch_bounds__(128) k_semcheck(DecompArgs a, u32 n, u32 *next, u8 *scratch, SemResult *out,
                                                  u64 seed, u64 kbase, u64 *counts) {
    const u32 wl = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (lane >= kSemEnvs)
        return;
    u8 *ws = scratch + (u64)wl * kSemEnvs * kSemLaneBytes;
    for (;;) {
        u32 i = 0;
        if (lane == 0)
            i = atomicAdd(next, 1u);
        i = __shfl_sync((1u << kSemEnvs) - 1, i, 0);
        if (i >= n)
            return;
        sem_one(a, i, lane, ws, out, seed, kbase, counts);
    }
}

} // namespace od
