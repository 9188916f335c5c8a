// ocldec-b200: k_emit (render + the warp's copy into the stage) and k_export
// in their own translation unit, compiled with -Xptxas -O1 like k_lower's:
// a module per phase keeps each phase's code apart from the others'
// (k_fold moved out the same way: k_lower 1819 -> 1791 ms, k_fold 377 ->
// 363 ms per C4 step).
#include "od_device.cuh"

namespace od {

// DUMP_BODY: the lowered statement tree of every kernel that emitted, as a
// step -3 dump (a separate launch: the emit path pays nothing for it).
__global__ void __launch_bounds__(OD_BLOCK) k_export(DecompArgs a) {
    Slot0 sl;
    if (!dk_slot(a, &sl))
        return;
    const u32 k = sl.k;
    if (a.res[k].status != KS_OK)
        return;
    KState S;
    kstate_load(S, reinterpret_cast<KState *>(sl.base));
    if (!dk_export(S))
        a.res[k].status = KS_STAGE_FULL; // the host grows the dump pool and re-runs the kernel
    if (a.res[k].status == KS_STAGE_FULL)
        atomicAdd(a.retry_cnt, 1u);
}

__device__ __noinline__ void emit_one(const DecompArgs &a, const Slot0 &sl, const uint4 **cs, uint4 **cd,
                                      u32 *cn);

__global__ void __launch_bounds__(OD_BLOCK, OD_MINB_EMIT * 128 / OD_BLOCK) k_emit(DecompArgs a) {
    Slot0 sl;
    const uint4 *cs = nullptr; // this lane's kernel text in its arena ...
    uint4 *cd = nullptr;       // ... and its place in the stage
    u32 cn = 0;                // 16-byte words
    if (dk_slot(a, &sl))
        emit_one(a, sl, &cs, &cd, &cn);
    // the whole warp copies each lane's text: coalesced 512-byte rows
    // instead of one lane's 16-byte stream
    const u32 lane = threadIdx.x & 31;
    for (u32 src = 0; src < 32; ++src) {
        const uint4 *s4 = reinterpret_cast<const uint4 *>(__shfl_sync(0xffffffffu, (unsigned long long)cs, src));
        uint4 *d4 = reinterpret_cast<uint4 *>(__shfl_sync(0xffffffffu, (unsigned long long)cd, src));
        const u32 n = __shfl_sync(0xffffffffu, cn, src);
        for (u32 q = lane; q < n; q += 32)
            d4[q] = s4[q];
    }
}

__device__ __noinline__ void emit_one(const DecompArgs &a, const Slot0 &sl, const uint4 **cs, uint4 **cd,
                                      u32 *cn) {
    KState *g = reinterpret_cast<KState *>(sl.base);
    KOut o;
    const u8 *src = nullptr;
    const Diag *dg = g->K.dg;
    u32 ndg = g->K.ndg;
    if (!g->done) {
#if OD_LOCAL_STATE
        KState S;
        kstate_load(S, g);
        dk_emit(S);
        o = S.out;
        src = S.w.p;
        ndg = S.K.ndg;
#else
        kstate_fix(*g);
        dk_emit(*g);
        o = g->out;
        src = g->w.p;
        ndg = g->K.ndg;
#endif
    } else {
        o = g->out;
    }
    const u32 k = sl.k;
    KRes r;
    r.ndiag = 0;
    r.diag_off = 0;
    r.stage_off = 0;
    r.out_len = 0;
    r.status = o.status;
    r.structured = o.structured;
    r.fallbacks = o.fallbacks;
    r.ninstr = o.ninstr;
    {
        Span nm, w, rest, extra;
        const LineRec &L = a.lines[a.kstart[k]];
        split_word(a.t, Span{L.off, L.len}, &w, &rest);
        split_word(a.t, rest, &nm, &extra);
        r.name_off = nm.off;
        r.name_len = nm.len;
    }
    if (o.status == KS_OK && o.out_len) {
        u64 padded = (o.out_len + 15ull) & ~15ull;
        u64 so = atomicAdd(a.stage_top, (unsigned long long)padded);
        if (so + padded > a.stage_cap) {
            r.status = KS_STAGE_FULL;
        } else {
            *cs = reinterpret_cast<const uint4 *>(src);
            *cd = reinterpret_cast<uint4 *>(a.stage + so);
            *cn = (u32)(padded / 16);
            r.stage_off = so;
            r.out_len = o.out_len;
        }
    }
    // diagnostics (the OOM attempts are re-run from scratch: not kept)
    if (ndg && o.status != KS_OOM && r.status != KS_STAGE_FULL) {
        const u64 dof = atomicAdd(a.dtop, (unsigned long long)ndg);
        if (dof + ndg > a.dcap) {
            r.status = KS_STAGE_FULL; // the host grows the pool and re-runs the kernel
        } else {
            for (u32 q = 0; q < ndg; ++q)
                a.dpool[dof + q] = dg[q];
            r.ndiag = ndg;
            r.diag_off = dof;
        }
    }
    if (r.status == KS_OOM || r.status == KS_STAGE_FULL)
        atomicAdd(a.retry_cnt, 1u);
    a.res[k] = r;
}

} // namespace od
