// ocldec-b200: k_front (dk_front: config, ABI, CFG, mask normalization,
// region reduction, liveness, pool carving), its own translation unit.
#include "od_device.cuh"

namespace od {

__device__ __noinline__ void front_one(const DecompArgs &a, const Slot0 &sl, u64 **names, u32 *names_cap,
                                       Slot **regs, const Collected &col, bool collected);

// collect_fill (od_kernel.cuh) for one kernel by the whole warp: 32 lines per
// step, label and instruction positions from warp scans, the labels pending
// before each instruction from the previous instruction line's label count.
__device__ __noinline__ Collected warp_collect(const DecompArgs &a, u32 lbeg, u32 lend, Ins *ins, u32 *kl) {
    const u32 lane = threadIdx.x & 31;
    const u32 full = 0xffffffffu;
    const u32 lt = (1u << lane) - 1;
    Collected c{0, 0, 0, a.line_base + lbeg + 1, 0};
    for (u32 l0 = lbeg + 1; l0 < lend; l0 += 32) {
        const u32 l = l0 + lane;
        LineIns L;
        bool has = false;
        u32 nl = 0;
        if (l < lend && a.lines[l].role == LR_TEXT) {
            L = a.lins[l];
            nl = L.nlabels;
            has = (L.flags & IF_HAS_INS) != 0;
        }
        u32 incl = nl;
        for (u32 d = 1; d < 32; d <<= 1) {
            const u32 t = __shfl_up_sync(full, incl, d);
            if (lane >= d)
                incl += t;
        }
        const u32 lab_incl = c.nkl + incl;
        for (u32 k = 0; k < nl; ++k)
            kl[lab_incl - nl + k] = L.lab_start + k;
        const u32 hb = __ballot_sync(full, has);
        const u32 before = hb & lt;
        const u32 pv = __shfl_sync(full, lab_incl, before ? 31 - __clz(before) : lane);
        if (has)
            collect_ins(ins[c.nins + __popc(before)], L, a.ops, a.line_base + l + 1, before ? pv : c.pend_b,
                        lab_incl - (before ? pv : c.pend_b));
        c.any_failed |= __ballot_sync(full, has && (L.flags & IF_PARSE_FAILED)) ? 1u : 0u;
        if (hb) {
            const u32 last = 31 - __clz(hb);
            c.pend_b = __shfl_sync(full, lab_incl, last);
            c.last_line = a.line_base + l0 + last + 1;
        }
        c.nins += __popc(hb);
        c.nkl = __shfl_sync(full, lab_incl, 31);
    }
    return c;
}

// One kernel per warp (lanes_per == 32): the whole warp runs the kernel's
// front redundantly (od_base.cuh "warp cooperation"), so the loops the front
// splits across lanes (liveness, ...) run 32 wide.
__device__ __noinline__ void front_warp(const DecompArgs &a) {
    const u32 full = 0xffffffffu;
    const u32 lane = threadIdx.x & 31;
    Slot0 sl{0, 0, nullptr};
    const bool mine = dk_slot(a, &sl); // lane 0 of the warp, when the wave has a kernel for it
    if (!__shfl_sync(full, mine, 0))
        return;
    sl.k = __shfl_sync(full, sl.k, 0);
    sl.i = __shfl_sync(full, sl.i, 0);
    sl.base = reinterpret_cast<u8 *>(__shfl_sync(full, (unsigned long long)sl.base, 0));
    Collected col{0, 0, 0, 0, 0};
    bool collected = false;
    {
        const u32 kb = (sizeof(KState) + 255) & ~255ull;
        const KSize z = a.sizes[sl.k];
        u64 kl_off;
        const u64 need = collect_bytes(z.nins, z.nlab, &kl_off);
        if (need <= a.boff[sl.i + 1] - a.boff[sl.i] - kb) { // else the front runs out of arena and retries
            const u32 lbeg = a.kstart[sl.k], lend = sl.k + 1 < a.nk ? a.kstart[sl.k + 1] : a.nlines;
            col = warp_collect(a, lbeg, lend, reinterpret_cast<Ins *>(sl.base + kb),
                               reinterpret_cast<u32 *>(sl.base + kb + kl_off));
            collected = true;
        }
    }
    __syncwarp();
    u64 *names = nullptr;
    u32 names_cap = 0;
    Slot *regs = nullptr;
    front_one(a, sl, &names, &names_cap, &regs, col, collected);
    __syncwarp();
    if (regs) {
        Slot d;
        reset_slot(d);
        d.pad[0] = d.pad[1] = d.pad[2] = 0;
        const uint4 dv = *reinterpret_cast<const uint4 *>(&d);
        for (u32 q = lane; q < kPhysSlots; q += 32)
            reinterpret_cast<uint4 *>(regs)[q] = dv;
    }
    if (names)
        for (u32 q = lane; q < names_cap / 2; q += 32)
            reinterpret_cast<uint4 *>(names)[q] = uint4{0, 0, 0, 0};
}

__global__ void __launch_bounds__(OD_BLOCK, OD_MINB_FRONT * 128 / OD_BLOCK) k_front(DecompArgs a) {
    if (a.lanes_per == 32) {
        front_warp(a);
        return;
    }
    Slot0 sl;
    u64 *names = nullptr; // this lane's name set, zeroed below by the whole warp
    u32 names_cap = 0;
    Slot *regs = nullptr; // and its register file (RegisterFile defaults)
    const u32 lane = threadIdx.x & 31;
    const bool mine = dk_slot(a, &sl);
    // the warp collects each of its kernels' instructions first
    Collected col{0, 0, 0, 0, 0};
    bool collected = false;
    const u32 kb = (sizeof(KState) + 255) & ~255ull;
    for (u32 src = 0; src < 32; ++src) {
        const u32 k = __shfl_sync(0xffffffffu, mine ? sl.k : 0xffffffffu, src);
        if (k == 0xffffffffu)
            continue;
        const u32 i = __shfl_sync(0xffffffffu, sl.i, src);
        u8 *base = reinterpret_cast<u8 *>(__shfl_sync(0xffffffffu, (unsigned long long)sl.base, src));
        const KSize z = a.sizes[k];
        u64 kl_off;
        const u64 need = collect_bytes(z.nins, z.nlab, &kl_off);
        if (need > a.boff[i + 1] - a.boff[i] - kb)
            continue; // the lane's own front runs out of arena and retries
        const u32 lbeg = a.kstart[k], lend = k + 1 < a.nk ? a.kstart[k + 1] : a.nlines;
        const Collected c = warp_collect(a, lbeg, lend, reinterpret_cast<Ins *>(base + kb),
                                         reinterpret_cast<u32 *>(base + kb + kl_off));
        if (lane == src) {
            col = c;
            collected = true;
        }
    }
    __syncwarp();
    if (mine)
        front_one(a, sl, &names, &names_cap, &regs, col, collected);
    {
        Slot d;
        reset_slot(d);
        d.pad[0] = d.pad[1] = d.pad[2] = 0;
        static_assert(sizeof(Slot) == 16, "one 16-byte store per slot");
        const uint4 dv = *reinterpret_cast<const uint4 *>(&d);
        for (u32 src = 0; src < 32; ++src) {
            uint4 *p = reinterpret_cast<uint4 *>(__shfl_sync(0xffffffffu, (unsigned long long)regs, src));
            if (p)
                for (u32 q = lane; q < kPhysSlots; q += 32)
                    p[q] = dv;
        }
    }
    // NameSet::keys must start zeroed: 32 lanes store 16 bytes each per
    // iteration instead of the kernel's lone lane walking the table
    for (u32 src = 0; src < 32; ++src) {
        uint4 *p = reinterpret_cast<uint4 *>(__shfl_sync(0xffffffffu, (unsigned long long)names, src));
        const u32 n4 = __shfl_sync(0xffffffffu, names_cap, src) / 2;
        for (u32 q = lane; q < n4; q += 32)
            p[q] = uint4{0, 0, 0, 0};
    }
}

__device__ __noinline__ void front_one(const DecompArgs &a, const Slot0 &sl, u64 **names, u32 *names_cap,
                                       Slot **regs, const Collected &col, bool collected) {
    const u32 k = sl.k;
    const u32 i = sl.i;
    KState *g = reinterpret_cast<KState *>(sl.base);
    const u64 kb = (sizeof(KState) + 255) & ~255ull;
    // Field-wise setup of the state in HBM.  (nvcc 12.9 miscompiled an
    // aggregate copy of a locally built KIn here into a copy of the first
    // bytes of the kernel parameters.)
    static_assert(sizeof(KState) % 8 == 0, "KState is zeroed in u64 words");
    for (u32 q = 0; q < sizeof(KState) / 8; ++q)
        reinterpret_cast<u64 *>(g)[q] = 0;
    KIn &in = g->in;
    in.t = a.t;
    in.lines = a.lines;
    in.lins = a.lins;
    in.ops = a.ops;
    in.labs = a.labs;
    in.lbeg = a.kstart[k];
    in.lend = k + 1 < a.nk ? a.kstart[k + 1] : a.nlines;
    in.line_base = a.line_base;
    in.fold_local_size = a.fold_local_size;
    in.scale = a.scale;
    in.prof = a.prof;
    {
        const KSize z = a.sizes[k];
        in.nblk_cap = a.scale <= 1 ? z.nb : 0;
        in.ncfg = z.ncfg;
        in.nins = z.nins;
        in.nlab = z.nlab;
    }
    in.ovr = a.ovr;
    in.novr = a.novr;
    in.ovr_text = a.ovr_text;
    in.dump = a.dump;
    in.kidx = k;
    in.names_zeroed_by_caller = 1;
    in.collected = collected ? 1 : 0;
    in.c_nins = col.nins;
    in.c_nkl = col.nkl;
    in.c_pend_b = col.pend_b;
    in.c_last_line = col.last_line;
    in.c_any_failed = col.any_failed;
    g->mem.base = sl.base + kb;
    g->mem.top = 0;
    g->mem.cap = a.boff[i + 1] - a.boff[i] - kb;
    g->mem.oom = false;
    g->out.status = KS_OK;
    kstate_fix(*g);
    Span nm;
    {
        Span w, rest, extra;
        const LineRec &L = a.lines[in.lbeg];
        split_word(a.t, Span{L.off, L.len}, &w, &rest);
        split_word(a.t, rest, &nm, &extra);
    }
    if (a.only && (nm.len != a.only_len || !bytes_eq(a.t + nm.off, a.only, nm.len))) {
        g->out.status = KS_SKIP;
        g->done = 1;
    } else {
#ifdef OD_DEBUG_FRONT
        printf("k=%u g=%p K.in=%p &g->in=%p g->in.t=%p g->in.lines=%p lbeg=%u lend=%u mem.base=%p cap=%llu\n",
               k, g, g->K.in, &g->in, g->in.t, g->in.lines, g->in.lbeg, g->in.lend, g->mem.base,
               (unsigned long long)g->mem.cap);
#endif
#if OD_LOCAL_STATE
        KState S;
        kstate_load(S, g);
        dk_front(S);
        kstate_store(g, S);
#else
        kstate_fix(*g);
        dk_front(*g);
#endif
        if (!g->done && g->K.pool.keys) {
            *names = g->K.pool.keys;
            *names_cap = g->K.pool.cap;
            *regs = g->K.regs;
        }
    }
}

} // namespace od
