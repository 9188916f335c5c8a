// ocldec-b200: k_lower, one translation unit compiled with
// -Xptxas -O1: these launches are bound by instruction fetch, and ptxas -O1
// emits smaller code for them (measured: lower -5 %, emit -12 %).
#include "od_device.cuh"

namespace od {

// Kernels with many if-joins (C5's long kernels) are lowered by the whole
// warp redundantly (od_base.cuh "warp cooperation"), so their joins
// (merge_join, collect_delta) split the slot work across the lanes: k_lower_
// wide, one kernel per warp.  k_lower keeps the lone-lane lowering of every
// other kernel.  The host enables the split only for chunks of long kernels
// (measured on C4, whose kernels are short: the second launch and the
// warp-wide entry cost 3-8 % of k_lower and gain nothing).
__global__ void __launch_bounds__(OD_BLOCK, OD_MINB_LOWER * 128 / OD_BLOCK) k_lower(DecompArgs a) {
    Slot0 sl;
    if (!dk_slot(a, &sl))
        return;
    KState *g = reinterpret_cast<KState *>(sl.base);
    if (g->done || g->K.nif >= a.wide_joins)
        return;
#if OD_LOCAL_LOWER
    KState S;
    kstate_load(S, g);
    dk_lower(S);
    kstate_store(g, S);
#else
    kstate_fix(*g); // the previous phase ran on a local copy: re-point into HBM
    dk_lower(*g);
#endif
}

__global__ void __launch_bounds__(OD_BLOCK, OD_MINB_LOWER * 128 / OD_BLOCK) k_lower_wide(DecompArgs a) {
    const u32 full = 0xffffffffu;
    Slot0 sl{0, 0, nullptr};
    const bool mine = dk_slot(a, &sl);
    if (!__shfl_sync(full, mine, 0))
        return;
    KState *g = reinterpret_cast<KState *>(__shfl_sync(full, (unsigned long long)sl.base, 0));
    if (g->done || g->K.nif < a.wide_joins)
        return;
    kstate_fix(*g);
    dk_lower(*g);
}


} // namespace od
