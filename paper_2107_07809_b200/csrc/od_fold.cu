// ocldec-b200: k_fold (fold_expr over each kernel's statements) in its own
// translation unit, so its ptxas level is chosen apart from k_lower / k_emit
// (Makefile PTXAS_od_fold).
#include "od_device.cuh"

namespace od {

__global__ void __launch_bounds__(OD_BLOCK, OD_MINB_FOLD * 128 / OD_BLOCK) k_fold(DecompArgs a) {
    Slot0 sl;
    if (!dk_slot(a, &sl))
        return;
    KState *g = reinterpret_cast<KState *>(sl.base);
    if (g->done)
        return;
#if OD_LOCAL_FOLD
    KState S;
    kstate_load(S, g);
    dk_fold(S);
    kstate_store(g, S);
#else
    kstate_fix(*g);
    dk_fold(*g);
#endif
}

} // namespace od
