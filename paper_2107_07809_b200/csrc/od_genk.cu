// ocldec-b200: the counter-based corpus generator kernel (od_gen.cuh) in its
// own translation unit (large code, compiled in parallel with the rest).
#include "od_device.cuh"

namespace od {

__global__ void k_gen(GenArgs a, int mode) {
    u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.count)
        return;
    Writer w;
    if (mode == 0) {
        w.p = nullptr;
        w.n = 0;
        w.cap = 0;
        w.overflow = false;
        u32 ni = gen_kernel(a.cfg, a.k0 + i, &w);
        a.len[i] = w.n;
        a.ninstr[i] = ni;
    } else {
        u64 off = a.len[i] - a.base;
        w.p = a.buf + off;
        w.n = 0;
        w.cap = 0xffffffffu;
        w.overflow = false;
        gen_kernel(a.cfg, a.k0 + i, &w);
    }
}


} // namespace od
