// ocldec-b200: device-wide scans (warp shuffle + shared-memory block scan,
// three-phase reduce/scan/apply) used by the line, section, decode and
// emit passes.
#pragma once

#include <cuda_runtime.h>

#include "od_base.cuh"

namespace od {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16; // elements per thread per block tile

// Inclusive warp scan.
template <class T, class Op> __device__ __forceinline__ T warp_inclusive(T v, Op op) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o = v;
        o = T::shfl_up(v, d);
        if (lane >= d)
            v = op(o, v);
    }
    return v;
}

// Exclusive block scan over blockDim.x == kScanThreads threads; *agg gets
// the block total.  smem must hold 32 T.
template <class T, class Op>
__device__ __forceinline__ T block_exclusive(T v, T ident, Op op, T *smem, T *agg) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    T inc = warp_inclusive(v, op);
    if (lane == 31)
        smem[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T w = lane < (kScanThreads >> 5) ? smem[lane] : ident;
        T wi = warp_inclusive(w, op);
        smem[lane] = wi;
    }
    __syncthreads();
    T warp_prefix = wid ? smem[wid - 1] : ident;
    T total = smem[(kScanThreads >> 5) - 1];
    T excl_in_warp = T::shfl_up(inc, 1);
    if (lane == 0)
        excl_in_warp = ident;
    __syncthreads();
    *agg = total;
    return op(warp_prefix, excl_in_warp);
}

// Scalar wrappers with shfl support.
struct SU32 {
    u32 v;
    __device__ static SU32 shfl_up(SU32 x, int d) { return SU32{__shfl_up_sync(0xffffffffu, x.v, d)}; }
};
struct AddU32 {
    __device__ SU32 operator()(SU32 a, SU32 b) const { return SU32{a.v + b.v}; }
};

// Section scan element: kernels seen, last directive line.
struct SecVal {
    u32 cnt;
    i32 last;
    __device__ static SecVal shfl_up(SecVal x, int d) {
        return SecVal{__shfl_up_sync(0xffffffffu, x.cnt, d), __shfl_up_sync(0xffffffffu, x.last, d)};
    }
};
struct SecOp {
    __device__ SecVal operator()(SecVal a, SecVal b) const {
        return SecVal{a.cnt + b.cnt, a.last > b.last ? a.last : b.last};
    }
};

// ---- generic 3-phase exclusive scan over n elements produced by Load(i)
// and consumed by Store(i, exclusive_prefix).
template <class T, class Op, class Load>
__global__ void k_scan_reduce(u64 n, T ident, Op op, Load load, T *block_agg) {
    __shared__ T sm[32];
    const u64 base = (u64)blockIdx.x * kScanThreads * kScanItems;
    T acc = ident;
    for (int j = 0; j < kScanItems; ++j) {
        u64 i = base + (u64)j * kScanThreads + threadIdx.x;
        if (i < n)
            acc = op(acc, load(i));
    }
    T agg;
    block_exclusive(acc, ident, op, sm, &agg);
    if (threadIdx.x == 0)
        block_agg[blockIdx.x] = agg;
}

template <class T, class Op>
__global__ void k_scan_blocks(u64 nb, T ident, Op op, T *block_agg, T *total) {
    __shared__ T sm[32];
    T carry = ident;
    for (u64 b0 = 0; b0 < nb; b0 += kScanThreads) {
        u64 i = b0 + threadIdx.x;
        T v = i < nb ? block_agg[i] : ident;
        T agg;
        T ex = block_exclusive(v, ident, op, sm, &agg);
        if (i < nb)
            block_agg[i] = op(carry, ex);
        carry = op(carry, agg);
        __syncthreads();
    }
    if (threadIdx.x == 0)
        *total = carry;
}

// Apply: each block rescans its tile in order (items are consecutive per
// thread so the per-thread sequential pass preserves order).
template <class T, class Op, class Load, class Store>
__global__ void k_scan_apply(u64 n, T ident, Op op, Load load, Store store, const T *block_agg) {
    __shared__ T sm[32];
    const u64 base = (u64)blockIdx.x * kScanThreads * kScanItems;
    const u64 mine = base + (u64)threadIdx.x * kScanItems;
    T acc = ident;
    for (int j = 0; j < kScanItems; ++j) {
        u64 i = mine + j;
        if (i < n)
            acc = op(acc, load(i));
    }
    T agg;
    T ex = block_exclusive(acc, ident, op, sm, &agg);
    T run = op(block_agg[blockIdx.x], ex);
    for (int j = 0; j < kScanItems; ++j) {
        u64 i = mine + j;
        if (i < n) {
            T v = load(i);
            store(i, run, v);
            run = op(run, v);
        }
    }
}

// The reduce phase must use the same element->thread mapping as apply for
// the block totals to be identical; both reduce over the whole tile, and a
// tile total does not depend on the mapping.
} // namespace od
