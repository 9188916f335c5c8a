// TEST INFRASTRUCTURE ONLY — input synthesis for the oracle side.
//
// Host build of the counter-based synthetic corpus generator
// (paper_2107_07809_b200/csrc/od_gen.cuh) linked into
// oracle/_ref/libocldec_ref.so, so that the CPU arms of bench.py (the
// `cpu_baseline` leg and `--impl reference`) and the parity tests can build
// their inputs without loading the product library.  Kernel k is a pure
// function of (shape, stress, seed, k): these bytes are identical to
// ocldec_b200_gen_host / ocldec_b200_gen_device (checked by
// tests/test_oracle_golden.py::test_oracle_generator_matches_product).
#include <cstdint>
#include <thread>
#include <vector>

#include "../paper_2107_07809_b200/csrc/od_gen.cuh"

using namespace od;

extern "C" {

// Writes kernels [k0, k0 + count) into buf (capacity cap); offsets gets
// count + 1 byte offsets.  buf == nullptr: sizes only.  Returns the bytes
// written (or needed), -2 when cap is too small.  nthreads > 1 splits the
// kernel range over host threads (both passes).
int64_t ref_gen_host(int shape, int stress, uint64_t seed, uint64_t k0, uint64_t count, char *buf,
                     uint64_t cap, uint64_t *offsets, uint64_t *instructions, int nthreads) {
    GenCfg g{(u32)shape, (u32)stress, seed};
    if (nthreads < 1)
        nthreads = 1;
    if ((uint64_t)nthreads > count)
        nthreads = count ? (int)count : 1;
    std::vector<uint64_t> len(count), ni(count);
    auto sizes = [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i) {
            Writer w{nullptr, 0, 0, false};
            ni[i] = gen_kernel(g, k0 + i, &w);
            len[i] = w.n;
        }
    };
    auto fill = [&](uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i) {
            Writer w{reinterpret_cast<u8 *>(buf) + offsets[i], 0, 0xffffffffu, false};
            gen_kernel(g, k0 + i, &w);
        }
    };
    auto par = [&](auto fn) {
        std::vector<std::thread> th;
        for (int t = 0; t < nthreads; ++t)
            th.emplace_back([&, t] { fn(count * t / nthreads, count * (t + 1) / nthreads); });
        for (auto &x : th)
            x.join();
    };
    par(sizes);
    uint64_t total = 0, nins = 0;
    for (uint64_t i = 0; i < count; ++i) {
        if (offsets)
            offsets[i] = total;
        total += len[i];
        nins += ni[i];
    }
    if (offsets)
        offsets[count] = total;
    if (instructions)
        *instructions = nins;
    if (!buf)
        return (int64_t)total;
    if (total > cap || !offsets)
        return -2;
    par(fill);
    return (int64_t)total;
}

} // extern "C"
