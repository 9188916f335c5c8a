// Developer tool: prints a synthetic corpus (host build of od_gen.cuh).
//   build/devgen SHAPE STRESS SEED K0 COUNT > corpus.s
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2107_07809_b200/csrc/od_gen.cuh"
using namespace od;
int main(int argc, char **argv) {
    GenCfg g{(u32)atoi(argv[1]), (u32)atoi(argv[2]), strtoull(argv[3], 0, 0)};
    u64 k0 = strtoull(argv[4], 0, 0), n = strtoull(argv[5], 0, 0);
    std::vector<u8> buf;
    for (u64 k = k0; k < k0 + n; ++k) {
        Writer cnt{nullptr, 0, 0, false};
        gen_kernel(g, k, &cnt);
        buf.resize(cnt.n);
        Writer w{buf.data(), 0, cnt.n, false};
        gen_kernel(g, k, &w);
        fwrite(buf.data(), 1, w.n, stdout);
    }
}
