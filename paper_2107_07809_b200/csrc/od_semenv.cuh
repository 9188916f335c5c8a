// ocldec-b200: execution environments and trace hashing of the batched
// semantic check, shared by the device check
// (od_oracle.cuh) and the host reference run that pins it
// (oracle/ref_driver.cpp ref_semcheck): both build environment n of kernel k
// from the same counter-based stream, so their write traces are comparable.
//
// Environment layout follows the reference harness's sampler
// (tests/support/envgen.cpp:50-82): per dimension a group count in [1, 4],
// a group id and a local id (all ids 0 in environment 0), a global offset in
// [0, 16]; pointer arguments get distinct 64-byte aligned bases far from zero
// and from the kernarg window; float scalars come from a small palette,
// 64-bit scalars from [0, 100000), narrower ones from [0, 300].  The random
// stream is splitmix64 (oracle.cpp:22-27) instead of std::mt19937_64, so the
// device can regenerate it.
#pragma once

#include "od_base.cuh"

namespace od {

struct SemRng {
    u64 st;
    OD_INL u64 next() {
        st += 0x9e3779b97f4a7c15ull;
        u64 z = st;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
};

// The NDRange part of an environment (OracleEnv, oracle.hpp:31-47).
struct SemEnv {
    u32 dims;
    u32 cws[3], num_groups[3], group_id[3], local_id[3];
    u64 global_offset[3];
    u64 mem_seed;
    u64 next_base; // next pointer-argument base
};

OD_INL SemRng sem_stream(u64 seed, u64 kernel, u32 env) {
    SemRng r{seed ^ (kernel * 0xd1342543de82ef95ull) ^ ((u64)env << 48)};
    r.next();
    return r;
}

OD_INL void sem_env(SemRng &r, u32 env, u32 dims, const u32 *cws, SemEnv *e) {
    e->dims = dims;
    e->mem_seed = r.next();
    const bool origin = env == 0;
    for (u32 d = 0; d < 3; ++d) {
        e->cws[d] = 1;
        e->num_groups[d] = 1;
        e->group_id[d] = 0;
        e->local_id[d] = 0;
        e->global_offset[d] = 0;
        if (d >= dims)
            continue;
        e->cws[d] = cws[d];
        e->num_groups[d] = 1 + (u32)(r.next() % 4);
        e->group_id[d] = origin ? 0 : (u32)(r.next() % e->num_groups[d]);
        e->local_id[d] = origin ? 0 : (u32)(r.next() % (e->cws[d] ? e->cws[d] : 1));
        e->global_offset[d] = origin ? 0 : r.next() % 17;
    }
    e->next_base = 0x104000000000ull + (r.next() % 1024) * 0x1000;
}

// The value of the next non-implicit argument (in declaration order).
OD_INL u64 sem_arg(SemRng &r, SemEnv *e, bool pointer, bool is_float, u32 bits) {
    if (pointer) {
        const u64 b = e->next_base;
        e->next_base += 0x40000000ull + (r.next() % 256) * 64;
        return b;
    }
    if (is_float) {
        // 0, 1, -1, 0.5, -0.25, 2, 3.5, -8, 100, 0.75, -0.125 (envgen.cpp:21-22)
        const u32 palette[11] = {0x00000000u, 0x3f800000u, 0xbf800000u, 0x3f000000u, 0xbe800000u, 0x40000000u,
                                 0x40600000u, 0xc1000000u, 0x42c80000u, 0x3f400000u, 0xbe000000u};
        return palette[r.next() % 11];
    }
    if (bits == 64)
        return r.next() % 100000;
    u64 v = r.next() % 301;
    if (bits < 32)
        v &= (1ull << bits) - 1;
    return v;
}

// OracleEnv::initial_memory (oracle.cpp:616-618)
OD_INL u32 sem_initial_memory(u64 mem_seed, u64 addr) {
    u64 x = (addr ^ mem_seed) + 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return (u32)(x ^ (x >> 31));
}

// Hash of one write trace: FNV-1a over (address, 8 bytes LE; value, 4 bytes LE).
OD_INL u64 sem_trace_step(u64 h, u64 addr, u32 value) {
    for (u32 i = 0; i < 8; ++i) {
        h ^= (addr >> (8 * i)) & 0xff;
        h *= 1099511628211ull;
    }
    for (u32 i = 0; i < 4; ++i) {
        h ^= (value >> (8 * i)) & 0xff;
        h *= 1099511628211ull;
    }
    return h;
}
constexpr u64 kSemTraceSeed = 1469598103934665603ull;

// The kernel's hash over its environments: an order-free sum, so each lane
// can hash its own environment.
OD_INL u64 sem_env_mix(u64 trace_hash, u64 count, u32 env) {
    u64 x = trace_hash ^ (count << 40) ^ ((u64)env * 0x9e3779b97f4a7c15ull);
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// Verdict of one kernel's check (SemResult::status).
enum SemStatus : u32 {
    SEM_EQUAL = 0,       // identical traces in every environment
    SEM_MISMATCH = 1,    // some environment's traces differ
    SEM_UNSUPPORTED = 2, // either side left the interpreted subset (OracleUnsupported)
    SEM_CAPACITY = 3,    // the device's trace or variable room ran out (not compared)
    SEM_NOT_RUN = 4,     // the kernel failed or was skipped
    SEM_INDETERMINATE = 5, // an operation met two NaNs of different payloads: IEEE 754
                           // leaves the result's payload open (od_oracle.cuh sem_nan)
    SEM_DEFERRED = 6,      // internal: over the in-wave step budget, re-checked at the run's end
};

struct SemResult {
    u32 status;
    u32 envs;
    u64 hash_asm;  // sum over environments of sem_env_mix(trace hash, length, env)
    u64 hash_body;
};

} // namespace od
