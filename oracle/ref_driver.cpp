// TEST INFRASTRUCTURE ONLY — the parity oracle, never the product path.
//
// Thin C ABI over the *unmodified* reference decompiler, compiled straight
// from its sources under /root/reference/proj/core/src by oracle/Makefile
// into oracle/_ref/libocldec_ref.so.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg may load it.
//
// Entry points wrap:
//   ocldec::decompile_listing          proj/core/src/decompiler.cpp:117-133
//   DecompileResult::combined_source   proj/core/src/decompiler.cpp:105-115
//   Diagnostic::render                 proj/core/src/diagnostics.cpp:22-26
//   ocldec_tests::corpus / make_nest   proj/tests/support/{corpus,nestgen}.cpp
//
// The reference recurses per region nesting level (lower.cpp:123-172) and
// overflows an 8 MB stack at ~230 nested regions, so every call
// runs on a pthread with a 1 GiB stack.

#include <pthread.h>
#include <cstdio>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ocldec/decompiler.hpp"
#include "ocldec/oracle.hpp"
#include "corpus.hpp"
#include "../paper_2107_07809_b200/csrc/od_semenv.cuh"
#include "nestgen.hpp"

namespace {

constexpr size_t kBigStack = size_t(1) << 30;

void run_on_big_stack(void *(*fn)(void *), void *arg) {
    pthread_attr_t attr;
    pthread_attr_init(&attr);
    pthread_attr_setstacksize(&attr, kBigStack);
    pthread_t th;
    if (pthread_create(&th, &attr, fn, arg) != 0) {
        fn(arg); // fall back to the caller's stack
    } else {
        pthread_join(th, nullptr);
    }
    pthread_attr_destroy(&attr);
}

char *dup_out(const std::string &s, size_t *len) {
    char *p = static_cast<char *>(std::malloc(s.size() + 1));
    std::memcpy(p, s.data(), s.size());
    p[s.size()] = 0;
    if (len)
        *len = s.size();
    return p;
}

struct DecompileJob {
    const char *listing;
    size_t len;
    int fold_local_size;
    const char *only_kernel;
    const char *abi_map; // override file text (parse_abi_overrides, abi_model.cpp:109-153) or null
    size_t abi_len;
    std::string serialized;
    int dumps = 0; // 1: dump_cfg, 2: dump_regions (DecompileOptions, decompiler.hpp:33-34),
                   // 4: the reduction record (merges, root / residue)
};

// Serialization (parsed by oracle/oracle.py):
//   "K <failed> <structured> <fallbacks> <name_len> <src_len>\n" name source
//   "D <severity> <line> <msg_len>\n" message
//   "C <len>\n" combined_source
//   "G <kernel> <len>\n" cfg_dot, "R <kernel> <step> <len>\n" reduction.dumps[step]
//   "M <kernel> <len>\n" reduction: "merge <kind> <result> <absorbed...>" lines,
//   then "root <id>" or "residue <ids...>"
void *decompile_job(void *p) {
    auto *job = static_cast<DecompileJob *>(p);
    ocldec::DecompileOptions opts;
    opts.folds.fold_local_size = job->fold_local_size != 0;
    if (job->only_kernel)
        opts.only_kernel = std::string(job->only_kernel);
    opts.dump_cfg = (job->dumps & 1) != 0;
    opts.dump_regions = (job->dumps & 2) != 0;
    std::string out;
    if (job->abi_map) {
        ocldec::DiagnosticSink osink;
        opts.abi_overrides = ocldec::parse_abi_overrides(std::string(job->abi_map, job->abi_len), osink);
        for (const auto &d : osink.all()) {
            out += "A " + std::to_string(int(d.severity)) + " " + std::to_string(d.line) + " " +
                   std::to_string(d.message.size()) + "\n";
            out += d.message;
        }
    }
    ocldec::DecompileResult res =
        ocldec::decompile_listing(std::string(job->listing, job->len), opts);
    for (const auto &k : res.kernels) {
        out += "K " + std::to_string(int(k.failed)) + " " + std::to_string(int(k.structured)) +
               " " + std::to_string(k.body.fallback_count) + " " + std::to_string(k.name.size()) +
               " " + std::to_string(k.source.size()) + "\n";
        out += k.name;
        out += k.source;
    }
    for (const auto &d : res.diagnostics.all()) {
        out += "D " + std::to_string(int(d.severity)) + " " + std::to_string(d.line) + " " +
               std::to_string(d.message.size()) + "\n";
        out += d.message;
    }
    for (size_t i = 0; i < res.kernels.size(); ++i) {
        const auto &k = res.kernels[i];
        if (!k.cfg_dot.empty()) {
            out += "G " + std::to_string(i) + " " + std::to_string(k.cfg_dot.size()) + "\n";
            out += k.cfg_dot;
        }
        if ((job->dumps & 4) && !k.failed) {
            std::string m;
            for (const auto &mr : k.reduction.merges) {
                m += "merge " + std::to_string(int(mr.kind)) + " " + std::to_string(mr.result);
                for (int a : mr.absorbed)
                    m += " " + std::to_string(a);
                m += "\n";
            }
            if (k.reduction.reduced) {
                m += "root " + std::to_string(k.reduction.root->id) + "\n";
            } else {
                m += "residue";
                for (const auto *r : k.reduction.residue)
                    m += " " + std::to_string(r->id);
                m += "\n";
            }
            out += "M " + std::to_string(i) + " " + std::to_string(m.size()) + "\n";
            out += m;
        }
        for (size_t j = 0; j < k.reduction.dumps.size(); ++j) {
            out += "R " + std::to_string(i) + " " + std::to_string(j) + " " +
                   std::to_string(k.reduction.dumps[j].size()) + "\n";
            out += k.reduction.dumps[j];
        }
    }
    std::string combined = res.combined_source();
    out += "C " + std::to_string(combined.size()) + "\n";
    out += combined;
    job->serialized = std::move(out);
    return nullptr;
}

struct BatchJob {
    const char *corpus;
    const uint64_t *offsets; // nkernels + 1 byte offsets of per-kernel listings
    size_t nkernels;
    std::atomic<size_t> *next;
    uint64_t *out_hash; // per kernel FNV-1a of source (0 when null)
    uint64_t *out_len;  // per kernel source length
    uint64_t instructions = 0;
};

uint64_t fnv1a(const std::string &s) {
    uint64_t h = 1469598103934665603ull;
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

void *batch_worker(void *p) {
    auto *job = static_cast<BatchJob *>(p);
    for (;;) {
        size_t k = job->next->fetch_add(1);
        if (k >= job->nkernels)
            break;
        std::string listing(job->corpus + job->offsets[k], job->offsets[k + 1] - job->offsets[k]);
        ocldec::DecompileResult res = ocldec::decompile_listing(listing);
        std::string src = res.combined_source();
        if (job->out_hash)
            job->out_hash[k] = fnv1a(src);
        if (job->out_len)
            job->out_len[k] = src.size();
        for (const auto &kk : res.kernels)
            job->instructions += kk.instructions.size();
    }
    return nullptr;
}

struct ParSlice {
    const char *text;
    size_t len;
    int fold_local_size;
    std::string kernels; // "K" records
    std::string diags;   // "D" records, lines shifted to the whole listing
    std::string combined;
    uint64_t line_base = 0;
};

struct ParJob {
    std::vector<ParSlice> *slices;
    std::atomic<size_t> *next;
};

void *par_worker(void *p) {
    auto *job = static_cast<ParJob *>(p);
    for (;;) {
        size_t i = job->next->fetch_add(1);
        if (i >= job->slices->size())
            break;
        ParSlice &sl = (*job->slices)[i];
        ocldec::DecompileOptions opts;
        opts.folds.fold_local_size = sl.fold_local_size != 0;
        ocldec::DecompileResult res = ocldec::decompile_listing(std::string(sl.text, sl.len), opts);
        for (const auto &k : res.kernels) {
            sl.kernels += "K " + std::to_string(int(k.failed)) + " " + std::to_string(int(k.structured)) +
                          " " + std::to_string(k.body.fallback_count) + " " + std::to_string(k.name.size()) +
                          " " + std::to_string(k.source.size()) + "\n";
            sl.kernels += k.name;
            sl.kernels += k.source;
        }
        for (const auto &d : res.diagnostics.all()) {
            const uint64_t line = d.line > 0 ? uint64_t(d.line) + sl.line_base : uint64_t(d.line);
            sl.diags += "D " + std::to_string(int(d.severity)) + " " + std::to_string(line) + " " +
                        std::to_string(d.message.size()) + "\n";
            sl.diags += d.message;
        }
        sl.combined = res.combined_source();
    }
    return nullptr;
}

} // namespace

extern "C" {

// Decompiles one listing; *out receives the serialized result (free with
// ref_free). Returns 0.
int ref_decompile(const char *listing, size_t len, int fold_local_size, const char *only_kernel,
                  char **out, size_t *out_len) {
    DecompileJob job{listing, len, fold_local_size, only_kernel, nullptr, 0, {}};
    run_on_big_stack(decompile_job, &job);
    *out = dup_out(job.serialized, out_len);
    return 0;
}

// The same with an ABI override file (the CLI's --abi-map, ocldec.cpp:116-131):
// its parse diagnostics come first as "A <severity> <line> <len>" records.
int ref_decompile_abi(const char *listing, size_t len, int fold_local_size, const char *only_kernel,
                      const char *abi_map, size_t abi_len, char **out, size_t *out_len) {
    DecompileJob job{listing, len, fold_local_size, only_kernel, abi_map, abi_len, {}};
    run_on_big_stack(decompile_job, &job);
    *out = dup_out(job.serialized, out_len);
    return 0;
}

// Everything: options, ABI override text (null = none) and the DOT dumps
// (dumps bit 0: dump_cfg, bit 1: dump_regions).
int ref_decompile_ex(const char *listing, size_t len, int fold_local_size, const char *only_kernel,
                     const char *abi_map, size_t abi_len, int dumps, char **out, size_t *out_len) {
    DecompileJob job{listing, len, fold_local_size, only_kernel, abi_map, abi_len, {}, dumps};
    run_on_big_stack(decompile_job, &job);
    *out = dup_out(job.serialized, out_len);
    return 0;
}

void ref_free(void *p) { std::free(p); }

// Decompiles nkernels independent per-kernel listings, slices
// corpus[offsets[k], offsets[k+1]), on nthreads pthreads with 1 GiB stacks
// pulling an atomic work index (the CPU-baseline recipe of SURVEY §8(d)).
// Writes per-kernel source hash/length when the arrays are non-null.
// Returns wall seconds; *instructions gets the parse_text instruction count
// (DecompiledKernel::instructions includes a synthetic trailing s_endpgm
// only when a listing ends on a label; the synthetic generator never does).
double ref_decompile_batch(const char *corpus, const uint64_t *offsets, size_t nkernels,
                           int nthreads, uint64_t *out_hash, uint64_t *out_len,
                           uint64_t *instructions) {
    if (nthreads < 1)
        nthreads = 1;
    std::atomic<size_t> next{0};
    std::vector<BatchJob> jobs(static_cast<size_t>(nthreads));
    std::vector<pthread_t> threads(static_cast<size_t>(nthreads));
    pthread_attr_t attr;
    pthread_attr_init(&attr);
    pthread_attr_setstacksize(&attr, kBigStack);
    auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < nthreads; ++t) {
        jobs[size_t(t)] = BatchJob{corpus, offsets, nkernels, &next, out_hash, out_len, 0};
        pthread_create(&threads[size_t(t)], &attr, batch_worker, &jobs[size_t(t)]);
    }
    uint64_t total = 0;
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(threads[size_t(t)], nullptr);
        total += jobs[size_t(t)].instructions;
    }
    auto t1 = std::chrono::steady_clock::now();
    pthread_attr_destroy(&attr);
    if (instructions)
        *instructions = total;
    return std::chrono::duration<double>(t1 - t0).count();
}

// The reference's 26-kernel test corpus (proj/tests/support/corpus.cpp).
int ref_corpus_count(void) { return int(ocldec_tests::corpus().size()); }

int ref_corpus_get(int i, char **name, char **listing, int *comparable, int *expected_fallbacks) {
    const auto &ks = ocldec_tests::corpus();
    if (i < 0 || size_t(i) >= ks.size())
        return -1;
    const auto &k = ks[size_t(i)];
    *name = dup_out(k.name, nullptr);
    *listing = dup_out(k.listing, nullptr);
    *comparable = k.comparable ? 1 : 0;
    *expected_fallbacks = k.expected_fallbacks;
    return 0;
}

// The reference's deterministic nest generator (proj/tests/support/nestgen.cpp).
char *ref_make_nest(uint64_t seed, int *conditionals) {
    ocldec_tests::NestSpec spec = ocldec_tests::make_nest(seed);
    if (conditionals)
        *conditionals = spec.conditionals;
    return dup_out(spec.listing, nullptr);
}


// decompile_listing over a listing whose kernel sections start at the byte
// offsets kstart[0..nk) (each a ".kernel" line; kstart[0] may follow a
// preamble that split_kernels ignores), computed in parallel: the sections
// are independent (decompiler.cpp:55-101), so slices of `per` kernels are
// decompiled on nthreads pthreads (1 GiB stacks) and joined as
// combined_source joins them (decompiler.cpp:105-115), diagnostic lines
// shifted by each slice's line offset.  Same serialization as ref_decompile
// (no dumps).  Only for listings without split_kernels errors.
int ref_decompile_par(const char *listing, size_t len, const uint64_t *kstart, size_t nk, size_t per,
                      int nthreads, int fold_local_size, char **out, size_t *out_len) {
    if (per < 1)
        per = 1;
    if (nthreads < 1)
        nthreads = 1;
    std::vector<ParSlice> slices;
    uint64_t line = 0, pos = 0;
    for (size_t k0 = 0; k0 < nk; k0 += per) {
        const uint64_t a = k0 == 0 ? 0 : kstart[k0];
        const uint64_t b = k0 + per < nk ? kstart[k0 + per] : len;
        for (; pos < a; ++pos)
            line += listing[pos] == '\n';
        ParSlice sl;
        sl.text = listing + a;
        sl.len = b - a;
        sl.fold_local_size = fold_local_size;
        sl.line_base = line;
        slices.push_back(std::move(sl));
    }
    std::atomic<size_t> next{0};
    std::vector<pthread_t> threads(static_cast<size_t>(nthreads));
    std::vector<ParJob> jobs(static_cast<size_t>(nthreads));
    pthread_attr_t attr;
    pthread_attr_init(&attr);
    pthread_attr_setstacksize(&attr, kBigStack);
    for (int t = 0; t < nthreads; ++t) {
        jobs[size_t(t)] = ParJob{&slices, &next};
        pthread_create(&threads[size_t(t)], &attr, par_worker, &jobs[size_t(t)]);
    }
    for (int t = 0; t < nthreads; ++t)
        pthread_join(threads[size_t(t)], nullptr);
    pthread_attr_destroy(&attr);
    std::string ser, combined;
    for (const auto &sl : slices)
        ser += sl.kernels;
    for (const auto &sl : slices)
        ser += sl.diags;
    for (const auto &sl : slices) {
        if (sl.combined.empty())
            continue;
        if (!combined.empty())
            combined += "\n";
        combined += sl.combined;
    }
    ser += "C " + std::to_string(combined.size()) + "\n";
    ser += combined;
    *out = dup_out(ser, out_len);
    return 0;
}


// The reference side of the batched semantic check (od_oracle.cuh): for every
// kernel of decompile_listing(listing), the reference's own interpret_asm and
// evaluate_decompiled (oracle.cpp:620-842) over the 8 environments
// od_semenv.cuh derives from (seed, kernel index, environment index).
// out: 4 u64 per kernel {status, envs, hash_asm, hash_body} with the device
// check's statuses (0 equal, 1 mismatch, 2 unsupported, 4 not run).  Returns
// the kernel count (<= cap).
struct SemJob {
    const char *listing;
    size_t len;
    uint64_t seed;
    uint64_t *out;
    size_t cap;
    uint64_t kbase = 0; // listing ordinal of the first kernel (slices of a larger listing)
    size_t nk = 0;
};

void *semcheck_job(void *p) {
    auto *job = static_cast<SemJob *>(p);
    using namespace ocldec;
    DecompileResult res = decompile_listing(std::string(job->listing, job->len));
    job->nk = res.kernels.size();
    for (size_t k = 0; k < res.kernels.size() && k < job->cap; ++k) {
        const DecompiledKernel &K = res.kernels[k];
        uint64_t *o = job->out + 4 * k;
        if (K.failed) {
            o[0] = od::SEM_NOT_RUN, o[1] = 0, o[2] = 0, o[3] = 0;
            continue;
        }
        bool unsupported = false, mismatch = false;
        uint64_t ha = 0, hb = 0;
        const uint32_t envs = 8;
        for (uint32_t n = 0; n < envs; ++n) {
            od::SemRng r = od::sem_stream(job->seed, job->kbase + k, n);
            od::SemEnv e;
            const uint32_t cws[3] = {K.config.cws[0], K.config.cws[1], K.config.cws[2]};
            od::sem_env(r, n, uint32_t(K.config.dims), cws, &e);
            OracleEnv env;
            env.dims = K.config.dims;
            for (int d = 0; d < 3; ++d) {
                env.cws[size_t(d)] = e.cws[d];
                env.num_groups[size_t(d)] = e.num_groups[d];
                env.group_id[size_t(d)] = e.group_id[d];
                env.local_id[size_t(d)] = e.local_id[d];
                env.global_offset[size_t(d)] = e.global_offset[d];
            }
            env.mem_seed = e.mem_seed;
            for (const ArgDecl &a : K.config.args)
                if (!a.is_implicit)
                    env.arg_values[a.name] =
                        od::sem_arg(r, &e, a.type.is_pointer(), a.type.is_float(), a.type.bits);
            WriteTrace A, B;
            try {
                A = interpret_asm(K.instructions, K.config, K.abi, env);
                B = evaluate_decompiled(K.body, K.config, env);
            } catch (const std::exception &) { // OracleUnsupported (or an out-of-range register)
                unsupported = true;
                continue;
            }
            if (getenv("OCLDEC_SEM_DEBUG")) {
                fprintf(stderr, "S %zu %u asm n=%zu [", k, n, A.size());
                for (const TraceEntry &t : A)
                    fprintf(stderr, " %llx:%x", (unsigned long long)t.addr, t.value);
                fprintf(stderr, " ] body n=%zu [", B.size());
                for (const TraceEntry &t : B)
                    fprintf(stderr, " %llx:%x", (unsigned long long)t.addr, t.value);
                fprintf(stderr, " ]\n");
            }
            uint64_t h = od::kSemTraceSeed;
            for (const TraceEntry &t : A)
                h = od::sem_trace_step(h, t.addr, t.value);
            ha += od::sem_env_mix(h, A.size(), n);
            h = od::kSemTraceSeed;
            for (const TraceEntry &t : B)
                h = od::sem_trace_step(h, t.addr, t.value);
            hb += od::sem_env_mix(h, B.size(), n);
            mismatch |= !(A == B);
        }
        o[0] = unsupported ? od::SEM_UNSUPPORTED : mismatch ? od::SEM_MISMATCH : od::SEM_EQUAL;
        o[1] = envs;
        o[2] = ha;
        o[3] = hb;
    }
    return nullptr;
}

int64_t ref_semcheck(const char *listing, size_t len, uint64_t seed, uint64_t *out, size_t cap) {
    SemJob job{listing, len, seed, out, cap};
    run_on_big_stack(semcheck_job, &job);
    return int64_t(job.nk);
}

// The same over a slice of a larger listing whose first kernel is kernel
// `kbase` of the whole (oracle.py runs slices on several threads).
int64_t ref_semcheck_at(const char *listing, size_t len, uint64_t seed, uint64_t kbase, uint64_t *out,
                        size_t cap) {
    SemJob job{listing, len, seed, out, cap, kbase};
    run_on_big_stack(semcheck_job, &job);
    return int64_t(job.nk);
}

} // extern "C"
