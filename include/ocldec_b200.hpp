// ocldec-b200: C++ front door with the reference's shape.
//
// Header-only shim over the C ABI (ocldec_b200.h) that mirrors
//   ocldec::decompile_listing(const std::string&, const DecompileOptions&)
//       /root/reference/proj/core/include/ocldec/decompiler.hpp:62
// with the fields a caller of the reference consumes on this path:
//   DecompiledKernel{name, source, structured, failed} (decompiler.hpp:39-52)
//   LoweredBody::fallback_count                        (lower.hpp:23-41)
//   DecompileResult::combined_source()                 (decompiler.cpp:105-115)
//   DecompileResult::diagnostics (DiagnosticSink, diagnostics.hpp:20-57):
//   every note / warning / error the reference emits on this path
//   DecompileOptions::abi_overrides (decompiler.hpp:31), given as the override
//   file text the CLI's --abi-map reads (parse_abi_overrides, abi_model.cpp);
//   its parse diagnostics come back in abi_diagnostics
//   DecompiledKernel::cfg_dot and reduction.dumps (the DOT dumps)
// The other inspection fields (config, instructions, cfg, regions, body tree)
// are not produced.  All work runs on the GPU; errors from the device runtime are
// thrown as std::runtime_error (API misuse / CUDA failure only — data errors
// come back in the result exactly as the reference reports them).
#ifndef OCLDEC_B200_HPP
#define OCLDEC_B200_HPP

#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "ocldec_b200.h"

namespace ocldec_b200 {

struct DecompileOptions {
    bool fold_local_size = false; // FoldOptions::fold_local_size (sym_state.hpp:27-29)
    std::string only_kernel;      // empty = all kernels (DecompileOptions::only_kernel)
    std::string abi_map;          // ABI override file text; empty = none
    bool dump_cfg = false;        // DecompileOptions::dump_cfg (decompiler.hpp:33)
    bool dump_regions = false;    // DecompileOptions::dump_regions (decompiler.hpp:34)
    bool record_reduction = false; // fill DecompiledKernel::reduction (merges, root / residue)
    bool export_body = false;     // fill DecompiledKernel::body_text (the lowered statement tree)
    bool semantic_check = false;  // the batched semantic check (DecompiledKernel::semantic)
    uint64_t semantic_seed = 0;   // its environment seed
    int device = 0;
    std::vector<int> devices;     // non-empty: shard across these devices (ocldec_b200_decompile_multi)
};

// MergeRecord (structurizer.hpp:54-58); kind: 1 Linear, 2 IfThen, 3 IfElse.
struct MergeRecord {
    int kind = 1;
    std::vector<int> absorbed;
    int result = 0;
};

// ReduceResult's inspection part (structurizer.hpp:98-104), region ids.
struct Reduction {
    std::vector<MergeRecord> merges;
    bool reduced = false;
    int root = 0;             // when reduced
    std::vector<int> residue; // top-level regions when not
};

struct DecompiledKernel {
    std::string name;
    std::string source;
    bool structured = false;
    bool failed = false;
    int fallback_count = 0;
    unsigned instructions = 0;
    std::string cfg_dot;                   // DecompiledKernel::cfg_dot when dump_cfg
    std::vector<std::string> region_dumps; // ReduceResult::dumps when dump_regions
    Reduction reduction;                   // when record_reduction
    std::string body_text;                 // the lowered statement tree when export_body (step -3)
    std::string cfg_text;                  // the normalized flow graph when export_body (step -4)
    ocldec_b200_semcheck semantic{4, 0, 0, 0}; // when semantic_check: status (0 equal, 1 mismatch,
                                               // 2 unsupported, 3 capacity, 4 not run, 5 indeterminate)
};

inline Reduction parse_reduction(const std::string &text) {
    Reduction r;
    size_t p = 0;
    while (p < text.size()) {
        size_t e = text.find('\n', p);
        if (e == std::string::npos)
            e = text.size();
        std::vector<int> v;
        std::string word;
        const char *c = text.c_str() + p, *end = text.c_str() + e;
        while (c < end && *c != ' ')
            word += *c++;
        while (c < end) {
            char *q = nullptr;
            v.push_back(static_cast<int>(std::strtol(c, &q, 10)));
            c = q;
        }
        if (word == "merge" && v.size() >= 2) {
            MergeRecord m;
            m.kind = v[0];
            m.result = v[1];
            m.absorbed.assign(v.begin() + 2, v.end());
            r.merges.push_back(std::move(m));
        } else if (word == "root" && !v.empty()) {
            r.reduced = true;
            r.root = v[0];
        } else if (word == "residue") {
            r.residue = v;
        }
        p = e + 1;
    }
    return r;
}

// Diagnostic (diagnostics.hpp:20-27); render() matches diagnostics.cpp:22-26.
struct Diagnostic {
    enum Severity { Note = 0, Warning = 1, Error = 2 } severity = Error;
    int line = 0;
    std::string message;
    std::string render(const std::string &file) const {
        static const char *names[] = {"note", "warning", "error"};
        return file + ":" + std::to_string(line) + ": " + names[severity] + ": " + message;
    }
};

struct DecompileResult {
    std::vector<DecompiledKernel> kernels;
    std::vector<Diagnostic> diagnostics;
    std::vector<Diagnostic> abi_diagnostics; // parse_abi_overrides' sink
    double device_ms = 0;
    bool has_errors() const {
        for (const auto &d : diagnostics)
            if (d.severity == Diagnostic::Error)
                return true;
        return false;
    }
    // decompiler.cpp:105-115: non-empty sources joined by "\n".
    std::string combined_source() const {
        std::string out;
        for (const auto &k : kernels) {
            if (k.source.empty())
                continue;
            if (!out.empty())
                out += "\n";
            out += k.source;
        }
        return out;
    }
};

inline const char *split_error_message(int kind) {
    switch (kind) {
    case 1: return ".kernel directive without a name";
    case 2: return ".config outside of a .kernel section";
    case 3: return ".text outside of a .kernel section";
    default: return "parse error";
    }
}

// parse_abi_overrides alone (the CLI's --abi-map check before decompiling).
inline std::vector<Diagnostic> check_abi_map(const std::string &text) {
    std::vector<char> buf(4096 + 4 * text.size());
    int rc;
    while ((rc = ocldec_b200_abi_map_check(text.data(), text.size(), buf.data(), buf.size())) == -2)
        buf.resize(buf.size() * 2);
    if (rc < 0)
        throw std::runtime_error(std::string("ocldec_b200_abi_map_check: ") + ocldec_b200_last_error());
    std::vector<Diagnostic> out;
    const char *p = buf.data();
    while (*p) {
        const char *e = std::strchr(p, '\n');
        Diagnostic d;
        char *q = nullptr;
        d.severity = static_cast<Diagnostic::Severity>(std::strtol(p, &q, 10));
        d.line = static_cast<int>(std::strtol(q, &q, 10));
        d.message.assign(static_cast<const char *>(q + 1), e);
        out.push_back(std::move(d));
        p = e + 1;
    }
    return out;
}

inline DecompileResult decompile_listing(const std::string &listing, const DecompileOptions &opts = {}) {
    ocldec_b200_options o{};
    o.fold_local_size = opts.fold_local_size ? 1 : 0;
    o.only_kernel = opts.only_kernel.empty() ? nullptr : opts.only_kernel.c_str();
    o.device = opts.device;
    o.arena_bytes = 0;
    o.abi_map = opts.abi_map.empty() ? nullptr : opts.abi_map.data();
    o.abi_map_len = opts.abi_map.size();
    o.dump_cfg = opts.dump_cfg ? 1 : 0;
    o.dump_regions = opts.dump_regions ? 1 : 0;
    o.record_reduction = opts.record_reduction ? 1 : 0;
    o.export_body = opts.export_body ? 1 : 0;
    o.semantic_check = opts.semantic_check ? 1 : 0;
    o.semantic_seed = opts.semantic_seed;
    ocldec_b200_result *r = nullptr;
    int rc = opts.devices.empty()
                 ? ocldec_b200_decompile(listing.data(), listing.size(), &o, &r)
                 : ocldec_b200_decompile_multi(listing.data(), listing.size(), &o, opts.devices.data(),
                                               (int)opts.devices.size(), &r);
    if (rc != 0)
        throw std::runtime_error(std::string("ocldec_b200_decompile: ") + ocldec_b200_last_error());
    DecompileResult res;
    res.device_ms = r->device_ms;
    for (uint64_t i = 0; i < r->nkernels; ++i) {
        const ocldec_b200_kernel &k = r->kernels[i];
        DecompiledKernel d;
        d.name.assign(r->names + k.name_off, k.name_len);
        if (k.src_len)
            d.source.assign(r->combined + k.src_off, k.src_len);
        d.structured = k.structured != 0;
        d.failed = k.failed != 0;
        d.fallback_count = k.fallback_count;
        if (r->sem)
            d.semantic = r->sem[i];
        d.instructions = k.instructions;
        res.kernels.push_back(std::move(d));
    }
    for (uint64_t i = 0; i < r->ndumps; ++i) {
        const ocldec_b200_dump &d = r->dumps[i];
        DecompiledKernel &k = res.kernels[d.kernel];
        std::string text(r->dump_text + d.off, d.len);
        if (d.step == -1)
            k.cfg_dot = std::move(text);
        else if (d.step == -3)
            k.body_text = std::move(text);
        else if (d.step == -4)
            k.cfg_text = std::move(text);
        else if (d.step == -2)
            k.reduction = parse_reduction(text);
        else
            k.region_dumps.push_back(std::move(text));
    }
    auto take = [&](const ocldec_b200_diag *v, uint64_t n, std::vector<Diagnostic> &out) {
        for (uint64_t i = 0; i < n; ++i) {
            Diagnostic dg;
            dg.severity = static_cast<Diagnostic::Severity>(v[i].severity);
            dg.line = v[i].line;
            dg.message.assign(r->diag_text + v[i].msg_off, v[i].msg_len);
            out.push_back(std::move(dg));
        }
    };
    take(r->diags, r->ndiags, res.diagnostics);
    take(r->abi_diags, r->nabi_diags, res.abi_diagnostics);
    ocldec_b200_free(r);
    return res;
}

} // namespace ocldec_b200

#endif // OCLDEC_B200_HPP
