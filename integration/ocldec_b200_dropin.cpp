// ocldec-b200 drop-in for the reference's front door (INTEGRATION.md §3,
// Option A): this translation unit REPLACES the reference's
// proj/core/src/decompiler.cpp in a build of the reference, defining
//
//   ocldec::decompile_listing   decompiler.hpp:62 / decompiler.cpp:117-133
//   DecompileResult::combined_source  decompiler.cpp:105-115
//
// over the C ABI of libocldec_b200.so (include/ocldec_b200.h).  Every other
// reference object links unchanged, so the reference's own callers (its
// acceptance harness, tests/acceptance/acceptance_main.cpp, and its CLI)
// run their decompile_listing calls on the GPU.  oracle/dropin.mk builds
// the reference's acceptance harness this way (tests/test_gpu_dropin.py).
//
// Filled from the GPU result: name, source, failed, structured,
// body.fallback_count, cfg_dot, reduction (merges, root / residue, dumps,
// and the region tree those describe, owned by `regions`), and
// DecompileResult::diagnostics in sink order.  Not filled: config,
// instructions, abi, cfg and body.stmts (in-memory inspection structures the
// GPU path does not produce).  No CPU fallback: a
// device or API failure throws std::runtime_error with the library's
// message, where the reference would have returned output.
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ocldec/decompiler.hpp"
#include "ocldec_b200.h"

namespace ocldec {

std::string DecompileResult::combined_source() const {
    std::string out;
    for (const DecompiledKernel &k : kernels) {
        if (k.source.empty())
            continue;
        if (!out.empty())
            out += "\n";
        out += k.source;
    }
    return out;
}

namespace {

// The region tree a reduction record describes (structurizer.hpp:54-104):
// leaf regions 1..L first, then one region per merge, in merge order (region
// ids increase monotonically, RegionGraph::make_region).
void rebuild_regions(const std::string &text, DecompiledKernel &k) {
    std::vector<MergeRecord> merges;
    int root = 0;
    std::vector<int> residue;
    bool reduced = false;
    std::istringstream in(text);
    std::string line;
    while (std::getline(in, line)) {
        std::istringstream w(line);
        std::string tag;
        w >> tag;
        if (tag == "merge") {
            int kind = 0;
            MergeRecord m;
            w >> kind >> m.result;
            m.kind = static_cast<RegionKind>(kind);
            for (int a; w >> a;)
                m.absorbed.push_back(a);
            merges.push_back(std::move(m));
        } else if (tag == "root") {
            w >> root;
            reduced = true;
        } else if (tag == "residue") {
            for (int a; w >> a;)
                residue.push_back(a);
        }
    }
    int leaves = 0;
    if (!merges.empty())
        leaves = merges.front().result - 1;
    else if (reduced)
        leaves = root;
    else
        for (int r : residue)
            leaves = std::max(leaves, r);
    auto g = std::make_unique<RegionGraph>();
    for (int i = 1; i <= leaves; ++i)
        g->add_block(-1); // block ids are not part of the record
    for (const MergeRecord &m : merges) {
        Region *r = g->add_block(-1);
        if (r->id != m.result)
            throw std::runtime_error("ocldec-b200: inconsistent reduction record");
        r->kind = m.kind;
        r->block_id = -1;
        for (int a : m.absorbed)
            r->children.push_back(g->region(a));
        r->join_absorbed = (m.kind == RegionKind::IfThen && m.absorbed.size() == 3) ||
                           (m.kind == RegionKind::IfElse && m.absorbed.size() == 4);
    }
    k.reduction.merges = std::move(merges);
    k.reduction.reduced = reduced;
    if (reduced)
        k.reduction.root = g->region(root);
    for (int r : residue)
        k.reduction.residue.push_back(g->region(r));
    k.regions = std::move(g);
}

} // namespace

DecompileResult decompile_listing(const std::string &listing, const DecompileOptions &opts) {
    ocldec_b200_options o{};
    o.fold_local_size = opts.folds.fold_local_size ? 1 : 0;
    o.only_kernel = opts.only_kernel ? opts.only_kernel->c_str() : nullptr;
    std::string amap; // abi_overrides back to the file form parse_abi_overrides reads
    for (const AbiOverride &ov : opts.abi_overrides)
        amap += std::to_string(ov.offset) + ":" + std::to_string(int(ov.dwords)) + "=" + ov.target + "\n";
    o.abi_map = opts.abi_overrides.empty() ? nullptr : amap.data();
    o.abi_map_len = amap.size();
    o.dump_cfg = opts.dump_cfg ? 1 : 0;
    o.dump_regions = opts.dump_regions ? 1 : 0;
    o.record_reduction = 1;
    ocldec_b200_result *r = nullptr;
    if (int rc = ocldec_b200_decompile(listing.data(), listing.size(), &o, &r))
        throw std::runtime_error("ocldec-b200: decompile failed (" + std::to_string(rc) +
                                 "): " + ocldec_b200_last_error());
    DecompileResult result;
    for (uint64_t i = 0; i < r->ndiags; ++i) { // DiagnosticSink, in order
        const ocldec_b200_diag &d = r->diags[i];
        std::string msg(r->diag_text + d.msg_off, d.msg_len);
        if (d.severity == 0)
            result.diagnostics.note(d.line, std::move(msg));
        else if (d.severity == 1)
            result.diagnostics.warning(d.line, std::move(msg));
        else
            result.diagnostics.error(d.line, std::move(msg));
    }
    result.kernels.resize(r->nkernels);
    for (uint64_t i = 0; i < r->nkernels; ++i) {
        const ocldec_b200_kernel &k = r->kernels[i];
        DecompiledKernel &d = result.kernels[i];
        d.name.assign(r->names + k.name_off, k.name_len);
        d.source.assign(r->combined + k.src_off, k.src_len);
        d.structured = k.structured != 0;
        d.failed = k.failed != 0;
        d.body.fallback_count = k.fallback_count;
    }
    for (uint64_t i = 0; i < r->ndumps; ++i) {
        const ocldec_b200_dump &d = r->dumps[i];
        std::string text(r->dump_text + d.off, d.len);
        DecompiledKernel &k = result.kernels[d.kernel];
        if (d.step == -1)
            k.cfg_dot = std::move(text);
        else if (d.step == -2)
            rebuild_regions(text, k);
        else
            k.reduction.dumps.push_back(std::move(text));
    }
    ocldec_b200_free(r);
    return result;
}

} // namespace ocldec
