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
// Filled from the GPU result: name, source, failed, structured, body (the
// lowered statement tree with its expressions, exported by the device as
// text, and fallback_count), cfg_dot, reduction (merges, root / residue,
// dumps, and the region tree those describe, owned by `regions`), and
// DecompileResult::diagnostics in sink order.  config, instructions and abi
// are the reference front end's own parse of the kernel's section (host,
// diagnostics discarded: the GPU's are the result's).  cfg is the GPU's flow
// graph after mask normalization (step -4 export): blocks, instruction
// ranges, labels, terminators, successors, reachability, absorbed and
// suppressed marks; preds, exec_ops and the masked terms' source operands
// are rebuilt from those by the reference's own rebuild_preds /
// annotate_exec (oracle/cfg_check.cpp checks the result field by field).
// No CPU fallback for the decompilation: a device or API failure throws
// std::runtime_error with the library's message.
#include <cstdlib>
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

// DataType from the device's packed form (base | bits << 8 | depth << 16 |
// space << 24; the enums share the reference's order).
DataType dtype_of(uint64_t t) {
    DataType d;
    d.base = static_cast<BaseType>(t & 0xff);
    d.bits = uint8_t((t >> 8) & 0xff);
    d.pointer_depth = uint8_t((t >> 16) & 0xff);
    d.addr_space = static_cast<AddressSpace>((t >> 24) & 0xff);
    return d;
}

// LoweredBody from the device's body export (od_lower.cuh body_text).
struct BodyReader {
    const std::string &t;
    size_t p = 0;
    std::vector<ExprPtr> nodes{nullptr}; // export number -> node
    uint64_t num() {
        while (p < t.size() && t[p] == ' ')
            ++p;
        uint64_t v = 0;
        while (p < t.size() && t[p] >= '0' && t[p] <= '9')
            v = v * 10 + uint64_t(t[p++] - '0');
        return v;
    }
    std::string str() { // "<len> <bytes>"
        const size_t n = num();
        ++p; // the separating space
        std::string s = t.substr(p, n);
        p += n;
        return s;
    }
    ExprPtr node(uint64_t id) {
        if (id >= nodes.size())
            throw std::runtime_error("ocldec-b200: bad body export (node " + std::to_string(id) + ")");
        return nodes[id];
    }
    void eol() {
        while (p < t.size() && t[p] != '\n')
            ++p;
        ++p;
    }
    void read_node() {
        auto e = std::make_shared<Expr>();
        const uint64_t kind = num(), op = num(), x = num(), type = num(), a = num(), b = num(), c = num();
        e->kind = static_cast<ExprKind>(kind - 1); // the device's kinds start with a null kind
        e->type = dtype_of(type);
        switch (e->kind) {
        case ExprKind::Const: e->const_value = a | (b << 32); break;
        case ExprKind::Builtin: e->builtin = BuiltinId{static_cast<BuiltinFn>(op), int(x)}; break;
        case ExprKind::KernelArg:
        case ExprKind::Var: e->name = str(); break;
        case ExprKind::Unary: e->un_op = static_cast<UnaryOp>(op), e->a = node(a); break;
        case ExprKind::Binary: e->bin_op = static_cast<BinaryOp>(op), e->a = node(a), e->b = node(b); break;
        case ExprKind::Ternary: e->a = node(a), e->b = node(b), e->c = node(c); break;
        case ExprKind::Deref: e->a = node(a); break;
        default: break;
        }
        eol();
        nodes.push_back(std::move(e));
    }
    // Statements up to the end of the text or of the current If arm.
    void read_list(std::vector<Stmt> &out, char *stop) {
        while (p < t.size()) {
            const char tag = t[p++];
            if (tag == 'N') {
                read_node();
                continue;
            }
            if (tag == 'E' || tag == 'F') {
                eol();
                *stop = tag;
                return;
            }
            Stmt s;
            switch (tag) {
            case 'A':
                s.base.kind = StatementKind::Assign;
                s.base.name = str();
                s.base.value = node(num());
                break;
            case 'D':
                s.base.kind = StatementKind::Decl;
                s.base.name = str();
                s.base.decl_type = dtype_of(num());
                s.base.value = node(num());
                break;
            case 'W':
                s.base.kind = StatementKind::Store;
                s.base.addr = node(num());
                s.base.value = node(num());
                s.base.elem_type = dtype_of(num());
                s.base.space = AddressSpace::Global;
                break;
            case 'R':
                s.base.kind = StatementKind::RawAsm;
                s.base.text = str();
                break;
            case 'L':
                s.kind = StmtKind::Label;
                s.label = str();
                break;
            case 'G':
                s.kind = StmtKind::Goto;
                s.cond = node(num());
                s.label = str();
                break;
            case 'I': {
                s.kind = StmtKind::If;
                s.cond = node(num());
                eol();
                char st = 0;
                read_list(s.then_body, &st);
                if (st == 'E')
                    read_list(s.else_body, &st);
                out.push_back(std::move(s));
                continue;
            }
            default:
                throw std::runtime_error(std::string("ocldec-b200: bad body export record ") + tag);
            }
            eol();
            out.push_back(std::move(s));
        }
        *stop = 0;
    }
};

void read_body(const std::string &text, LoweredBody &body) {
    BodyReader r{text};
    char stop = 0;
    r.read_list(body.stmts, &stop);
}

// decompile_section's parse steps (decompiler.cpp:59-67) for the inspection
// fields: the reference front end on the host, its diagnostics discarded.
// DecompiledKernel::cfg from the device's step -4 record (od_kernel.cuh
// cfg_text) over the kernel's instruction list.
void rebuild_cfg(const std::string &text, DecompiledKernel &k) {
    std::istringstream in(text);
    size_t nb = 0;
    in >> nb;
    Cfg cfg;
    cfg.blocks.resize(nb);
    for (size_t b = 0; b < nb; ++b) {
        BasicBlock &B = cfg.blocks[b];
        std::string tag;
        size_t ib = 0, ie = 0;
        unsigned kind = 0, cc = 0, taken = 0, not_taken = 0, line = 0, reach = 0, absorbed = 0, nsucc = 0;
        in >> tag >> ib >> ie >> kind >> cc >> taken >> not_taken >> line >> reach >> absorbed >> nsucc;
        if (!in || tag != "B" || ib > ie || ie > k.instructions.size())
            throw std::runtime_error("ocldec-b200: malformed cfg record");
        B.id = int(b);
        B.instructions.assign(k.instructions.begin() + long(ib), k.instructions.begin() + long(ie));
        B.suppressed.assign(ie - ib, false);
        B.term.kind = TermKind(kind);
        B.term.cc = CondCode(cc);
        B.term.taken = int(taken) - 1;
        B.term.not_taken = int(not_taken) - 1;
        B.term.line = int(line);
        B.reachable = reach != 0;
        B.mask_absorbed = absorbed != 0;
        for (unsigned q = 0; q < nsucc; ++q) {
            int sc = 0;
            in >> sc;
            B.succs.push_back(sc);
        }
        size_t ns = 0;
        in >> tag >> ns;
        for (size_t q = 0; q < ns; ++q) {
            size_t i = 0;
            in >> i;
            if (i < B.suppressed.size())
                B.suppressed[i] = true;
        }
        size_t nl = 0;
        in >> tag >> nl;
        for (size_t q = 0; q < nl; ++q) {
            std::string l;
            in >> l;
            B.labels.push_back(std::move(l));
        }
        if (B.term.kind == TermKind::Conditional && B.term.cc == CondCode::Masked) {
            // the rewritten header's saved condition: the source operand of
            // its (now suppressed) s_and_saveexec (structurizer.cpp:599-601)
            for (size_t i = B.instructions.size(); i-- > 0;) {
                const Instruction &ins = B.instructions[i];
                if (B.suppressed[i] && !ins.parse_failed && ins.parts.prefix == "s" &&
                    ins.parts.root == "and_saveexec" && ins.operands.size() >= 2) {
                    B.term.mask_source = ins.operands[1];
                    break;
                }
            }
        }
    }
    cfg.entry = 0;
    cfg.rebuild_preds();
    annotate_exec(cfg);
    k.cfg = std::move(cfg);
}

void front_fields(const KernelSection &section, const DecompileOptions &opts, DecompiledKernel &k) {
    DiagnosticSink scratch;
    try {
        k.config = parse_config(section, scratch);
        std::vector<std::string> trailing;
        k.instructions = parse_text(section, scratch, &trailing);
        if (!trailing.empty()) { // attach_trailing_labels (decompiler.cpp:20-31)
            Instruction end;
            end.line = k.instructions.empty() ? section.line : k.instructions.back().line;
            end.labels = std::move(trailing);
            end.source_text = "s_endpgm";
            end.mnemonic = "s_endpgm";
            end.parts = decompose_mnemonic(end.mnemonic);
            k.instructions.push_back(std::move(end));
        }
        k.abi = build_abi_map(k.config, scratch, opts.abi_overrides);
    } catch (const ParseError &) {
    }
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
    o.export_body = 1;
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
    std::vector<std::string> cfg_text(r->nkernels);
    for (uint64_t i = 0; i < r->ndumps; ++i) {
        const ocldec_b200_dump &d = r->dumps[i];
        std::string text(r->dump_text + d.off, d.len);
        DecompiledKernel &k = result.kernels[d.kernel];
        if (d.step == -1)
            k.cfg_dot = std::move(text);
        else if (d.step == -2)
            rebuild_regions(text, k);
        else if (d.step == -3 && !getenv("OCLDEC_B200_DROPIN_NO_BODY")) // (a negative control for tests)
            read_body(text, k.body);
        else if (d.step == -4)
            cfg_text[d.kernel] = std::move(text);
        else if (d.step == -3)
            ;
        else
            k.reduction.dumps.push_back(std::move(text));
    }
    ocldec_b200_free(r);
    // config / instructions / abi: the sections of the kernels returned
    std::vector<KernelSection> sections;
    try {
        sections = split_kernels(listing);
    } catch (const ParseError &) {
    }
    size_t ki = 0;
    for (const KernelSection &section : sections) {
        if (opts.only_kernel && section.name != *opts.only_kernel)
            continue;
        if (ki < result.kernels.size())
            front_fields(section, opts, result.kernels[ki++]);
    }
    for (size_t i = 0; i < result.kernels.size(); ++i)
        if (!cfg_text[i].empty())
            rebuild_cfg(cfg_text[i], result.kernels[i]);
    return result;
}

} // namespace ocldec
