// TEST INFRASTRUCTURE (never shipped): DecompiledKernel::cfg from the GPU
// drop-in (integration/ocldec_b200_dropin.cpp, device step -4 export)
// against the reference pipeline's own flow graph for the same kernel:
// parse_text (+ attach_trailing_labels), build_cfg, annotate_exec,
// normalize_if_else, exactly as decompile_section builds k.cfg
// (decompiler.cpp:60-71).  Every field of every block is compared.
//   _ref/cfg_check_b200 LISTING  -> "cfg_check kernels=N compared=M mismatches=X"
#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "ocldec/decompiler.hpp"
#include "ocldec/structurizer.hpp"

using namespace ocldec;

namespace {

std::string op_str(const Operand &o) {
    std::ostringstream s;
    s << int(o.kind) << ',' << o.first << ',' << o.count << ',' << int(o.special) << ',' << o.value << ','
      << o.text;
    return s.str();
}

std::string ins_str(const Instruction &i) {
    std::ostringstream s;
    s << i.line << '|' << i.source_text << '|' << i.parse_failed << '|';
    for (const std::string &l : i.labels)
        s << l << ';';
    return s.str();
}

std::string block_str(const BasicBlock &b) {
    std::ostringstream s;
    s << "id=" << b.id << " labels=";
    for (const std::string &l : b.labels)
        s << l << ';';
    s << " n=" << b.instructions.size() << " ins=";
    for (const Instruction &i : b.instructions)
        s << ins_str(i) << '#';
    s << " supp=";
    for (bool x : b.suppressed)
        s << (x ? '1' : '0');
    s << " term=" << int(b.term.kind) << ',' << int(b.term.cc) << ',' << b.term.taken << ',' << b.term.not_taken
      << ',' << b.term.line << ',' << op_str(b.term.mask_source);
    s << " preds=";
    for (int p : b.preds)
        s << p << ',';
    s << " succs=";
    for (int p : b.succs)
        s << p << ',';
    s << " xops=";
    for (const ExecOp &x : b.exec_ops)
        s << int(x.kind) << ':' << x.index << ':' << x.mask_sgpr << ':' << op_str(x.source) << ';';
    s << " reach=" << b.reachable << " absorbed=" << b.mask_absorbed;
    return s.str();
}

} // namespace

int main(int argc, char **argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: cfg_check LISTING\n");
        return 2;
    }
    std::ifstream f(argv[1], std::ios::binary);
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string listing = ss.str();
    const DecompileResult r = decompile_listing(listing, {});
    std::vector<KernelSection> sections;
    try {
        sections = split_kernels(listing);
    } catch (const ParseError &) {
    }
    size_t compared = 0, mismatches = 0;
    for (size_t i = 0; i < sections.size() && i < r.kernels.size(); ++i) {
        const DecompiledKernel &k = r.kernels[i];
        if (k.failed)
            continue;
        DiagnosticSink sink;
        Cfg ref;
        try {
            std::vector<std::string> trailing;
            std::vector<Instruction> ins = parse_text(sections[i], sink, &trailing);
            if (!trailing.empty()) {
                Instruction end;
                end.line = ins.empty() ? sections[i].line : ins.back().line;
                end.labels = std::move(trailing);
                end.source_text = "s_endpgm";
                end.mnemonic = "s_endpgm";
                end.parts = decompose_mnemonic(end.mnemonic);
                ins.push_back(std::move(end));
            }
            ref = build_cfg(ins, sink);
            annotate_exec(ref);
            normalize_if_else(ref, sink);
        } catch (const ParseError &) {
            continue;
        }
        ++compared;
        bool bad = ref.entry != k.cfg.entry || ref.blocks.size() != k.cfg.blocks.size();
        std::string why = bad ? "block count " + std::to_string(ref.blocks.size()) + " vs " +
                                    std::to_string(k.cfg.blocks.size())
                              : "";
        for (size_t b = 0; !bad && b < ref.blocks.size(); ++b) {
            const std::string a = block_str(ref.blocks[b]), g = block_str(k.cfg.blocks[b]);
            if (a != g) {
                bad = true;
                why = "block " + std::to_string(b) + "\n  ref: " + a.substr(0, 600) + "\n  gpu: " + g.substr(0, 600);
            }
        }
        if (bad && ++mismatches <= 5)
            std::printf("MISMATCH kernel %zu (%s): %s\n", i, k.name.c_str(), why.c_str());
    }
    std::printf("cfg_check kernels=%zu compared=%zu mismatches=%zu\n", r.kernels.size(), compared, mismatches);
    return mismatches ? 1 : 0;
}
