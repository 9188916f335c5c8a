// Developer harness (NOT part of the shipped library, never used by tests or
// bench): compiles the device pipeline headers for the host so the per-kernel
// algorithm can be diffed against the oracle in this GPU-less container.
// The shipped path is paper_2107_07809_b200/csrc/ocldec_b200.cu on sm_100a.
//
//   g++ -O2 -std=c++17 -o build/devhost tools/devhost.cpp
//   build/devhost < listing.s
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "../paper_2107_07809_b200/csrc/od_kernel.cuh"
#include "../paper_2107_07809_b200/csrc/od_oracle.cuh"

using namespace od;

int main(int argc, char **argv) {
    std::string in;
    {
        char buf[1 << 16];
        size_t n;
        while ((n = fread(buf, 1, sizeof buf, stdin)) > 0)
            in.append(buf, n);
    }
    std::vector<u8> t(in.begin(), in.end());
    const u32 corpus_len = (u32)t.size();
    // P1a lines
    std::vector<u32> starts;
    {
        u32 s = 0;
        for (u32 i = 0; i < corpus_len; ++i)
            if (t[i] == '\n') {
                starts.push_back(s);
                s = i + 1;
            }
        if (s < corpus_len)
            starts.push_back(s);
    }
    u32 nl = (u32)starts.size();
    std::vector<LineRec> lines(nl);
    std::vector<u8> aux;
    for (u32 l = 0; l < nl; ++l) {
        u32 b = starts[l];
        u32 e = l + 1 < nl ? starts[l + 1] - 1 : corpus_len;
        if (l + 1 >= nl && e > b && t[e - 1] == '\n')
            --e;
        bool cx;
        u32 cut = strip_scan(t.data() + b, e - b, &cx);
        LineRec &L = lines[l];
        memset(&L, 0, sizeof L);
        if (!cx) {
            L.off = b;
            L.len = rtrim_len(t.data() + b, cut);
        } else {
            std::vector<u8> tmp(e - b + 1);
            u32 k = strip_materialize(t.data() + b, e - b, tmp.data());
            k = rtrim_len(tmp.data(), k);
            L.off = corpus_len + (u32)aux.size();
            L.len = k;
            aux.insert(aux.end(), tmp.begin(), tmp.begin() + k);
            L.complex = 1;
        }
    }
    t.insert(t.end(), aux.begin(), aux.end());
    for (u32 l = 0; l < nl; ++l)
        lines[l].kind = classify_content(t.data(), Span{lines[l].off, lines[l].len});
    // section scan
    std::vector<u32> kstart;
    int err_line = -1;
    {
        bool in_kernel = false;
        int mode = 0; // 0 preamble 1 config 2 text
        for (u32 l = 0; l < nl; ++l) {
            LineRec &L = lines[l];
            L.role = LR_NONE;
            switch (L.kind) {
            case LK_BLANK: break;
            case LK_KERNEL_NONAME: err_line = (int)l; break;
            case LK_KERNEL:
                kstart.push_back(l);
                in_kernel = true;
                mode = 0;
                break;
            case LK_DIR_CONFIG:
            case LK_DIR_TEXT:
                if (!in_kernel)
                    err_line = (int)l;
                mode = L.kind == LK_DIR_CONFIG ? 1 : 2;
                break;
            default:
                if (in_kernel)
                    L.role = mode == 2 ? LR_TEXT : LR_CONFIG;
            }
            if (err_line >= 0)
                break;
        }
    }
    if (err_line >= 0) {
        printf("E %d\nC 0\n", err_line + 1);
        return 0;
    }
    RootTable rt;
    build_root_table(&rt);
    std::vector<LineIns> lins(nl);
    std::vector<Opnd> ops;
    std::vector<Label> labs;
    for (u32 l = 0; l < nl; ++l) {
        if (lines[l].role != LR_TEXT)
            continue;
        LineIns tmp;
        decode_line(t.data(), Span{lines[l].off, lines[l].len}, &rt, &tmp, nullptr, 0, nullptr);
        u32 o0 = (u32)ops.size(), l0 = (u32)labs.size();
        ops.resize(o0 + tmp.nops + 1);
        labs.resize(l0 + tmp.nlabels + 1);
        decode_line(t.data(), Span{lines[l].off, lines[l].len}, &rt, &lins[l], ops.data() + o0,
                    tmp.nops, labs.data() + l0);
        lins[l].op_start = o0;
        lins[l].lab_start = l0;
        ops.resize(o0 + lins[l].nops);
        labs.resize(l0 + lins[l].nlabels);
    }
    std::string combined, per;
    // OD_DUMP=1|2|3: DOT dumps (DumpFlags), printed as "G/R" records
    std::vector<u8> dtext(getenv("OD_DUMP") ? (256u << 20) : 0);
    std::vector<DumpRec> drec(getenv("OD_DUMP") ? (1u << 20) : 0);
    unsigned long long dtop[2] = {0, 0};
    DumpCfg dcfg{dtext.data(), dtext.size(), drec.data(), drec.size(), dtop,
                 getenv("OD_DUMP") ? (u32)atoi(getenv("OD_DUMP")) : 0u};
    for (size_t k = 0; k < kstart.size(); ++k) {
        KIn kin;
        kin.t = t.data();
        kin.lines = lines.data();
        kin.lins = lins.data();
        kin.ops = ops.data();
        kin.labs = labs.data();
        kin.lbeg = kstart[k];
        kin.lend = k + 1 < kstart.size() ? kstart[k + 1] : nl;
        kin.line_base = 0;
        kin.fold_local_size = argc > 1 && std::string(argv[1]) == "--fold-local-size";
        kin.prof = nullptr;
        kin.ovr = nullptr;
        kin.novr = 0;
        kin.ovr_text = nullptr;
        kin.dump = dcfg.flags ? &dcfg : nullptr;
        kin.kidx = (u32)k;
        kin.names_zeroed_by_caller = 0;
        kin.collected = 0;
        KOut ko;
        const u8 *src = nullptr;
        std::vector<u8> arena;
        const KSize z = kernel_size(lines.data(), lins.data(), ops.data(), kin.lbeg, kin.lend);
        for (kin.scale = 1;; kin.scale *= 4) {
            kin.nblk_cap = kin.scale <= 1 ? z.nb : 0;
            kin.ncfg = z.ncfg;
            kin.nins = z.nins;
            kin.nlab = z.nlab;
            u64 cap = arena_budget(z, kin.scale);
            arena.assign(cap, 0);
            Bump mem{arena.data(), 0, cap, false};
            auto t0 = std::chrono::steady_clock::now();
            if (getenv("OD_TIME_FRONT")) {
                KState F;
                kstate_init(F, kin, mem);
                dk_front(F);
                fprintf(stderr, "F %zu %u %u %.1f\n", k, F.out.ninstr, F.K.nblk,
                        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
                t0 = std::chrono::steady_clock::now();
            }
            if (getenv("OD_SEMCHECK")) { // the semantic check on the host, per environment traces
                KState A;
                kstate_init(A, kin, mem);
                dk_front(A);
                if (!A.done) dk_lower(A);
                if (!A.done) dk_fold(A);
                if (!A.done) {
                    const u64 seed = strtoull(getenv("OD_SEMCHECK"), nullptr, 0);
                    for (u32 lane = 0; lane < kSemEnvs; ++lane) {
                        SemCtx c;
                        c.K = &A.K;
                        c.unsupported = false;
                        c.nan_choice = false;
                        SemRng r = sem_stream(seed, k, lane);
                        sem_env(r, lane, A.K.cfg.dims, A.K.cfg.cws, &c.env);
                        sem_args(c, r);
                        std::vector<u8> sc(kSemLaneBytes);
                        u8 *base = sc.data();
                        SemMem ma, mb;
                        ma.init(base, c.env.mem_seed);
                        mb.init(base, c.env.mem_seed);
                        u64 *vk = reinterpret_cast<u64 *>(base), *vv = vk + kSemVarCap;
                        base += kSemVarCap * 16;
                        SemMachine m{c, ma};
                        m.init();
                        m.run();
                        SemEval ev{c, mb, SemVars{vk, vv, false}, reinterpret_cast<u64 *>(base), false, false};
                        ev.run(A.hoist, A.body);
                        fprintf(stderr, "S %zu %u asm bad=%d nan=%d steps=%ld n=%u [", k, lane, m.bad, (int)c.nan_choice, m.steps, ma.count);
                        for (u32 q = 0; q < ma.n; ++q)
                            fprintf(stderr, " %llx:%x", (unsigned long long)ma.addr[q], ma.val[q]);
                        fprintf(stderr, " ] body bad=%d full=%d n=%u [", ev.bad, ev.full, mb.count);
                        for (u32 q = 0; q < mb.n; ++q)
                            fprintf(stderr, " %llx:%x", (unsigned long long)mb.addr[q], mb.val[q]);
                        fprintf(stderr, " ]\n");
                    }
                }
                mem = Bump{arena.data(), 0, cap, false};
                arena.assign(cap, 0);
            }
            ko = decompile_kernel(kin, mem, &src);
            if (getenv("OD_TIME"))
                fprintf(stderr, "T %zu %u %.1f\n", k, ko.ninstr,
                        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
            if (ko.status != KS_OOM || kin.scale > 1024)
                break;
            if (getenv("OD_USAGE") || getenv("OD_RETRY"))
                fprintf(stderr, "retry kernel %zu scale %u\n", k, kin.scale * 4);
        }
        Span nm;
        {
            Span w, rest, extra;
            split_word(t.data(), Span{lines[kin.lbeg].off, lines[kin.lbeg].len}, &w, &rest);
            split_word(t.data(), rest, &nm, &extra);
        }
        std::string name((const char *)t.data() + nm.off, nm.len);
        std::string s;
        if (ko.status == KS_OK)
            s.assign((const char *)src, ko.out_len);
        per += "K " + std::to_string(ko.status == KS_FAILED ? 1 : 0) + " " +
               std::to_string(ko.structured) + " " + std::to_string(ko.fallbacks) + " " +
               std::to_string(name.size()) + " " + std::to_string(s.size()) + "\n" + name + s;
        if (ko.status == KS_OOM)
            fprintf(stderr, "kernel %zu: OOM\n", k);
        if (getenv("OD_USAGE"))
            fprintf(stderr, "U %u %u %u %u %u %u %u %u %u %u %u %u\n", kin.lend - kin.lbeg, ko.ninstr,
                    ko.u_fixed, ko.u_nodes, ko.u_stmts, ko.u_log, ko.u_dstk, ko.u_fresh, ko.u_names,
                    ko.u_stack, ko.u_tasks, ko.out_len);
        if (!s.empty()) {
            if (!combined.empty())
                combined += "\n";
            combined += s;
        }
    }
    {
        // last record of each (kernel, step) wins (retries re-emit)
        std::map<std::pair<u32, i32>, std::string> dm;
        for (u64 i = 0; i < dtop[1]; ++i)
            dm[{drec[i].k, drec[i].step}] = std::string((const char *)dtext.data() + drec[i].off, drec[i].len);
        for (auto &e : dm) {
            if (e.first.second == -2)
                per += "M " + std::to_string(e.first.first) + " " + std::to_string(e.second.size()) + "\n";
            else if (e.first.second < 0)
                per += "G " + std::to_string(e.first.first) + " " + std::to_string(e.second.size()) + "\n";
            else
                per += "R " + std::to_string(e.first.first) + " " + std::to_string(e.first.second) + " " +
                       std::to_string(e.second.size()) + "\n";
            per += e.second;
        }
    }
    fwrite(per.data(), 1, per.size(), stdout);
    printf("C %zu\n", combined.size());
    fwrite(combined.data(), 1, combined.size(), stdout);
    return 0;
}
