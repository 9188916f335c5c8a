// ocldec-b200: the per-kernel decompilation pipeline (passes P1c-P4a), run by
// one thread per .kernel section over its own arena in HBM.
//
//   parse_config / type_from_arg_decl   asm_frontend.cpp:283-373, type_recovery.cpp:151-169
//   build_abi_map / find / find_dword   abi_model.cpp:15-55, 155-245
//   build_cfg / annotate_exec            cfg.cpp:64-226
//   normalize_if_else (+ helpers)        structurizer.cpp:407-654
//   RegionGraph / reduce / matchers      structurizer.cpp:70-403
//   instruction_use_def / live_in_sets   cfg.cpp:230-398
//   step / merge_at_join                 sym_state.cpp:56-957
//   lower_kernel / lower_goto_form       lower.cpp:17-269
//   hoist_fresh_decls / decompile_section decompiler.cpp:37-101
//   emit_kernel / emit_statement         codegen.cpp:358-467
//
// Every data structure is a fixed-width array in the arena; recursion in the
// reference (lower_region, render, expr_equal, fold_expr) is replaced by
// explicit stacks, and RegisterFile snapshots by an undo log.
#pragma once

#include "od_parse.cuh"
#include "od_render.cuh"

namespace od {

// ---------------------------------------------------------------- arena
struct Bump {
    u8 *base;
    u64 top, cap;
    bool oom;
    template <class T> OD_INL T *get(u64 n) {
        u64 a = (top + 15) & ~15ull;
        u64 bytes = n * sizeof(T);
        if (a + bytes > cap) {
            oom = true;
            return nullptr;
        }
        top = a + bytes;
        return (T *)(base + a);
    }
};

enum KStatus : u32 { KS_OK = 0, KS_FAILED = 1, KS_OOM = 2, KS_SPLIT_ERROR = 3, KS_SKIP = 4, KS_STAGE_FULL = 5 };

// One ABI override (DecompileOptions::abi_overrides, abi_model.hpp:64-68),
// resolved on the host except for the per-kernel argument lookup.
enum OvrKind : u8 { OV_ARG = 0, OV_BUILTIN, OV_BAD_TARGET, OV_BAD_DIM };
struct AbiOvr {
    u32 offset;
    u8 dwords, kind, fn, dim;
    u32 name_off, name_len; // OV_ARG: argument name in the override text
};

// DOT dumps (DecompileOptions::dump_cfg / dump_regions, decompiler.hpp:33-34):
// text appended to a run-wide pool, one record per dump.
enum DumpFlags : u32 { DUMP_CFG = 1, DUMP_REGIONS = 2, DUMP_MERGES = 4, DUMP_BODY = 8 };
struct DumpRec {
    u32 k;      // kernel (chunk result index)
    i32 step;   // -1: cfg_dot, -2: ReduceResult merges/root/residue text, else dumps[step]
    u64 off, len;
};
struct DumpCfg {
    u8 *text;
    u64 cap;
    DumpRec *rec;
    u64 rcap;
    unsigned long long *top; // [0] text bytes, [1] records (may pass the caps: pool full)
    u32 flags;
};

// Inputs for one kernel section.
struct KIn {
    const u8 *t;          // listing bytes (+ aux area)
    const LineRec *lines; // chunk line records
    const LineIns *lins;  // decoded text lines
    const Opnd *ops;      // operand pool
    const Label *labs;    // label pool
    u32 lbeg, lend;       // [.kernel line, next .kernel line) (chunk-relative)
    u32 line_base;        // global 1-based line number of chunk line 0 is line_base + 1
    u32 fold_local_size;
    u32 scale;            // pool capacity multiplier (retries)
    u32 nblk_cap;         // block capacity (KSize::nb; 0 = one per instruction)
    u32 ncfg, nins, nlab; // KSize counts of the section (config lines, instructions, labels)
    const AbiOvr *ovr;    // ABI overrides (novr), applied by build_abi
    u32 novr;
    const u8 *ovr_text;
    const DumpCfg *dump;  // DOT dumps (null: none)
    u32 names_zeroed_by_caller; // k_front's warp zeroes the name set and writes the
                                // default register slots after dk_front
    u32 collected;        // k_front's warp filled the instruction / label arrays:
    u32 c_nins, c_nkl, c_pend_b, c_last_line, c_any_failed; // ... with this tail
    u32 kidx;             // chunk result index (dump records)
    u64 *prof;            // optional per-phase cycle counters
};

struct KOut {
    u32 status;
    u32 structured;
    u32 fallbacks;
    u32 ninstr;      // parse_text instructions (synthetic s_endpgm excluded)
    u32 out_len;     // bytes of source written to the writer
    // high-water marks (arena budgeting)
    u32 u_fixed;     // bytes before the dynamic pools
    u32 u_nodes, u_stmts, u_log, u_dstk, u_fresh, u_names, u_stack, u_tasks, u_regions;
};

// -------------------------------------------------------- instructions
enum ExecKind : u8 { XK_NONE = 0, XK_SAVE, XK_INVERT, XK_RESTORE };

struct Ins {
    u16 root;
    u8 prefix;
    u8 rflags;
    u16 sfx[2];
    u16 nops;
    u8 flags;
    u8 xkind;      // static exec-op classification (annotate_exec), suppression aside
    u32 xmask;     // saved-mask first SGPR
    u32 op_start;  // operand pool index
    u32 line;      // 1-based listing line
    Span src;      // source_text
    u32 lab_b, lab_n; // labels (indices into the kernel label list)
};

enum TermKind : u8 { T_FALL = 0, T_UNCOND, T_COND, T_END };
enum CondCode : u8 { C_SCC0 = 0, C_SCC1, C_VCCZ, C_VCCNZ, C_EXECZ, C_EXECNZ, C_MASKED };

struct Term {
    u8 kind, cc;
    u16 pad;
    i32 taken, not_taken;
    Opnd mask_source;
    u32 line;
};

OD_INL void term_default(Term &t) {
    t.kind = T_FALL;
    t.cc = C_SCC0;
    t.pad = 0;
    t.taken = -1;
    t.not_taken = -1;
    t.mask_source.kind = OK_ANNOT; // Operand{} default: Annotation, count 1
    t.mask_source.special = SP_EXEC;
    t.mask_source.pad = 0;
    t.mask_source.count = 1;
    t.mask_source.value = 0;
    t.line = 0;
}

struct XOp {
    u8 kind;   // ExecKind (0 = none)
    u32 index; // within block
    u32 mask;
    u32 ins;   // global instruction index
};

struct Block {
    u32 ib, ie;       // instruction range
    u32 lab_b, lab_n; // labels of the leader (split-off blocks: none)
    Term term;
    i32 succ[2];
    u8 nsucc;
    u8 reachable;
    u8 absorbed;
    u8 pad;
    XOp xfront, xback; // annotate_exec: first / last exec op
};

// ------------------------------------------------------------ regions
enum RKind : u8 { RK_BLOCK = 0, RK_LINEAR, RK_IFTHEN, RK_IFELSE };

struct Region {
    u8 kind;
    u8 join_absorbed;
    u8 cc;
    u8 then_is_taken;
    i32 block_id;
    i32 join_block;
    u8 has_term; // cond came from a terminator (make_cond(term))
    u8 pad[3];
    Opnd mask_source;
    u32 ch_b, ch_n; // children (region ids) in the child pool
    i32 succ[2];
    u32 nsucc;
};

// -------------------------------------------------------------- lowering
enum Integrity : u8 { IN_ENTIRE = 0, IN_LOW, IN_HIGH };

struct Slot {
    u32 version;
    u32 expr;
    DT type;
    u8 integ;
    u8 pad[3];
};

// An undo record is the slot's old value with its slot id in the pad bytes:
// one 16-byte load and one 16-byte store per record.
struct UndoRec {
    u32 version;
    u32 expr;
    DT type;
    u32 integ_phys; // integ | phys << 8
    OD_INL u32 phys() const { return integ_phys >> 8; }
};
static_assert(sizeof(UndoRec) == 16 && sizeof(Slot) == 16, "undo records are Slot-shaped");

struct Pending {
    u32 valid;
    u32 lo_vgpr;
    u32 lo_version;
    u32 base64;
    u32 addend;
};

enum SKind : u8 { SK_ASSIGN = 0, SK_DECL, SK_STORE, SK_RAW, SK_IF, SK_LABEL, SK_GOTO };

struct Stmt {
    u8 kind;
    u8 pad;
    u16 cls;   // Assign/Decl: var name class
    u32 next;  // list link (0 = end)
    u32 a;     // Assign/Decl: var number; Store: addr; If/Goto: cond; Raw: text off; Label/Goto: block
    u32 b;     // Assign/Decl/Store: value; If: then head; Raw: text len
    u32 c;     // Decl: type; Store: elem type; If: else head; Goto: target block
    u32 d;     // Raw/Goto/Label spare
};

struct SList {
    u32 head, tail;
};

struct Fresh {
    u32 cls, num;
    DT type;
};

// One lowering frame (lower_region made iterative).
struct Frame {
    u32 region;
    u32 phase;
    u32 out;       // SList index receiving statements
    u32 then_l;    // SList index (If)
    u32 else_l;    // SList index (If)
    u32 cond;      // If condition
    u32 log_p0;    // undo log position at the split
    u32 dstk_p0;   // delta stack position
    u32 then_d, then_n; // then-arm delta (slot records in delta stack)
    u32 child;     // Linear: next child
    Pending pend;  // pending add at the split
};

// Name set (std::set<std::string> name_pool / hoist dedup) as open addressing
// over (class, number) keys.
struct NameSet {
    u64 *keys; // 0 = empty; key = (cls+1)<<32 | num
    u32 cap, count;
    bool oom;
    OD_INL bool insert(u32 cls, u32 num) {
        u64 k = ((u64)(cls + 1) << 32) | num;
        if (count * 2 >= cap) {
            oom = true;
            return true;
        }
        u64 h = k * 0x9E3779B97F4A7C15ull;
        u32 i = (u32)(h >> 32) & (cap - 1);
        while (keys[i]) {
            if (keys[i] == k)
                return false;
            i = (i + 1) & (cap - 1);
        }
        keys[i] = k;
        ++count;
        return true;
    }
    // hoist_fresh_decls' dedupe over names already in the set: true the
    // first time (cls, num) is marked (bit 63 of its key).
    OD_INL bool mark(u32 cls, u32 num) {
        const u64 k = ((u64)(cls + 1) << 32) | num;
        u64 h = k * 0x9E3779B97F4A7C15ull;
        u32 i = (u32)(h >> 32) & (cap - 1);
        while (keys[i]) {
            if ((keys[i] & ~(1ull << 63)) == k) {
                if (keys[i] >> 63)
                    return false;
                keys[i] |= 1ull << 63;
                return true;
            }
            i = (i + 1) & (cap - 1);
        }
        return true; // not recorded (cannot happen: bind_fresh inserts every fresh name)
    }
};

struct AbiEntry {
    u32 offset;
    u8 dwords;
    u8 has_builtin;
    u8 fn;
    u8 dim;
    i32 arg_index;
    DT type;
};

// ------------------------------------------------------------ diagnostics
// DiagnosticSink entries (diagnostics.hpp:20-57) of one kernel, in emission
// order; the host renders the message text (ocldec_b200.cu render_diag) from
// the code and the listing spans.  Catalogue: SURVEY A.4.
enum DiagCode : u16 {
    DG_DIMS = 1,        // error   "bad .dims axes '<a>'"                        asm_frontend.cpp:307
    DG_CWS_COUNT,       // error   "cws expects 1 to 3 sizes"                    :313
    DG_CWS_VALUE,       // error   "bad cws value '<a>'"                         :319
    DG_SGPRS,           // error   "bad sgprsnum value"                          :329
    DG_VGPRS,           // error   "bad vgprsnum value"                          :335
    DG_ARG_FIELDS,      // error   "arg directive needs name, type string and type" :341
    DG_ARG_TYPE,        // warning "unrecognized argument type '<a>' for '<b>'"  :365
    DG_OPERAND,         // warning "<operand ParseError c, token a>; keeping the line as inline assembly" :159-183, 478
    DG_BR_NOLABEL,      // error   "branch without a label operand"              cfg.cpp:105
    DG_BR_UNDEF,        // error   "branch to undefined label '<a>'"             cfg.cpp:108
    DG_CBR_UNSUP,       // error   "unsupported conditional branch s_<root of a>" cfg.cpp:127
    DG_CBR_END,         // error   "conditional branch at end of kernel"         cfg.cpp:130
    DG_UNREACHABLE,     // note    "unreachable code"                            cfg.cpp:154
    DG_MASK_MULTI,      // warning "exec mask saved in s[c:c+1] has multiple join points" structurizer.cpp:533
    DG_MASK_NONE,       // warning "exec mask save without inversion or restore" :539
    DG_MASK_EXECZ_INV,  // warning "execz branch does not meet the mask inversion" :555
    DG_MASK_NO_RESTORE, // warning "mask inversion without a matching restore"   :575
    DG_MASK_EXECZ_RST,  // warning "execz branch does not meet the mask restore" :586
    DG_SLOAD_UNMAPPED,  // warning "scalar load from unmapped settings offset"   sym_state.cpp:394
    DG_ADDC,            // warning "v_addc_u32 outside the 64-bit add idiom; carry treated as zero" :688
    DG_GOTO,            // warning "control flow not fully structured; emitting labeled blocks" lower.cpp:189
    DG_EXEC_BRANCH,     // warning "exec-dependent branch kept as inline asm"    lower.cpp:225
    DG_OVR_ARG,         // error   "override names unknown argument '<tail c>'" abi_model.cpp:209
    DG_OVR_TARGET,      // error   "unknown override target '<target c>'"       :227
    DG_OVR_DIM,         // error   "override dimension must be 0..2"            :234
};

struct Diag {
    u32 line;
    u16 code;
    u16 c;    // small argument (operand error kind, mask SGPR)
    u32 a_off, a_len, b_off, b_len; // listing spans
};

// The whole per-kernel working set.
struct KCtx {
    const KIn *in;
    Bump *mem;
    bool failed;  // ParseError
    bool oom;

    KConfig cfg;
    Span *arg_sname;
    AbiEntry *abi;
    u32 nabi;

    Ins *ins;
    u32 nins, nins_real;
    u32 *kl;     // kernel label list (global label pool indices)
    u32 nkl;
    u8 *supp;    // suppressed flag per instruction

    Block *blk;
    u32 nblk, blk_cap;
    u32 *stamp;  // per-block traversal stamps
    u32 *sx;     // compact successor pairs (kNoSucc = none), kept in sync with Block::succ
    u32 *rbits;  // reachability bitmap (BasicBlock::reachable)
    u32 stamp_gen;
    u32 *work;   // block work stack
    bool acyclic; // the flow graph has no cycle (set by normalize)

    // label map
    u32 *lmap;   // label-list index + 1 (0 empty)
    u32 lmap_cap;

    // regions
    Region *rg;  // 1-based
    u32 nrg, rg_cap;
    u32 *child;  // child pool
    u32 nchild, child_cap;
    u32 *live;   // live region list
    u32 nlive;
    u32 *pred_n, *pred_x; // per region: live predecessor count and xor of their ids
    u32 *phead;           // per region: predecessor edge list (edge pool index, 0 = end)
    u32 *enext, *efrom;   // edge pool
    u32 etop, efree, ecap;
    u32 *rstamp; // region stamps
    u32 rstamp_gen;
    u32 *dmark;  // dirty-neighbourhood stamps (region_replace)
    u32 dmark_gen;
    u32 *rank;   // region -> position in the reverse post-order (kNoRank: none)
    u32 *at;     // position -> region (0: removed)
    u64 *cand;   // positions still to try: present and not known to fail
    u32 ncand_w;
    u32 *rpo;    // rpo output
    u32 *dfs;    // dfs stack (pairs)
    i32 entry_r;
    u32 root_r;
    bool reduced;
    u32 nif;      // IfThen / IfElse merges (joins need liveness)
    u32 nmerge;   // merges so far (dump step numbers)
    bool dump_full; // the dump pool overflowed
    u32 exp_lists[2]; // body export (DUMP_BODY): the hoisted decls and the body statement lists
    u32 exp_pass;     // body export: printing pass (its export ids are tagged per pass)

    // liveness
    u32 *live_in; // [nblk][12]

    // expressions / lowering
    EArena E;
    FoldScratch fs;
    U32Stack eqst;
    Slot *regs;   // kPhysSlots
    u32 dirty[kLiveWords]; // slots written since the last initial_register_state
    UndoRec *log;
    u32 nlog, log_cap, log_hw;
    u32 log_depth; // > 0 while inside an if arm
    Pending pend;
    Stmt *st;
    u32 nst, st_cap;
    SList *lists;
    u32 nlists, lists_cap;
    Fresh *fresh;
    u32 nfresh, fresh_cap;
    NameSet pool;
    u32 fallbacks;
    Frame *frames;
    u32 nframes, frames_cap;
    Slot *dstk;   // delta stack (values)
    u32 *dstk_id; // delta stack (phys ids)
    u32 ndstk, dstk_cap, dstk_hw;
    u32 stack_hw;

    // rendering
    RenderCtx rc;

    // diagnostics
    Diag *dg;
    u32 ndg, dg_cap;
};

OD_NOINL void diag(KCtx &K, u16 code, u32 line, u16 c = 0, Span a = Span{0, 0}, Span b = Span{0, 0}) {
#ifdef OD_DIAG_OFF
    return;
#endif
    if (!K.dg)
        return;
    if (K.ndg >= K.dg_cap) {
        K.oom = true; // retried with a larger arena
        return;
    }
    Diag &d = K.dg[K.ndg++];
    d.line = line;
    d.code = code;
    d.c = c;
    d.a_off = a.off;
    d.a_len = a.len;
    d.b_off = b.off;
    d.b_len = b.len;
}

OD_INL const Opnd &op_at(const KCtx &K, const Ins &I, u32 k) { return K.in->ops[I.op_start + k]; }
OD_INL DT suffix_type0(const Ins &I, DT fb) { return I.sfx[0] ? dt_from_suffix(I.sfx[0]) : fb; }

// ============================================================ config
// split_fields (asm_frontend.cpp:80-107) returning up to maxf field spans;
// the return value is the field count after dropping trailing empties.
OD_INL u32 split_fields_spans(const u8 *t, Span s, Span *f, u32 maxf) {
    int depth = 0;
    bool inq = false;
    u32 nf = 0, last_nonempty = 0;
    u32 start = s.off, end = s.off + s.len;
    for (u32 i = s.off; i <= end; ++i) {
        bool cut = false;
        if (i == end)
            cut = true;
        else {
            u8 c = t[i];
            if (c == '"')
                inq = !inq;
            if (!inq) {
                if (c == '[' || c == '(')
                    ++depth;
                else if (c == ']' || c == ')')
                    --depth;
                else if (c == ',' && depth == 0)
                    cut = true;
            }
        }
        if (!cut)
            continue;
        u32 b = start, e = i;
        while (b < e && c_space(t[b]))
            ++b;
        while (e > b && c_space(t[e - 1]))
            --e;
        if (i == end && e == b) {
            // final empty field is never pushed
        } else {
            if (nf < maxf) {
                f[nf].off = b;
                f[nf].len = e - b;
            }
            ++nf;
            if (e > b)
                last_nonempty = nf;
        }
        start = i + 1;
    }
    return last_nonempty;
}

// type_from_arg_decl  type_recovery.cpp:151-169
OD_INL DT type_from_arg_decl(const u8 *t, Span m, u32 space) {
    u32 n = m.len;
    u32 depth = 0;
    while (n > 0 && t[m.off + n - 1] == '*') {
        --n;
        while (n > 0 && t[m.off + n - 1] == ' ')
            --n;
        ++depth;
    }
    Span nm = {m.off, n};
    DT ty = DT_UNKNOWN;
    if (span_eq(t, nm, "char")) ty = dt_make(B_SIGNED, 8);
    else if (span_eq(t, nm, "uchar")) ty = dt_make(B_UNSIGNED, 8);
    else if (span_eq(t, nm, "short")) ty = dt_make(B_SIGNED, 16);
    else if (span_eq(t, nm, "ushort")) ty = dt_make(B_UNSIGNED, 16);
    else if (span_eq(t, nm, "int")) ty = dt_make(B_SIGNED, 32);
    else if (span_eq(t, nm, "uint")) ty = dt_make(B_UNSIGNED, 32);
    else if (span_eq(t, nm, "long")) ty = dt_make(B_SIGNED, 64);
    else if (span_eq(t, nm, "ulong")) ty = dt_make(B_UNSIGNED, 64);
    else if (span_eq(t, nm, "size_t")) ty = dt_make(B_UNSIGNED, 64);
    else if (span_eq(t, nm, "float")) ty = dt_make(B_FLOAT, 32);
    else if (span_eq(t, nm, "double")) ty = dt_make(B_FLOAT, 64);
    else if (span_eq(t, nm, "void")) ty = dt_make(B_VOID, 0);
    else if (span_eq(t, nm, "structure")) ty = dt_make(B_UNSIGNED, 8);
    for (u32 i = 0; i < depth; ++i)
        ty = dt_pointer_to(ty, space);
    return ty;
}

OD_INL bool sanitized_eq(const u8 *t, Span a, Span b) {
    if (a.len != b.len)
        return false;
    for (u32 i = 0; i < a.len; ++i) {
        u8 x = t[a.off + i], y = t[b.off + i];
        if (x == '.')
            x = '_';
        if (y == '.')
            y = '_';
        if (x != y)
            return false;
    }
    return true;
}

// parse_config  asm_frontend.cpp:283-373 (diagnostics are not materialized)
// One config line of parse_config (asm_frontend.cpp:287-371), out of line:
// the scan over the section's lines stays a tight loop.
OD_NOINL void config_line(KCtx &K, u32 l) {
    const KIn &in = *K.in;
    const u8 *t = in.t;
    KConfig &c = K.cfg;
    do {
        const LineRec &L = in.lines[l];
        if (L.role != LR_CONFIG)
            break;
        Span w, rest;
        split_word(t, Span{L.off, L.len}, &w, &rest);
        Span key = w;
        if (key.len && t[key.off] == '.') {
            key.off++;
            key.len--;
        }
        if (span_eq(t, key, "dims")) {
            Span axes, extra;
            split_word(t, rest, &axes, &extra);
            u32 dims = 0;
            bool ok = axes.len > 0;
            for (u32 i = 0; i < axes.len; ++i) {
                u8 ch = t[axes.off + i];
                if (ch >= 'A' && ch <= 'Z')
                    ch = ch - 'A' + 'a';
                if (ch == 'x')
                    dims = dims > 1 ? dims : 1;
                else if (ch == 'y')
                    dims = dims > 2 ? dims : 2;
                else if (ch == 'z')
                    dims = 3;
                else
                    ok = false;
            }
            if (ok)
                c.dims = dims;
            else
                diag(K, DG_DIMS, in.line_base + l + 1, 0, axes);
        } else if (span_eq(t, key, "cws") || span_eq(t, key, "reqd_work_group_size")) {
            Span f[4];
            u32 nf = split_fields_spans(t, rest, f, 4);
            if (nf == 0 || nf > 3) {
                diag(K, DG_CWS_COUNT, in.line_base + l + 1);
                break;
            }
            for (u32 i = 0; i < nf; ++i) {
                i64 v;
                if (!parse_int(t + f[i].off, f[i].len, &v) || v <= 0) {
                    diag(K, DG_CWS_VALUE, in.line_base + l + 1, 0, f[i]);
                    break;
                }
                c.cws[i] = (u32)v;
            }
        } else if (span_eq(t, key, "sgprsnum") || span_eq(t, key, "sgprnum") || span_eq(t, key, "vgprsnum") ||
                   span_eq(t, key, "vgprnum")) {
            // the counts are not used downstream; only a bad value is reported
            Span v = trim_span(t, rest);
            i64 x;
            if (!(parse_int(t + v.off, v.len, &x) && x >= 0))
                diag(K, t[key.off] == 's' ? DG_SGPRS : DG_VGPRS, in.line_base + l + 1);
        } else if (span_eq(t, key, "useargs")) {
            c.useargs = 1;
        } else if (span_eq(t, key, "arg")) {
            Span f[4];
            u32 nf = split_fields_spans(t, rest, f, 4);
            if (nf < 3) {
                diag(K, DG_ARG_FIELDS, in.line_base + l + 1);
                break;
            }
            KArg &a = c.args[c.nargs];
            a.name = f[0];
            u32 space = AS_NONE;
            Span mt = f[2];
            if (nf > 3) {
                if (span_eq(t, f[3], "global"))
                    space = AS_GLOBAL;
                else if (span_eq(t, f[3], "local"))
                    space = AS_LOCAL;
                else if (span_eq(t, f[3], "constant"))
                    space = AS_CONSTANT;
            } else {
                for (u32 i = 0; i < mt.len; ++i)
                    if (t[mt.off + i] == '*') {
                        space = AS_GLOBAL;
                        break;
                    }
            }
            a.type = type_from_arg_decl(t, mt, space);
            a.implicit = (a.name.len >= 2 && t[a.name.off] == '_' && t[a.name.off + 1] == '.');
            if (dt_base(a.type) == B_UNKNOWN)
                diag(K, DG_ARG_TYPE, in.line_base + l + 1, 0, mt, a.name);
            // canonical sanitized-name id
            u32 id = c.nargs;
            for (u32 j = 0; j < c.nargs; ++j)
                if (sanitized_eq(t, c.args[j].name, a.name)) {
                    id = c.args[j].name_id;
                    break;
                }
            a.name_id = id;
            K.arg_sname[c.nargs] = a.name;
            c.nargs++;
        }
    } while (false);
}

OD_NOINL bool parse_config(KCtx &K) {
    const KIn &in = *K.in;
    const u8 *t = in.t;
    KConfig &c = K.cfg;
    c.dims = 1;
    c.cws[0] = c.cws[1] = c.cws[2] = 1;
    c.useargs = 0;
    c.nargs = 0;
    c.fold_local_size = in.fold_local_size;
    // name: second word of the .kernel line
    {
        const LineRec &L = in.lines[in.lbeg];
        Span w, rest, nm, extra;
        split_word(t, Span{L.off, L.len}, &w, &rest);
        split_word(t, rest, &nm, &extra);
        c.name = nm;
    }
    const u32 ncfg = in.ncfg;
    c.args = K.mem->get<KArg>(ncfg + 1);
    K.arg_sname = K.mem->get<Span>(ncfg + 1);
    if (!c.args || !K.arg_sname)
        return false;
    const LineRec *__restrict__ lines = in.lines;
    for (u32 l = in.lbeg + 1, e = in.lend; l < e; ++l)
        if (lines[l].role == LR_CONFIG)
            config_line(K, l);
    return true;
}

// ============================================================ ABI map
OD_INL void abi_add(KCtx &K, const AbiEntry &e) {
    u32 w = 0;
    for (u32 i = 0; i < K.nabi; ++i)
        if (!(K.abi[i].offset == e.offset && K.abi[i].dwords == e.dwords))
            K.abi[w++] = K.abi[i];
    K.nabi = w;
    K.abi[K.nabi++] = e;
}

// build_abi_map  abi_model.cpp:155-245; overrides resolved on the host by
// parse_overrides (parse_abi_overrides abi_model.cpp:109-153)
OD_NOINL bool build_abi(KCtx &K) {
    K.abi = K.mem->get<AbiEntry>(8 + K.cfg.nargs + K.in->novr);
    if (!K.abi)
        return false;
    K.nabi = 0;
    if (K.cfg.useargs) {
        const u32 off[7] = {0x0, 0x8, 0x10, 0xc, 0x10, 0x14, 0x20010};
        const u8 dw[7] = {2, 2, 2, 1, 1, 1, 1};
        const u8 fn[7] = {F_GLOBAL_OFFSET, F_GLOBAL_OFFSET, F_GLOBAL_OFFSET, F_GLOBAL_SIZE,
                          F_GLOBAL_SIZE, F_GLOBAL_SIZE, F_WORK_DIM};
        const u8 dm[7] = {0, 1, 2, 0, 1, 2, 0};
        for (int i = 0; i < 7; ++i) {
            AbiEntry e;
            e.offset = off[i];
            e.dwords = dw[i];
            e.has_builtin = 1;
            e.fn = fn[i];
            e.dim = dm[i];
            e.arg_index = -1;
            e.type = fn[i] == F_GLOBAL_OFFSET ? DT_U64 : DT_U32;
            abi_add(K, e);
        }
    }
    u32 offset = 0;
    const u8 *t = K.in->t;
    for (u32 i = 0; i < K.cfg.nargs; ++i) {
        const KArg &a = K.cfg.args[i];
        u32 sz = dt_byte_size(a.type);
        if (sz < 4)
            sz = 4;
        offset = (offset + sz - 1) & ~(sz - 1);
        AbiEntry e;
        e.offset = offset;
        e.dwords = (u8)(sz / 4 > 1 ? sz / 4 : 1);
        e.has_builtin = 0;
        e.fn = 0;
        e.dim = 0;
        e.arg_index = (i32)i;
        e.type = a.type;
        if (a.implicit && a.name.len == 17 && starts_with(t + a.name.off, a.name.len, "_.global_offset_")) {
            u8 last = t[a.name.off + 16];
            if (last >= '0' && last <= '2') {
                e.has_builtin = 1;
                e.fn = F_GLOBAL_OFFSET;
                e.dim = last - '0';
            }
        }
        if (e.dwords <= 2)
            abi_add(K, e);
        offset += sz;
    }
    // overrides last (abi_model.cpp:196-243); AbiMap::add replaces exact matches
    const KIn &in = *K.in;
    for (u32 q = 0; q < in.novr; ++q) {
        const AbiOvr &o = in.ovr[q];
        AbiEntry e;
        e.offset = o.offset;
        e.dwords = o.dwords;
        e.has_builtin = 0;
        e.fn = 0;
        e.dim = 0;
        e.arg_index = -1;
        e.type = DT_UNKNOWN;
        if (o.kind == OV_ARG) {
            i32 hit = -1;
            for (u32 i = 0; i < K.cfg.nargs && hit < 0; ++i) {
                const Span nm = K.cfg.args[i].name;
                if (nm.len == o.name_len && bytes_eq(t + nm.off, in.ovr_text + o.name_off, nm.len))
                    hit = (i32)i;
            }
            if (hit < 0) {
                diag(K, DG_OVR_ARG, 0, (u16)q);
                continue;
            }
            e.arg_index = hit;
            e.type = K.cfg.args[hit].type;
        } else if (o.kind == OV_BUILTIN) {
            e.has_builtin = 1;
            e.fn = o.fn;
            e.dim = o.dim;
            e.type = o.fn == F_GLOBAL_OFFSET ? DT_U64 : DT_U32;
        } else {
            diag(K, o.kind == OV_BAD_TARGET ? DG_OVR_TARGET : DG_OVR_DIM, 0, (u16)q);
            continue;
        }
        abi_add(K, e);
    }
    return true;
}

OD_INL const AbiEntry *abi_find(const KCtx &K, u32 offset, u32 dwords) {
    for (u32 i = 0; i < K.nabi; ++i)
        if (K.abi[i].offset == offset && K.abi[i].dwords == dwords)
            return &K.abi[i];
    return nullptr;
}

OD_INL const AbiEntry *abi_find_dword(const KCtx &K, u32 offset, bool *second) {
    *second = false;
    for (u32 i = 0; i < K.nabi; ++i)
        if (K.abi[i].offset == offset && K.abi[i].dwords == 1)
            return &K.abi[i];
    for (u32 i = 0; i < K.nabi; ++i)
        if (K.abi[i].offset == offset && K.abi[i].dwords == 2)
            return &K.abi[i];
    for (u32 i = 0; i < K.nabi; ++i)
        if (K.abi[i].dwords == 2 && K.abi[i].offset + 4 == offset) {
            *second = true;
            return &K.abi[i];
        }
    return nullptr;
}

// match_settings_load  builtin_detector.cpp:70-84
OD_INL u32 match_settings_load(KCtx &K, u32 offset, u32 dwords) {
    const AbiEntry *e = abi_find(K, offset, dwords);
    if (!e)
        return 0;
    if (e->has_builtin)
        return K.E.builtin(e->fn, e->dim, dwords == 2 ? DT_U64 : DT_U32);
    if (e->arg_index >= 0 && (u32)e->arg_index < K.cfg.nargs)
        return K.E.arg(K.cfg.args[e->arg_index].name_id, e->type);
    return 0;
}

// ====================================================== instructions
// annotate_exec's per-instruction classification (cfg.cpp:158-226) from the
// decoded fields; *mask gets the saved-mask SGPR.
OD_INL u32 exec_kind_of(u32 root, u32 prefix, u32 flags, u32 n, const Opnd *o, u32 *mask) {
    *mask = 0;
    if ((flags & IF_PARSE_FAILED) || prefix != PX_S)
        return XK_NONE;
    if (root == R_AND_SAVEEXEC && n >= 2 && o[0].kind == OK_SREG && o[0].count == 2) {
        *mask = o[0].r.a;
        return XK_SAVE;
    }
    bool dst_exec = n >= 1 && op_is_special(o[0], SP_EXEC);
    if (!dst_exec)
        return XK_NONE;
    if (root == R_MOV && n >= 2 && op_is_sreg_pair(o[1])) {
        *mask = o[1].r.a;
        return XK_RESTORE;
    }
    if (root == R_OR && n >= 3) {
        if (op_is_special(o[1], SP_EXEC) && op_is_sreg_pair(o[2])) {
            *mask = o[2].r.a;
            return XK_RESTORE;
        }
        if (op_is_special(o[2], SP_EXEC) && op_is_sreg_pair(o[1])) {
            *mask = o[1].r.a;
            return XK_RESTORE;
        }
    }
    if ((root == R_ANDN2 || root == R_XOR) && n >= 3) {
        if (op_is_sreg_pair(o[1]) && op_is_special(o[2], SP_EXEC)) {
            *mask = o[1].r.a;
            return XK_INVERT;
        }
        if (op_is_sreg_pair(o[2]) && op_is_special(o[1], SP_EXEC)) {
            *mask = o[2].r.a;
            return XK_INVERT;
        }
    }
    return XK_NONE;
}

OD_NOINL void classify_exec(const KCtx &K, Ins &I) {
    u32 m;
    I.xkind = (u8)exec_kind_of(I.root, I.prefix, I.flags, I.nops, K.in->ops + I.op_start, &m);
    I.xmask = m;
}

// Per-kernel sizes that bound every allocation decompile_kernel makes
// (kernel_budget): counted from the decoded lines before the wave layout.
struct KSize {
    u32 n;    // lines of the section (incl. the .kernel line)
    u32 ncfg; // config lines
    u32 nins; // instruction lines
    u32 nlab; // labels
    u32 nb;   // blocks: leaders (first, labelled, after a branch/endpgm) + exec-op splits + the synthetic end
    u32 novr; // ABI overrides of the run
};

OD_INL KSize kernel_size(const LineRec *lines, const LineIns *lins, const Opnd *ops, u32 lbeg, u32 lend) {
    KSize z;
    z.n = lend - lbeg;
    z.ncfg = z.nins = z.nlab = 0;
    u32 labelled = 0, enders = 0, xops = 0;
    for (u32 l = lbeg + 1; l < lend; ++l) {
        const u8 role = lines[l].role;
        if (role == LR_CONFIG) {
            ++z.ncfg;
            continue;
        }
        if (role != LR_TEXT)
            continue;
        const LineIns &L = lins[l];
        z.nlab += L.nlabels;
        labelled += L.nlabels ? 1 : 0;
        if (!(L.flags & IF_HAS_INS))
            continue;
        ++z.nins;
        if (L.prefix == PX_S && (L.root == R_BRANCH || L.root == R_ENDPGM || (L.rflags & RF_CBRANCH)))
            ++enders;
        u32 m;
        if (L.prefix == PX_S && exec_kind_of(L.root, L.prefix, L.flags, L.nops, ops + L.op_start, &m) != XK_NONE)
            ++xops;
    }
    z.nb = 3 + labelled + enders + xops;
    z.novr = 0;
    return z;
}

// parse_instruction's downgraded ParseErrors (asm_frontend.cpp:478), in
// instruction order; out of the collection loop (rare).
OD_NOINL void note_parse_failures(KCtx &K) {
    for (u32 i = 0; i < K.nins; ++i) {
        const Ins &I = K.ins[i];
        if (!(I.flags & IF_PARSE_FAILED))
            continue;
        const Opnd &e = K.in->ops[I.op_start];
        diag(K, DG_OPERAND, I.line, e.special, Span{e.r.a, e.r.b});
    }
}

// parse_text + attach_trailing_labels (asm_frontend.cpp:486-521,
// decompiler.cpp:20-31), in three parts: the instruction and label arrays are
// the kernel's first arena allocations (k_front's warp fills them at these
// fixed addresses before the kernel's lane starts), the fill (here: the
// serial form), and the common tail.
OD_INL u64 collect_bytes(u32 nins, u32 nlab, u64 *kl_off) {
    const u64 ib = (u64)(nins + 2) * sizeof(Ins); // + synthetic s_endpgm
    *kl_off = (ib + 15) & ~15ull;
    return *kl_off + (u64)(nlab + 1) * 4;
}

OD_NOINL bool collect_alloc(KCtx &K) {
    K.ins = K.mem->get<Ins>(K.in->nins + 2);
    K.kl = K.mem->get<u32>(K.in->nlab + 1);
    return K.ins && K.kl;
}

// One text line of the collection: its labels, then its instruction (if any)
// with the labels pending since the previous instruction.
OD_INL void collect_ins(Ins &I, const LineIns &L, const Opnd *ops, u32 line, u32 lab_b, u32 lab_n) {
    I.root = L.root;
    I.prefix = L.prefix;
    I.rflags = L.rflags;
    I.sfx[0] = L.sfx[0];
    I.sfx[1] = L.sfx[1];
    I.nops = L.nops;
    I.flags = L.flags;
    I.op_start = L.op_start;
    I.line = line;
    I.src.off = L.src_off;
    I.src.len = L.src_len;
    I.lab_b = lab_b;
    I.lab_n = lab_n;
    u32 m = 0;
    I.xkind = L.prefix == PX_S ? (u8)exec_kind_of(L.root, L.prefix, L.flags, L.nops, ops + L.op_start, &m)
                               : (u8)XK_NONE;
    I.xmask = m;
}

struct Collected {
    u32 nins, nkl, pend_b, last_line, any_failed;
};

OD_NOINL Collected collect_fill(KCtx &K) {
    const KIn &in = *K.in;
    // locals: the stores below go through generic pointers, which would
    // otherwise force the KCtx fields to be reloaded every iteration
    const LineRec *__restrict__ lines = in.lines;
    const LineIns *__restrict__ lins = in.lins;
    const Opnd *__restrict__ ops = in.ops;
    Ins *__restrict__ ins = K.ins;
    u32 *__restrict__ kl = K.kl;
    const u32 lbeg = in.lbeg, lend = in.lend, line_base = in.line_base;
    Collected c{0, 0, 0, line_base + lbeg + 1, 0}; // last_line starts at section.line
    for (u32 l = lbeg + 1; l < lend; ++l) {
        if (lines[l].role != LR_TEXT)
            continue;
        const LineIns L = lins[l];
        for (u32 k = 0; k < L.nlabels; ++k)
            kl[c.nkl++] = L.lab_start + k;
        if (!(L.flags & IF_HAS_INS))
            continue;
        c.any_failed |= L.flags & IF_PARSE_FAILED;
        collect_ins(ins[c.nins++], L, ops, line_base + l + 1, c.pend_b, c.nkl - c.pend_b);
        c.pend_b = c.nkl;
        c.last_line = line_base + l + 1;
    }
    return c;
}

OD_NOINL void collect_finish(KCtx &K, const Collected &c) {
    K.nins = c.nins;
    K.nkl = c.nkl;
    K.nins_real = K.nins;
    if (c.any_failed)
        note_parse_failures(K);
    if (K.nkl > c.pend_b) {
        Ins &I = K.ins[K.nins++];
        I.root = R_ENDPGM;
        I.prefix = PX_S;
        I.rflags = 0;
        I.sfx[0] = I.sfx[1] = 0;
        I.nops = 0;
        I.flags = IF_HAS_INS | IF_SYNTH;
        I.op_start = 0;
        I.line = c.last_line;
        I.src.off = 0;
        I.src.len = 0;
        I.lab_b = c.pend_b;
        I.lab_n = K.nkl - c.pend_b;
        I.xkind = XK_NONE;
        I.xmask = 0;
    }
}

// ============================================================== CFG
OD_INL bool is_branch(const Ins &I) {
    return I.prefix == PX_S && (I.root == R_BRANCH || (I.rflags & RF_CBRANCH));
}
OD_INL bool is_endpgm(const Ins &I) { return I.prefix == PX_S && I.root == R_ENDPGM; }

OD_INL const Label &klabel(const KCtx &K, u32 kli) { return K.in->labs[K.kl[kli]]; }

// lmap_put for lanes inserting concurrently: a slot is claimed with a CAS on
// its key; a label repeated across blocks keeps the highest block, which is
// what inserting in block order (the last insert wins) gives.
OD_INL void lmap_put_atomic(KCtx &K, u32 kli, u32 block) {
    const Label &L = klabel(K, kli);
    u32 i = (u32)(L.hash >> 32) & (K.lmap_cap - 1);
    for (;;) {
        const u32 cur = cas_u32(&K.lmap[2 * i], 0u, kli + 1);
        if (cur == 0) {
            max_u32(&K.lmap[2 * i + 1], block);
            return;
        }
        const Label &M = klabel(K, cur - 1);
        if (M.hash == L.hash && M.len == L.len && bytes_eq(K.in->t + M.off, K.in->t + L.off, L.len)) {
            max_u32(&K.lmap[2 * i + 1], block);
            return;
        }
        i = (i + 1) & (K.lmap_cap - 1);
    }
}

OD_INL int lmap_get(const KCtx &K, Span name) {
    u64 h = fnv1a64(K.in->t + name.off, name.len);
    u32 i = (u32)(h >> 32) & (K.lmap_cap - 1);
    while (K.lmap[2 * i]) {
        const Label &M = klabel(K, K.lmap[2 * i] - 1);
        if (M.hash == h && M.len == name.len &&
            bytes_eq(K.in->t + M.off, K.in->t + name.off, name.len))
            return (int)K.lmap[2 * i + 1];
        i = (i + 1) & (K.lmap_cap - 1);
    }
    return -1;
}

OD_NOINL int resolve_target(KCtx &K, const Ins &I) {
    if (I.nops == 0 || op_at(K, I, 0).kind != OK_SYMBOL) {
        K.failed = true;
        diag(K, DG_BR_NOLABEL, I.line);
        return -1;
    }
    const Opnd &o = op_at(K, I, 0);
    int b = lmap_get(K, Span{o.r.a, o.r.b});
    if (b < 0) {
        K.failed = true;
        diag(K, DG_BR_UNDEF, I.line, 0, Span{o.r.a, o.r.b});
    }
    return b;
}

constexpr u32 kNoSucc = 0xffffffffu;

OD_INL void sync_succ(KCtx &K, u32 b) {
    const Block &B = K.blk[b];
    K.sx[2 * b] = B.nsucc > 0 ? (u32)B.succ[0] : kNoSucc;
    K.sx[2 * b + 1] = B.nsucc > 1 ? (u32)B.succ[1] : kNoSucc;
}
OD_INL bool blk_reach(const KCtx &K, u32 b) { return (K.rbits[b >> 5] >> (b & 31)) & 1; }
OD_INL void set_reach(KCtx &K, u32 b) { K.rbits[b >> 5] |= 1u << (b & 31); }

// Returns the number of reachable blocks.
// cfg.mark_reachable (cfg.cpp:23-39): the set of blocks reachable from block
// 0, computed by forward sweeps over the block list instead of a depth-first
// walk (the set is the same): words of 32 blocks are visited in order, a set
// bit's successors are marked, a successor in the same word is picked up in
// the same visit, and an edge back into an earlier word reopens that word.
// Every block is expanded once; the successor pairs stream in order.
OD_NOINL u32 mark_reachable(KCtx &K) {
    u32 *__restrict__ rb = K.rbits;
    const u32 *__restrict__ sx = K.sx;
    u32 *__restrict__ done = K.work; // per word: blocks already expanded
    const u32 nb = K.nblk;
    const u32 nw = (nb + 31) / 32;
    for (u32 w = 0; w < nw; ++w) {
        rb[w] = 0;
        done[w] = 0;
    }
    if (!nb)
        return 0;
    rb[0] = 1;
    u32 lo = 0;
    while (lo < nw) {
        u32 w = lo;
        lo = nw;
        for (; w < nw; ++w) {
            u32 cur = rb[w];
            u32 pend = cur & ~done[w];
            if (!pend)
                continue;
            u32 dn = done[w];
            while (pend) {
                const u32 i = ctz32(pend);
                dn |= 1u << i;
                const u32 b = 32 * w + i;
                const u32 s2[2] = {sx[2 * b], sx[2 * b + 1]};
                for (u32 q = 0; q < 2; ++q) {
                    const u32 t = s2[q];
                    if (t == kNoSucc)
                        continue;
                    const u32 tw = t >> 5, tb = 1u << (t & 31);
                    if (tw == w) {
                        cur |= tb;
                    } else if (!(rb[tw] & tb)) {
                        rb[tw] |= tb;
                        if (tw < w && tw < lo)
                            lo = tw;
                    }
                }
                pend = cur & ~dn;
            }
            rb[w] = cur;
            done[w] = dn;
        }
    }
    u32 nr = 0;
    for (u32 w = 0; w < nw; ++w)
        nr += popc32(rb[w]);
    return nr;
}

// build_cfg's conditional-branch ParseErrors (cfg.cpp:125-130).
OD_NOINL void cbranch_error(KCtx &K, const Ins &last, bool unsupported) {
    K.failed = true;
    if (unsupported) { // the mnemonic: "s_" + root (+ suffixes); the host strips it
        Span w, rest;
        split_word(K.in->t, last.src, &w, &rest);
        diag(K, DG_CBR_UNSUP, last.line, 0, w);
    } else {
        diag(K, DG_CBR_END, last.line);
    }
}

// build_cfg's "unreachable code" notes (cfg.cpp:152-154), block order.
OD_NOINL void note_unreachable(KCtx &K) {
    for (u32 b = 0; b < K.nblk; ++b)
        if (!blk_reach(K, b))
            diag(K, DG_UNREACHABLE, K.ins[K.blk[b].ib].line);
}

// build_cfg  cfg.cpp:64-156
// Terminator of block bi (cfg.cpp:100-146) without its diagnostics: returns
// the ParseError it would raise (0 none; 1 branch without a label operand,
// 2 undefined label, 3 unsupported conditional branch, 4 conditional branch
// at the end).
OD_INL u32 block_term(KCtx &K, u32 bi) {
    Block &B = K.blk[bi];
    const Ins &last = K.ins[B.ie - 1];
    const int next = bi + 1 < K.nblk ? (int)bi + 1 : -1;
    Term &t = B.term;
    t.line = last.line;
    u32 err = 0;
    auto target = [&](const Ins &I) -> int {
        if (I.nops == 0 || op_at(K, I, 0).kind != OK_SYMBOL) {
            err = 1;
            return -1;
        }
        const Opnd &o = op_at(K, I, 0);
        const int tb = lmap_get(K, Span{o.r.a, o.r.b});
        if (tb < 0)
            err = 2;
        return tb;
    };
    if (is_endpgm(last)) {
        t.kind = T_END;
    } else if (last.prefix == PX_S && last.root == R_BRANCH) {
        t.kind = T_UNCOND;
        t.taken = target(last);
    } else if (last.prefix == PX_S && (last.rflags & RF_CBRANCH)) {
        int cc = -1;
        switch (last.root) {
        case R_CBRANCH_SCC0: cc = C_SCC0; break;
        case R_CBRANCH_SCC1: cc = C_SCC1; break;
        case R_CBRANCH_VCCZ: cc = C_VCCZ; break;
        case R_CBRANCH_VCCNZ: cc = C_VCCNZ; break;
        case R_CBRANCH_EXECZ: cc = C_EXECZ; break;
        case R_CBRANCH_EXECNZ: cc = C_EXECNZ; break;
        default: break;
        }
        if (cc < 0 || next < 0)
            return cc < 0 ? 3 : 4;
        t.kind = T_COND;
        t.cc = (u8)cc;
        t.taken = target(last);
        t.not_taken = next;
    } else if (next >= 0) {
        t.kind = T_FALL;
        t.taken = next;
    } else {
        t.kind = T_END;
    }
    if (t.kind == T_COND) {
        B.succ[0] = t.taken;
        B.succ[1] = t.not_taken;
        B.nsucc = 2;
    } else if (t.taken >= 0) {
        B.succ[0] = t.taken;
        B.nsucc = 1;
    }
    sync_succ(K, bi);
    return err;
}

// build_cfg  cfg.cpp:64-156, split across the warp: leaders from a ballot
// over 32 instructions at a time (block ids = a running prefix count), the
// label map filled in block order, terminators per block in parallel.  The
// reference stops at the first block (in order) whose terminator raises a
// ParseError: the lowest such block's diagnostic is the one emitted.
OD_NOINL bool build_cfg(KCtx &K) {
    u32 n = K.nins;
    K.blk_cap = n + 2;
    if (K.in->nblk_cap && K.in->nblk_cap < K.blk_cap)
        K.blk_cap = K.in->nblk_cap;
    K.blk = K.mem->get<Block>(K.blk_cap);
    K.stamp = K.mem->get<u32>(K.blk_cap);
    K.sx = K.mem->get<u32>(2 * K.blk_cap);
    K.rbits = K.mem->get<u32>(K.blk_cap / 32 + 1);
    K.work = K.mem->get<u32>(2 * K.blk_cap + 4);
    K.supp = K.mem->get<u8>(n + 1);
    u32 lc = 16;
    while (lc < 2 * (K.nkl + 1))
        lc <<= 1;
    K.lmap_cap = lc;
    K.lmap = K.mem->get<u32>(2 * lc);
    if (!K.blk || !K.stamp || !K.work || !K.supp || !K.lmap || !K.sx || !K.rbits)
        return false;
    const u32 m = wmask(), r = wrank(m), nl = wsize(m);
    for (u32 i = r; i < 2 * lc; i += nl)
        K.lmap[i] = 0;
    for (u32 i = r; i < n; i += nl)
        K.supp[i] = 0;
    for (u32 i = r; i < K.blk_cap; i += nl)
        K.stamp[i] = 0;
    K.stamp_gen = 0;
    K.nblk = 0;
    wsync(m);
    if (n == 0) {
        Block &B = K.blk[K.nblk++];
        B.ib = B.ie = 0;
        B.lab_b = B.lab_n = 0;
        term_default(B.term);
        B.term.kind = T_END;
        B.nsucc = 0;
        B.reachable = 1;
        B.absorbed = 0;
        B.xfront.kind = B.xback.kind = XK_NONE;
        sync_succ(K, 0);
        K.rbits[0] = 1;
        return true;
    }
    // leaders: instruction 0, labelled instructions, and the instruction after
    // a branch or s_endpgm
    u32 nb = 0;
    for (u32 i0 = 0; i0 < n; i0 += nl) {
        const u32 i = i0 + r;
        bool lead = false;
        if (i < n) {
            lead = i == 0 || K.ins[i].lab_n > 0;
            if (i > 0 && !lead) {
                const Ins &P = K.ins[i - 1];
                lead = is_branch(P) || is_endpgm(P);
            }
        }
        const u32 bal = wballot(m, lead);
        if (lead) {
            const u32 id = nb + wbelow(bal);
            if (id < K.blk_cap) {
                const Ins &I = K.ins[i];
                Block &B = K.blk[id];
                B.ib = i;
                B.ie = n;
                B.lab_b = I.lab_b;
                B.lab_n = I.lab_n;
                term_default(B.term);
                B.nsucc = 0;
                B.reachable = 1;
                B.absorbed = 0;
                B.xfront.kind = B.xback.kind = XK_NONE;
                if (id)
                    K.blk[id - 1].ie = i;
            }
        }
        nb += popc32(bal);
    }
    wsync(m);
    if (nb > K.blk_cap)
        return false; // size bound too tight: KS_OOM, retried at the worst case
    K.nblk = nb;
    // the label map (a label repeated across blocks maps to its last block),
    // blocks split across the lanes
    for (u32 bi = r; bi < nb; bi += nl) {
        const Block &B = K.blk[bi];
        for (u32 k = 0; k < B.lab_n; ++k)
            lmap_put_atomic(K, B.lab_b + k, bi);
    }
    wsync(m);
    u32 first_err = 0xffffffffu;
    for (u32 bi = r; bi < nb; bi += nl)
        if (block_term(K, bi) && bi < first_err)
            first_err = bi;
    first_err = wmin(m, first_err);
    wsync(m);
    if (first_err != 0xffffffffu) { // the reference's ParseError: the first block's diagnostic
        const Ins &last = K.ins[K.blk[first_err].ie - 1];
        const int next = first_err + 1 < nb ? (int)first_err + 1 : -1;
        if (last.prefix == PX_S && (last.rflags & RF_CBRANCH) && !is_endpgm(last) && last.root != R_BRANCH) {
            const bool unsupported = !(last.root == R_CBRANCH_SCC0 || last.root == R_CBRANCH_SCC1 ||
                                       last.root == R_CBRANCH_VCCZ || last.root == R_CBRANCH_VCCNZ ||
                                       last.root == R_CBRANCH_EXECZ || last.root == R_CBRANCH_EXECNZ);
            if (unsupported || next < 0) {
                cbranch_error(K, last, unsupported);
                return true;
            }
        }
        resolve_target(K, last); // emits the branch-target diagnostic and fails the kernel
        return true;
    }
    if (mark_reachable(K) < K.nblk)
        note_unreachable(K);
    return true;
}

// annotate_exec for one block: first and last non-suppressed exec op.
OD_NOINL void annotate_block(KCtx &K, u32 b) {
    Block &B = K.blk[b];
    B.xfront.kind = B.xback.kind = XK_NONE;
    for (u32 i = B.ib; i < B.ie; ++i) {
        if (K.supp[i])
            continue;
        const Ins &I = K.ins[i];
        if (I.xkind == XK_NONE)
            continue;
        XOp x;
        x.kind = I.xkind;
        x.index = i - B.ib;
        x.mask = I.xmask;
        x.ins = i;
        if (B.xfront.kind == XK_NONE)
            B.xfront = x;
        B.xback = x;
    }
}

// split_block  structurizer.cpp:416-435
OD_NOINL u32 split_block(KCtx &K, u32 id, u32 at) {
    if (K.nblk >= K.blk_cap) { // the size bound was too tight: retry at the worst case
        K.oom = true;
        return id;
    }
    u32 nid = K.nblk++;
    Block &B = K.blk[id];
    Block &N = K.blk[nid];
    N.ib = B.ib + at;
    N.ie = B.ie;
    N.lab_b = N.lab_n = 0;
    N.term = B.term;
    N.nsucc = B.nsucc;
    N.succ[0] = B.succ[0];
    N.succ[1] = B.succ[1];
    N.reachable = 1; // BasicBlock default (reachability is not recomputed)
    N.absorbed = 0;
    N.xfront.kind = N.xback.kind = XK_NONE;
    B.ie = B.ib + at;
    term_default(B.term);
    B.term.kind = T_FALL;
    B.term.taken = (i32)nid;
    B.term.line = K.ins[N.ib].line;
    B.succ[0] = (i32)nid;
    B.nsucc = 1;
    sync_succ(K, id);
    sync_succ(K, nid);
    set_reach(K, nid); // BasicBlock default (reachability is not recomputed)
    return nid;
}

// canonicalize_exec_blocks run to its fixed point (structurizer.cpp:440-463,
// 613-615).  The reference restarts its scan after every split; blocks
// before the split point are already canonical and a split block becomes
// canonical, so one forward pass over the growing block list performs the
// identical split sequence.
OD_NOINL void canonicalize(KCtx &K) {
    const u32 m = wmask(), r = wrank(m), nl = wsize(m);
    for (u32 b = 0; b < K.nblk; ++b) {
        Block &B = K.blk[b];
        const u32 size = B.ie - B.ib;
        const bool tail = B.term.kind == T_COND && (B.term.cc == C_EXECZ || B.term.cc == C_EXECNZ);
        const u32 want = tail ? size - 2 : size - 1; // (unsigned, as the reference's size_t)
        // the first exec op that forces a split, 32 instructions at a time
        for (u32 i0 = B.ib; i0 < B.ie; i0 += nl) {
            const u32 i = i0 + r;
            bool hit = false;
            if (i < B.ie && !K.supp[i]) {
                const Ins &I = K.ins[i];
                const u32 index = i - B.ib;
                hit = I.xkind != XK_NONE && (I.xkind == XK_SAVE ? index < want : index > 0);
            }
            const u32 bal = wballot(m, hit);
            if (bal) {
                const u32 pos = ctz32(bal);
                const u32 first = i0 + popc32(m & ((1u << pos) - 1)) - B.ib;
                split_block(K, b, K.ins[B.ib + first].xkind == XK_SAVE ? first + 1 : first);
                break;
            }
        }
    }
    wsync(m);
    for (u32 b = r; b < K.nblk; b += nl) // annotate_block edits only its own block
        annotate_block(K, b);
    wsync(m);
}

OD_INL bool first_exec_op_is(const KCtx &K, u32 b, u32 kind, u32 mask) {
    const Block &B = K.blk[b];
    if (B.xfront.kind == XK_NONE || B.ie == B.ib)
        return false;
    return B.xfront.kind == kind && B.xfront.mask == mask && B.xfront.index == 0;
}

// mask_stops  structurizer.cpp:482-507.  Returns the number of stops found
// (saturating at 2) and the first in *stop.
OD_NOINL u32 mask_stops(KCtx &K, const i32 *starts, u32 nstarts, u32 mask, i32 header, i32 *stop) {
    u32 gen = ++K.stamp_gen;
    u32 sp = 0;
    u32 nstops = 0;
    for (u32 s = 0; s < nstarts; ++s)
        K.work[sp++] = (u32)starts[s];
    while (sp) {
        i32 id = (i32)K.work[--sp];
        if (id < 0 || (u32)id >= K.nblk || K.stamp[id] == gen)
            continue;
        K.stamp[id] = gen;
        const Block &B = K.blk[id];
        if (id != header) {
            if (first_exec_op_is(K, (u32)id, XK_INVERT, mask) ||
                first_exec_op_is(K, (u32)id, XK_RESTORE, mask)) {
                if (nstops == 0)
                    *stop = id;
                ++nstops;
                continue;
            }
            if (B.xback.kind == XK_SAVE && B.xback.mask == mask)
                continue;
        }
        for (u32 s = 0; s < B.nsucc; ++s)
            K.work[sp++] = (u32)B.succ[s];
    }
    return nstops;
}

// retarget_preds  structurizer.cpp:512-525
// Returns whether some reachable block now has an edge to `to`.
OD_NOINL bool retarget_preds(KCtx &K, i32 from, i32 to, i32 keep) {
    const u32 f = (u32)from;
    const u32 m = wmask(); // blocks split across the warp: each edits only its own edges
    bool fed = false;
    for (u32 p = wrank(m); p < K.nblk; p += wsize(m)) {
        if ((K.sx[2 * p] != f && K.sx[2 * p + 1] != f) || (i32)p == keep)
            continue;
        fed |= blk_reach(K, p);
        Block &P = K.blk[p];
        for (u32 s = 0; s < P.nsucc; ++s)
            if (P.succ[s] == from)
                P.succ[s] = to;
        if (P.term.taken == from)
            P.term.taken = to;
        if (P.term.not_taken == from)
            P.term.not_taken = to;
        sync_succ(K, p);
    }
    fed = wor(m, fed ? 1u : 0u) != 0;
    wsync(m);
    return fed;
}

// Whether some reachable block has an edge to b (lanes over the blocks).
OD_NOINL bool has_reachable_pred(const KCtx &K, u32 b) {
    const u32 m = wmask();
    bool any = false;
    for (u32 p = wrank(m); p < K.nblk && !any; p += wsize(m))
        any = (K.sx[2 * p] == b || K.sx[2 * p + 1] == b) && blk_reach(K, p);
    return wor(m, any ? 1u : 0u) != 0;
}

// Whether the flow graph has no cycle (Kahn's algorithm over the successor
// pairs).  normalize_if_else's rewrites never create one: a new edge
// header -> else or pred -> join shortcuts a path that already existed, and
// split_block only inserts a block on an edge.
OD_NOINL bool flow_acyclic(KCtx &K) {
    const u32 nb = K.nblk;
    u32 *indeg = K.stamp, *q = K.work;
    for (u32 b = 0; b < nb; ++b)
        indeg[b] = 0;
    for (u32 b = 0; b < nb; ++b)
        for (u32 k = 0; k < 2; ++k)
            if (K.sx[2 * b + k] != kNoSucc)
                indeg[K.sx[2 * b + k]]++;
    u32 qh = 0, qt = 0;
    for (u32 b = 0; b < nb; ++b)
        if (!indeg[b])
            q[qt++] = b;
    while (qh < qt) {
        const u32 b = q[qh++];
        for (u32 k = 0; k < 2; ++k) {
            const u32 t = K.sx[2 * b + k];
            if (t != kNoSucc && --indeg[t] == 0)
                q[qt++] = t;
        }
    }
    for (u32 b = 0; b < nb; ++b) // the traversal stamps start clear again
        K.stamp[b] = 0;
    K.stamp_gen = 0;
    return qt == nb;
}

struct MaskPattern {
    i32 header;
    u32 mask;
    u32 src_ins; // instruction holding the save (source operand = ops[1])
    bool has_bypass;
    i32 then_entry;
    i32 bypass;
};

// apply_mask_pattern  structurizer.cpp:527-609
OD_NOINL bool apply_mask_pattern(KCtx &K, const MaskPattern &pat, u32 *touched, u32 *ntouched) {
    Block &h = K.blk[pat.header];
    const u32 save_index = h.xback.index;
    i32 stop = -1;
    i32 starts[2] = {pat.then_entry, 0};
    u32 ns = mask_stops(K, starts, 1, pat.mask, pat.header, &stop);
    if (ns != 1) {
        diag(K, ns > 1 ? DG_MASK_MULTI : DG_MASK_NONE, h.term.line, (u16)pat.mask);
        return false;
    }
    const i32 invert = first_exec_op_is(K, (u32)stop, XK_INVERT, pat.mask) ? stop : -1;
    i32 then_entry = pat.then_entry, else_entry = -1, join = -1;
    bool reach_may_shrink = false;
    i32 reach_drop = -1; // the one block that leaves the reachable set (acyclic shortcut)
    *ntouched = 0;
    if (invert >= 0) {
        Block &ib = K.blk[invert];
        const bool invert_only = (ib.ie - ib.ib) <= 2 && ib.term.kind == T_COND && ib.term.cc == C_EXECZ;
        if (pat.has_bypass && pat.bypass != invert) {
            diag(K, DG_MASK_EXECZ_INV, h.term.line);
            return false;
        }
        if (invert_only) {
            else_entry = ib.term.not_taken;
            join = ib.term.taken;
            K.supp[ib.ib] = 1;
            if (ib.ie - ib.ib > 1)
                K.supp[ib.ib + 1] = 1;
            const bool join_fed = retarget_preds(K, invert, join, pat.header);
            ib.absorbed = 1;
            ib.nsucc = 0;
            sync_succ(K, (u32)invert);
            reach_may_shrink = true;
            // On an acyclic graph the inverted block is the only block that can
            // drop out, unless the join lost its last reachable predecessor:
            // every other block that lost an in-edge (the else entry) gained
            // one from the header, and in an acyclic graph a set in which every
            // non-entry block has a predecessor in the set is reachable.
            if (K.acyclic && join >= 0 && (join_fed || has_reachable_pred(K, (u32)join))) {
                reach_may_shrink = false;
                reach_drop = invert;
            }
        } else {
            i32 rstop = -1;
            u32 nr = mask_stops(K, ib.succ, ib.nsucc, pat.mask, invert, &rstop);
            if (nr != 1 || !first_exec_op_is(K, (u32)rstop, XK_RESTORE, pat.mask)) {
                diag(K, DG_MASK_NO_RESTORE, h.term.line);
                return false;
            }
            else_entry = invert;
            join = rstop;
            K.supp[ib.ib] = 1;
            retarget_preds(K, invert, join, pat.header);
        }
        touched[(*ntouched)++] = (u32)invert;
    } else {
        if (pat.has_bypass && pat.bypass != stop) {
            diag(K, DG_MASK_EXECZ_RST, h.term.line);
            return false;
        }
        join = stop;
    }
    if (join >= 0) {
        Block &jb = K.blk[join];
        if (first_exec_op_is(K, (u32)join, XK_RESTORE, pat.mask))
            K.supp[jb.ib] = 1;
        touched[(*ntouched)++] = (u32)join;
    }
    K.supp[h.ib + save_index] = 1;
    h.term.kind = T_COND;
    h.term.cc = C_MASKED;
    h.term.mask_source = op_at(K, K.ins[pat.src_ins], 1);
    h.term.not_taken = then_entry;
    h.term.taken = else_entry >= 0 ? else_entry : join;
    h.succ[0] = h.term.taken;
    h.succ[1] = h.term.not_taken;
    h.nsucc = 2;
    sync_succ(K, (u32)pat.header);
    touched[(*ntouched)++] = (u32)pat.header;
    // cfg.mark_reachable() (structurizer.cpp:606).  Every new edge targets a
    // block the mask walk reached from the (reachable) header, so
    // reachability can only shrink, and it can only shrink when the inverted
    // block loses its out-edges (invert-only form); in the other forms the
    // edge changes keep every block reachable, so the walk is skipped.
    if (reach_may_shrink) {
        mark_reachable(K);
    } else if (reach_drop >= 0) {
        K.rbits[reach_drop >> 5] &= ~(1u << (reach_drop & 31));
    }
#ifdef OD_HOST_CHECK
    if (!reach_may_shrink) {
        for (u32 b = 0; b < K.nblk; ++b)
            K.stamp[b] = blk_reach(K, b);
        mark_reachable(K);
        for (u32 b = 0; b < K.nblk; ++b)
            if (K.stamp[b] != (u32)blk_reach(K, b))
                abort();
        K.stamp_gen = 0;
        for (u32 b = 0; b < K.nblk; ++b)
            K.stamp[b] = 0;
    }
#endif
    return true;
}

// normalize_if_else  structurizer.cpp:613-654
OD_NOINL void normalize(KCtx &K) {
    canonicalize(K);
    K.acyclic = flow_acyclic(K);
    const u32 nb = K.nblk;
    for (u32 scan = 0; scan < nb; ++scan) {
        Block &b = K.blk[scan];
        if (!blk_reach(K, scan) || b.xback.kind == XK_NONE)
            continue;
        const XOp op = b.xback;
        if (op.kind != XK_SAVE || K.supp[b.ib + op.index])
            continue;
        MaskPattern pat;
        pat.header = (i32)scan;
        pat.mask = op.mask;
        pat.src_ins = op.ins;
        pat.has_bypass = false;
        pat.bypass = -1;
        if (b.term.kind == T_COND && b.term.cc == C_EXECZ) {
            pat.has_bypass = true;
            pat.then_entry = b.term.not_taken;
            pat.bypass = b.term.taken;
            if (b.ie > b.ib)
                K.supp[b.ie - 1] = 1;
        } else if (b.term.kind == T_FALL) {
            pat.then_entry = b.term.taken;
        } else {
            continue;
        }
        u32 touched[4];
        u32 nt = 0;
        if (apply_mask_pattern(K, pat, touched, &nt)) {
            for (u32 k = 0; k < nt; ++k)
                annotate_block(K, touched[k]);
        } else if (pat.has_bypass) {
            Block &hb = K.blk[pat.header];
            K.supp[hb.ie - 1] = 0;
        }
    }
}

// ========================================================== regions
OD_INL i32 entry_block(const KCtx &K, u32 r) {
    while (K.rg[r].kind != RK_BLOCK)
        r = K.child[K.rg[r].ch_b];
    return K.rg[r].block_id;
}

OD_INL i32 exit_block(const KCtx &K, u32 r) {
    for (;;) {
        const Region &R = K.rg[r];
        switch (R.kind) {
        case RK_BLOCK: return R.block_id;
        case RK_LINEAR: r = K.child[R.ch_b + R.ch_n - 1]; break;
        default:
            if (!R.join_absorbed)
                return -1;
            r = K.child[R.ch_b + R.ch_n - 1];
            break;
        }
    }
}

OD_INL u32 make_region(KCtx &K, u8 kind) {
    u32 id = ++K.nrg;
    Region &R = K.rg[id];
    R.kind = kind;
    R.join_absorbed = 0;
    R.cc = C_SCC1;
    R.then_is_taken = 0;
    R.block_id = -1;
    R.join_block = -1;
    R.has_term = 0;
    R.mask_source.kind = OK_ANNOT;
    R.mask_source.special = SP_EXEC;
    R.mask_source.pad = 0;
    R.mask_source.count = 1;
    R.mask_source.value = 0;
    R.ch_b = K.nchild;
    R.ch_n = 0;
    R.nsucc = 0;
    return id;
}

// Predecessors are kept as (count, xor of ids) per region: the matchers only
// ask for the count and, when it is 1, for the single predecessor
// (structurizer.cpp:230-352), and the xor of a one-element set is that
// element.  Succ lists are duplicate-free, so each edge counts once.
OD_INL void pred_add(KCtx &K, u32 t, u32 from) {
    K.pred_n[t]++;
    K.pred_x[t] ^= from;
    u32 e = K.efree;
    if (e)
        K.efree = K.enext[e];
    else if (K.etop < K.ecap)
        e = K.etop++;
    else {
        K.oom = true;
        return;
    }
    K.efrom[e] = from;
    K.enext[e] = K.phead[t];
    K.phead[t] = e;
}
OD_INL void pred_del(KCtx &K, u32 t, u32 from) {
    K.pred_n[t]--;
    K.pred_x[t] ^= from;
    u32 *link = &K.phead[t];
    while (*link) {
        const u32 e = *link;
        if (K.efrom[e] == from) {
            *link = K.enext[e];
            K.enext[e] = K.efree;
            K.efree = e;
            return;
        }
        link = &K.enext[e];
    }
}

OD_NOINL void rebuild_region_preds(KCtx &K) {
    K.etop = 1; // edge 0 = end of list
    K.efree = 0;
    for (u32 i = 0; i < K.nlive; ++i) {
        K.pred_n[K.live[i]] = 0;
        K.pred_x[K.live[i]] = 0;
        K.phead[K.live[i]] = 0;
    }
    for (u32 i = 0; i < K.nlive; ++i) {
        const Region &R = K.rg[K.live[i]];
        for (u32 s = 0; s < R.nsucc; ++s)
            pred_add(K, (u32)R.succ[s], K.live[i]);
    }
}

OD_INL void region_add_edge(KCtx &K, u32 from, u32 to) {
    Region &R = K.rg[from];
    for (u32 s = 0; s < R.nsucc; ++s)
        if ((u32)R.succ[s] == to)
            return;
    R.succ[R.nsucc++] = (i32)to;
}

// RegionGraph::from_cfg  structurizer.cpp:88-111
OD_NOINL bool build_regions(KCtx &K) {
    u32 cap = 2 * K.nblk + 4;
    K.rg_cap = cap;
    K.rg = K.mem->get<Region>(cap + 1);
    K.child_cap = 4 * cap + 8;
    K.child = K.mem->get<u32>(K.child_cap);
    K.live = K.mem->get<u32>(cap + 1);
    K.pred_n = K.mem->get<u32>(cap + 1);
    K.pred_x = K.mem->get<u32>(cap + 1);
    K.phead = K.mem->get<u32>(cap + 1);
    K.ecap = 2 * cap + 4;
    K.enext = K.mem->get<u32>(K.ecap);
    K.efrom = K.mem->get<u32>(K.ecap);
    K.rstamp = K.mem->get<u32>(cap + 1);
    K.dmark = K.mem->get<u32>(cap + 1);
    K.rank = K.mem->get<u32>(cap + 1);
    K.at = K.mem->get<u32>(cap + 1);
    K.cand = K.mem->get<u64>(cap / 64 + 2);
    K.rpo = K.mem->get<u32>(cap + 1);
    K.dfs = K.mem->get<u32>(2 * cap + 4);
    u32 *by_block = K.mem->get<u32>(K.nblk + 1);
    if (!K.rg || !K.child || !K.live || !K.pred_n || !K.pred_x || !K.phead || !K.enext || !K.efrom || !K.rstamp ||
        !K.rpo || !K.dfs || !by_block || !K.dmark || !K.rank || !K.at || !K.cand)
        return false;
    for (u32 i = 0; i <= cap; ++i) {
        K.rstamp[i] = 0;
        K.dmark[i] = 0;
        K.rank[i] = kNoRank;
    }
    K.rstamp_gen = 0;
    K.dmark_gen = 0;
    K.nrg = 0;
    K.nchild = 0;
    K.nlive = 0;
    K.entry_r = -1;
    for (u32 b = 0; b < K.nblk; ++b) {
        by_block[b] = 0;
        const Block &B = K.blk[b];
        if (!blk_reach(K, b) || B.absorbed)
            continue;
        u32 r = make_region(K, RK_BLOCK);
        K.rg[r].block_id = (i32)b;
        K.live[K.nlive++] = r;
        if (K.entry_r < 0)
            K.entry_r = (i32)r;
        by_block[b] = r;
        if (b == 0)
            K.entry_r = (i32)r;
    }
    for (u32 b = 0; b < K.nblk; ++b) {
        if (!by_block[b])
            continue;
        const Block &B = K.blk[b];
        for (u32 s = 0; s < B.nsucc; ++s) {
            u32 to = by_block[B.succ[s]];
            if (to)
                region_add_edge(K, by_block[b], to);
        }
    }
    rebuild_region_preds(K);
    return true;
}

OD_INL bool single_pred_is(const KCtx &K, u32 node, u32 pred) {
    return K.pred_n[node] == 1 && K.pred_x[node] == pred;
}

OD_INL void cand_set(KCtx &K, u32 r) {
    const u32 k = K.rank[r];
    if (k != kNoRank)
        K.cand[k >> 6] |= 1ull << (k & 63);
}
OD_INL void cand_clear(KCtx &K, u32 r) {
    const u32 k = K.rank[r];
    if (k != kNoRank)
        K.cand[k >> 6] &= ~(1ull << (k & 63));
}

// RegionGraph::replace  structurizer.cpp:141-185
OD_NOINL void region_replace(KCtx &K, const u32 *old, u32 nold, u32 merged) {
    const u32 gen = ++K.rstamp_gen;
    const u32 dg = ++K.dmark_gen;
    for (u32 i = 0; i < nold; ++i)
        K.rstamp[old[i]] = gen;
    Region &M = K.rg[merged];
    M.nsucc = 0;
    K.pred_n[merged] = 0;
    K.pred_x[merged] = 0;
    K.phead[merged] = 0;
    // M's successors: the old regions' exits in order (self edges to the
    // header become M's self edge), at most two.
    for (u32 i = 0; i < nold; ++i) {
        const Region &O = K.rg[old[i]];
        for (u32 s = 0; s < O.nsucc; ++s) {
            const u32 t0 = (u32)O.succ[s];
            if (K.rstamp[t0] != gen)
                pred_del(K, t0, old[i]);
            u32 t = t0 == old[0] ? merged : t0;
            if (t != merged && K.rstamp[t] == gen)
                continue;
            bool dup = false;
            for (u32 k = 0; k < M.nsucc; ++k)
                if ((u32)M.succ[k] == t)
                    dup = true;
            if (!dup && M.nsucc < 2)
                M.succ[M.nsucc++] = (i32)t;
        }
    }
    for (u32 k = 0; k < M.nsucc; ++k)
        pred_add(K, (u32)M.succ[k], merged);
    // Outside predecessors of the old regions now point at M (their succ
    // lists keep their order; duplicates collapse).
    for (u32 i = 0; i < nold; ++i) {
        for (u32 e = K.phead[old[i]]; e; e = K.enext[e]) {
            const u32 u = K.efrom[e];
            if (K.rstamp[u] == gen || K.dmark[u] == dg)
                continue;
            Region &R = K.rg[u];
            i32 out[2];
            u32 no = 0;
            for (u32 s = 0; s < R.nsucc; ++s) {
                u32 t = K.rstamp[R.succ[s]] == gen ? merged : (u32)R.succ[s];
                bool dup = false;
                for (u32 k = 0; k < no; ++k)
                    if ((u32)out[k] == t)
                        dup = true;
                if (!dup)
                    out[no++] = (i32)t;
            }
            R.nsucc = no;
            for (u32 k = 0; k < no; ++k)
                R.succ[k] = out[k];
            K.dmark[u] = dg; // u is a predecessor of M: its succ list changed
        }
    }
    // (pred lists of the old regions die with them; the marked ones gain M)
    for (u32 i = 0; i < nold; ++i)
        for (u32 e = K.phead[old[i]]; e; e = K.enext[e]) {
            const u32 u = K.efrom[e];
            if (K.dmark[u] == dg && K.rstamp[u] != gen) {
                K.dmark[u] = dg + 1; // once per predecessor
                pred_add(K, merged, u);
            }
        }
    K.dmark_gen = dg + 1;
    const u32 pg = dg + 1;   // P marked pg now
    K.nlive -= nold - 1;
    if (K.entry_r >= 0 && K.rstamp[K.entry_r] == gen)
        K.entry_r = (i32)merged;
    // The reverse post-order after the merge is the old one with the
    // absorbed regions dropped and M at the header's position: the absorbed
    // regions are reachable only through the header, and the merged region
    // has the single exit (or the join's exits, in order) the header's walk
    // reached them through (structurizer.cpp:113-139 recomputes it instead).
    const u32 hr = K.rank[old[0]];
    for (u32 i = 0; i < nold; ++i) {
        cand_clear(K, old[i]);
        if (K.rank[old[i]] != kNoRank)
            K.at[K.rank[old[i]]] = 0;
        K.rank[old[i]] = kNoRank;
    }
    K.rank[merged] = hr;
    if (hr != kNoRank)
        K.at[hr] = merged;
    // A cached matcher failure of r stays valid while r's succ list, and the
    // pred counts / single pred / succ lists of r's successors, are unchanged
    // (structurizer.cpp:230-352 read nothing else on the failing paths).
    // Changed succ lists: M and its preds P; changed pred sets: M and
    // succs(M).  So the dirty regions are M, P, and the predecessors of
    // succs(M) and of P.
    cand_set(K, merged);
    for (u32 e = K.phead[merged]; e; e = K.enext[e]) {
        const u32 u = K.efrom[e];
        cand_set(K, u);
        for (u32 f = K.phead[u]; f; f = K.enext[f])
            cand_set(K, K.efrom[f]);
    }
    for (u32 k = 0; k < M.nsucc; ++k)
        for (u32 e = K.phead[M.succ[k]]; e; e = K.enext[e])
            cand_set(K, K.efrom[e]);
    (void)pg;
}

OD_INL const Term *header_term(const KCtx &K, u32 r, bool *usable) {
    i32 ex = exit_block(K, r);
    const Term *t = ex >= 0 ? &K.blk[ex].term : nullptr;
    if (!t) {
        *usable = true;
        return nullptr;
    }
    *usable = t->kind == T_COND && t->cc != C_EXECZ && t->cc != C_EXECNZ;
    return t;
}

OD_INL void set_cond(KCtx &K, u32 m, const Term *term, bool then_is_taken) {
    Region &M = K.rg[m];
    if (term) {
        M.cc = term->cc;
        M.mask_source = term->mask_source;
        M.has_term = 1;
    }
    M.then_is_taken = then_is_taken ? 1 : 0;
}

OD_INL void push_children(KCtx &K, u32 m, const u32 *c, u32 n) {
    Region &M = K.rg[m];
    M.ch_b = K.nchild;
    for (u32 i = 0; i < n; ++i)
        K.child[K.nchild++] = c[i];
    M.ch_n = n;
}

// match_if_else  structurizer.cpp:230-274
OD_NOINL u32 match_if_else(KCtx &K, u32 r) {
    const Region &R = K.rg[r];
    if (R.nsucc != 2 || R.succ[0] == R.succ[1])
        return 0;
    bool usable;
    const Term *term = header_term(K, r, &usable);
    if (!usable)
        return 0;
    u32 a = (u32)R.succ[0], b = (u32)R.succ[1];
    if (!single_pred_is(K, a, r) || !single_pred_is(K, b, r))
        return 0;
    const Region &A = K.rg[a], &B = K.rg[b];
    if (A.nsucc != 1 || B.nsucc != 1 || A.succ[0] != B.succ[0])
        return 0;
    u32 j = (u32)A.succ[0];
    if (j == r)
        return 0;
    u32 then_r = a, else_r = b;
    if (term && term->kind == T_COND) {
        if (entry_block(K, a) == term->taken) {
            then_r = b;
            else_r = a;
        }
    }
    const bool absorb = K.pred_n[j] == 2;
    if (K.nchild + 4 > K.child_cap || K.nrg + 1 > K.rg_cap) {
        K.oom = true;
        return 0;
    }
    u32 m = make_region(K, RK_IFELSE);
    K.nif++;
    set_cond(K, m, term, false);
    K.rg[m].join_block = entry_block(K, j);
    u32 ch[4] = {r, then_r, else_r, j};
    u32 n = absorb ? 4 : 3;
    push_children(K, m, ch, n);
    K.rg[m].join_absorbed = absorb ? 1 : 0;
    region_replace(K, ch, n, m);
    return m;
}

// match_if  structurizer.cpp:276-323
OD_NOINL u32 match_if(KCtx &K, u32 r) {
    const Region &R = K.rg[r];
    if (R.nsucc != 2 || R.succ[0] == R.succ[1])
        return 0;
    bool usable;
    const Term *term = header_term(K, r, &usable);
    if (!usable)
        return 0;
    u32 then_r = 0;
    u32 j = 0;
    for (u32 k = 0; k < 2; ++k) {
        u32 cand = (u32)R.succ[k];
        u32 other = (u32)R.succ[1 - k];
        if (!single_pred_is(K, cand, r))
            continue;
        const Region &C = K.rg[cand];
        if (C.nsucc == 1 && (u32)C.succ[0] == other && other != r) {
            then_r = cand;
            j = other;
            break;
        }
    }
    if (!then_r)
        return 0;
    bool then_is_taken = false;
    if (term && term->kind == T_COND)
        then_is_taken = entry_block(K, then_r) == term->taken;
    const bool absorb = K.pred_n[j] == 2;
    if (K.nchild + 3 > K.child_cap || K.nrg + 1 > K.rg_cap) {
        K.oom = true;
        return 0;
    }
    u32 m = make_region(K, RK_IFTHEN);
    K.nif++;
    set_cond(K, m, term, then_is_taken);
    K.rg[m].join_block = entry_block(K, j);
    u32 ch[3] = {r, then_r, j};
    u32 n = absorb ? 3 : 2;
    push_children(K, m, ch, n);
    K.rg[m].join_absorbed = absorb ? 1 : 0;
    region_replace(K, ch, n, m);
    return m;
}

// match_linear  structurizer.cpp:325-352
OD_NOINL u32 match_linear(KCtx &K, u32 r) {
    u32 cb = K.nchild; // build the chain directly in the child pool
    u32 n = 0;
    if (cb + 1 > K.child_cap) {
        K.oom = true;
        return 0;
    }
    K.child[cb + n++] = r;
    u32 cur = r;
    for (;;) {
        const Region &C = K.rg[cur];
        if (C.nsucc != 1)
            break;
        u32 next = (u32)C.succ[0];
        if (next == r || !single_pred_is(K, next, cur))
            break;
        if (K.rg[next].nsucc > 1)
            break;
        if (cb + n + 1 > K.child_cap) {
            K.oom = true;
            return 0;
        }
        K.child[cb + n++] = next;
        cur = next;
    }
    if (n < 2)
        return 0;
    if (K.nrg + 1 > K.rg_cap) {
        K.oom = true;
        return 0;
    }
    u32 m = make_region(K, RK_LINEAR);
    K.rg[m].ch_b = cb;
    K.rg[m].ch_n = n;
    K.nchild = cb + n;
    region_replace(K, K.child + cb, n, m);
    return m;
}

// RegionGraph::rpo  structurizer.cpp:113-139
OD_NOINL u32 region_rpo(KCtx &K) {
    if (K.entry_r < 0)
        return 0;
    u32 gen = ++K.rstamp_gen;
    u32 sp = 0, npost = 0;
    K.dfs[2 * sp] = (u32)K.entry_r;
    K.dfs[2 * sp + 1] = 0;
    ++sp;
    K.rstamp[K.entry_r] = gen;
    while (sp) {
        u32 node = K.dfs[2 * (sp - 1)];
        u32 &idx = K.dfs[2 * (sp - 1) + 1];
        const Region &R = K.rg[node];
        if (idx < R.nsucc) {
            u32 s = (u32)R.succ[idx++];
            if (K.rstamp[s] != gen) {
                K.rstamp[s] = gen;
                K.dfs[2 * sp] = s;
                K.dfs[2 * sp + 1] = 0;
                ++sp;
            }
        } else {
            K.rpo[npost++] = node;
            --sp;
        }
    }
    // reverse in place
    for (u32 i = 0; i < npost / 2; ++i) {
        u32 x = K.rpo[i];
        K.rpo[i] = K.rpo[npost - 1 - i];
        K.rpo[npost - 1 - i] = x;
    }
    return npost;
}

// reduce  structurizer.cpp:354-403.  The reference rescans a fresh reverse
// post-order after every merge and takes the first region a matcher accepts.
// Here the order is maintained across merges (region_replace) and a region
// whose matchers failed is only retried once a merge touched its
// neighbourhood, which selects the same region at every step.
// ========================================================== DOT dumps
// Two passes over the same printer: count (p == null), then write.
struct DotSink {
    u8 *p;
    u64 n;
    OD_INL void c(u8 ch) {
        if (p)
            p[n] = ch;
        ++n;
    }
    OD_NOINL void s(const char *z) {
        while (*z)
            c((u8)*z++);
    }
    OD_NOINL void m(const u8 *b, u32 len) {
        for (u32 i = 0; i < len; ++i)
            c(b[i]);
    }
    OD_NOINL void u(u64 v) {
        u8 b[24];
        int i = 0;
        do {
            b[i++] = (u8)('0' + v % 10);
            v /= 10;
        } while (v);
        while (i)
            c(b[--i]);
    }
};

// to_dot  cfg.cpp:400-424 (after normalize_if_else, decompiler.cpp:72-73)
OD_NOINL void cfg_dot(const KCtx &K, DotSink &o) {
    const u8 *t = K.in->t;
    Span nm;
    {
        Span w, rest, extra;
        const LineRec &L = K.in->lines[K.in->lbeg];
        split_word(t, Span{L.off, L.len}, &w, &rest);
        split_word(t, rest, &nm, &extra);
    }
    o.s("digraph \"");
    o.m(t + nm.off, nm.len);
    o.s("\" {\n  node [shape=box, fontname=\"monospace\"];\n");
    for (u32 b = 0; b < K.nblk; ++b) {
        const Block &B = K.blk[b];
        o.s("  b");
        o.u(b);
        o.s(" [label=\"B");
        o.u(b);
        for (u32 l = 0; l < B.lab_n; ++l) {
            const Label &L = klabel(K, B.lab_b + l);
            o.c(' ');
            o.m(t + L.off, L.len);
        }
        o.s("\\n");
        o.u(B.ie - B.ib);
        o.s(" ins");
        if (!blk_reach(K, b))
            o.s(" (dead)");
        o.s("\"];\n");
    }
    for (u32 b = 0; b < K.nblk; ++b) {
        const Block &B = K.blk[b];
        if (B.term.kind == T_COND) {
            o.s("  b");
            o.u(b);
            o.s(" -> b");
            o.u((u32)B.term.taken);
            o.s(" [label=\"T\"];\n  b");
            o.u(b);
            o.s(" -> b");
            o.u((u32)B.term.not_taken);
            o.s(" [label=\"F\"];\n");
        } else {
            for (u32 q = 0; q < B.nsucc; ++q) {
                o.s("  b");
                o.u(b);
                o.s(" -> b");
                o.u((u32)B.succ[q]);
                o.s(";\n");
            }
        }
    }
    o.s("}\n");
}

// region_graph_dot  structurizer.cpp:669-688.  Live regions in id order (the
// reference appends each merged region to live_, so its order is by id);
// a region is dead once it is a child of a merged region.
OD_NOINL void region_dot(const KCtx &K, DotSink &o, u32 step) {
    const u32 gen = ++const_cast<KCtx &>(K).rstamp_gen;
    for (u32 r = 1; r <= K.nrg; ++r)
        if (K.rg[r].kind != RK_BLOCK)
            for (u32 c = 0; c < K.rg[r].ch_n; ++c)
                K.rstamp[K.child[K.rg[r].ch_b + c]] = gen;
    o.s("digraph \"step");
    o.u(step);
    o.s("\" {\n  node [shape=ellipse, fontname=\"monospace\"];\n");
    for (u32 r = 1; r <= K.nrg; ++r) {
        if (K.rstamp[r] == gen)
            continue;
        const Region &R = K.rg[r];
        o.s("  r");
        o.u(r);
        o.s(" [label=\"");
        o.u(r);
        switch (R.kind) {
        case RK_BLOCK:
            o.s(" B");
            o.u((u32)R.block_id);
            break;
        case RK_LINEAR: o.s(" lin"); break;
        case RK_IFTHEN: o.s(" if"); break;
        default: o.s(" if/else"); break;
        }
        o.s("\"];\n");
    }
    for (u32 r = 1; r <= K.nrg; ++r) {
        if (K.rstamp[r] == gen)
            continue;
        const Region &R = K.rg[r];
        for (u32 q = 0; q < R.nsucc; ++q) {
            o.s("  r");
            o.u(r);
            o.s(" -> r");
            o.u((u32)R.succ[q]);
            o.s(";\n");
        }
    }
    o.s("}\n");
}

// ReduceResult as text (the inspection record of reduce, structurizer.cpp:
// 354-403): one "merge <kind> <result> <absorbed...>" line per MergeRecord in
// order (merged regions are created in merge order, after the leaves), then
// "root <id>" or "residue <ids...>" (live regions in id order).
OD_NOINL void reduce_text(const KCtx &K, DotSink &o) {
    const u32 gen = ++const_cast<KCtx &>(K).rstamp_gen;
    for (u32 r = 1; r <= K.nrg; ++r) {
        const Region &R = K.rg[r];
        if (R.kind == RK_BLOCK)
            continue;
        o.s("merge ");
        o.u(R.kind);
        o.c(' ');
        o.u(r);
        for (u32 c = 0; c < R.ch_n; ++c) {
            o.c(' ');
            o.u(K.child[R.ch_b + c]);
            K.rstamp[K.child[R.ch_b + c]] = gen;
        }
        o.c('\n');
    }
    if (K.reduced) {
        o.s("root ");
        o.u(K.root_r);
    } else {
        o.s("residue");
        for (u32 r = 1; r <= K.nrg; ++r)
            if (K.rstamp[r] != gen) {
                o.c(' ');
                o.u(r);
            }
    }
    o.c('\n');
}

// DecompiledKernel::cfg export (step -4, with DUMP_BODY): the flow graph as
// normalize_if_else leaves it (decompiler.cpp:69-71), one line per block:
//   B <ib> <ie> <kind> <cc> <taken> <not_taken> <line> <reachable> <absorbed>
//     <nsucc> <succ...> S <nsupp> <suppressed index in block...> L <nlab> <label...>
// Instruction ranges index the kernel's instruction list; kind / cc are
// TermKind / CondCode (cfg.hpp:20-37).  preds (rebuild_preds), exec_ops
// (annotate_exec) and the Masked term's source operand follow from these and
// are rebuilt by the binding (integration/ocldec_b200_dropin.cpp).
OD_NOINL void cfg_text(const KCtx &K, DotSink &o) {
    const u8 *t = K.in->t;
    o.u(K.nblk);
    o.c('\n');
    for (u32 b = 0; b < K.nblk; ++b) {
        const Block &B = K.blk[b];
        o.s("B ");
        o.u(B.ib);
        o.c(' ');
        o.u(B.ie);
        o.c(' ');
        o.u(B.term.kind);
        o.c(' ');
        o.u(B.term.cc);
        o.c(' ');
        o.u((u64)(i64)(B.term.taken + 1)); // -1 -> 0
        o.c(' ');
        o.u((u64)(i64)(B.term.not_taken + 1));
        o.c(' ');
        o.u(B.term.line);
        o.c(' ');
        o.u(blk_reach(K, b) ? 1 : 0);
        o.c(' ');
        o.u(B.absorbed ? 1 : 0);
        o.c(' ');
        o.u(B.nsucc);
        for (u32 q = 0; q < B.nsucc; ++q) {
            o.c(' ');
            o.u((u32)B.succ[q]);
        }
        u32 ns = 0;
        for (u32 i = B.ib; i < B.ie; ++i)
            ns += K.supp[i] ? 1 : 0;
        o.s(" S ");
        o.u(ns);
        for (u32 i = B.ib; i < B.ie; ++i)
            if (K.supp[i]) {
                o.c(' ');
                o.u(i - B.ib);
            }
        o.s(" L ");
        o.u(B.lab_n);
        for (u32 l = 0; l < B.lab_n; ++l) {
            const Label &L = klabel(K, B.lab_b + l);
            o.c(' ');
            o.m(t + L.off, L.len);
        }
        o.c('\n');
    }
}

// body export printer (od_lower.cuh, after the renderer's label helper)
OD_NOINL void body_text(KCtx &K, DotSink &o);

OD_INL void dump_print(KCtx &K, DotSink &o, i32 step) {
    if (step == -3) {
        body_text(K, o);
        return;
    }
    if (step == -4) {
        cfg_text(K, o);
        return;
    }
    if (step == -1)
        cfg_dot(K, o);
    else if (step == -2)
        reduce_text(K, o);
    else
        region_dot(K, o, (u32)step);
}

// Appends one dump (step -1: the CFG, -2: the reduction record) to the run's pool.
OD_NOINL void dump_emit(KCtx &K, i32 step) {
    const DumpCfg &D = *K.in->dump;
    DotSink c{nullptr, 0};
    dump_print(K, c, step);
    // one reservation per executing lane group (k_front runs redundantly on
    // the warp): the leader reserves, every lane writes the same bytes
    const u32 m = wmask();
    u64 off = 0, ri = 0;
    if (wleader(m)) {
        off = fetch_add_u64(&D.top[0], c.n);
        ri = fetch_add_u64(&D.top[1], 1);
    }
    off = wbcast64(m, off);
    ri = wbcast64(m, ri);
    if (off + c.n > D.cap || ri >= D.rcap) {
        K.dump_full = true;
        return;
    }
    DotSink w{D.text + off, 0};
    dump_print(K, w, step);
    DumpRec &R = D.rec[ri];
    R.k = K.in->kidx;
    R.step = step;
    R.off = off;
    R.len = c.n;
}

OD_NOINL void reduce(KCtx &K) {
    const u32 n = region_rpo(K);
    K.ncand_w = n / 64 + 1;
    for (u32 w = 0; w < K.ncand_w; ++w)
        K.cand[w] = 0;
    for (u32 i = 0; i < n; ++i) {
        K.rank[K.rpo[i]] = i;
        K.at[i] = K.rpo[i];
        K.cand[i >> 6] |= 1ull << (i & 63);
    }
    const bool dump = K.in->dump && (K.in->dump->flags & DUMP_REGIONS);
    if (dump)
        dump_emit(K, 0);
    while (K.nlive > 1 && !K.oom) {
        u32 pos = kNoRank;
        for (u32 w = 0; w < K.ncand_w; ++w)
            if (K.cand[w]) {
                pos = w * 64 + ctz64(K.cand[w]);
                break;
            }
        if (pos == kNoRank)
            break; // no progress: residue
        const u32 r = K.at[pos];
        u32 m = match_if_else(K, r);
        if (!m)
            m = match_if(K, r);
        if (!m)
            m = match_linear(K, r);
        if (!m && !K.oom)
            K.cand[pos >> 6] &= ~(1ull << (pos & 63)); // fails until its neighbourhood changes
        if (m && dump)
            dump_emit(K, (i32)++K.nmerge);
    }
    K.reduced = K.nlive == 1;
    K.root_r = K.reduced ? (u32)K.entry_r : 0; // the one live region holds the entry
}

// ========================================================== liveness
// Per-block gen/kill accumulation (cfg.cpp:360-372): a use counts unless an
// earlier instruction of the block defined the register; an instruction's
// own defs are buffered and committed after it (use before def).
struct LvSink {
    u32 U[kLiveWords], D[kLiveWords]; // the block's gen / kill, accumulated locally
    u32 dd[kLiveWords];
    u32 touched;
};

OD_INL void lv_mark(LvSink &S, u32 id, bool is_def) {
    if (id >= kNumRegIds)
        return;
    const u32 w = id >> 5, bit = 1u << (id & 31);
    if (is_def) {
        S.dd[w] |= bit;
        S.touched |= 1u << w;
    } else if (!(S.D[w] & bit)) {
        S.U[w] |= bit;
    }
}

OD_INL void lv_commit(LvSink &S) {
    while (S.touched) {
        const u32 w = ctz32(S.touched);
        S.touched &= S.touched - 1;
        S.D[w] |= S.dd[w];
        S.dd[w] = 0;
    }
}

// add_operand_regs  cfg.cpp:230-265
OD_INL void add_operand_regs(const Opnd &op, LvSink &set, bool is_def) {
    switch (op.kind) {
    case OK_SREG:
        for (u32 i = 0; i < op.count && op.r.a + i < kNumRegIds; ++i)
            lv_mark(set, op.r.a + i, is_def);
        break;
    case OK_VREG:
        for (u32 i = 0; i < op.count && kRegIdVgpr0 + op.r.a + i < kNumRegIds; ++i)
            lv_mark(set, kRegIdVgpr0 + op.r.a + i, is_def);
        break;
    case OK_SPECIAL:
        switch (op.special) {
        case SP_EXEC:
            lv_mark(set, kRegIdExecLo, is_def);
            lv_mark(set, kRegIdExecHi, is_def);
            break;
        case SP_EXEC_LO: lv_mark(set, kRegIdExecLo, is_def); break;
        case SP_EXEC_HI: lv_mark(set, kRegIdExecHi, is_def); break;
        case SP_VCC:
            lv_mark(set, kRegIdVccLo, is_def);
            lv_mark(set, kRegIdVccHi, is_def);
            break;
        case SP_VCC_LO: lv_mark(set, kRegIdVccLo, is_def); break;
        case SP_VCC_HI: lv_mark(set, kRegIdVccHi, is_def); break;
        case SP_SCC: lv_mark(set, kRegIdScc, is_def); break;
        case SP_M0: lv_mark(set, kRegIdM0, is_def); break;
        }
        break;
    default:
        break;
    }
}

// instruction_use_def  cfg.cpp:272-352
OD_NOINL void instruction_use_def(const KCtx &K, const Ins &I, LvSink &S) {
    const Opnd *o = K.in->ops + I.op_start;
    const u32 n = (I.flags & IF_SYNTH) ? 0 : I.nops;
    if (I.flags & IF_PARSE_FAILED) {
        for (u32 k = 0; k < n; ++k)
            add_operand_regs(o[k], S, false);
        return;
    }
    const u32 root = I.root;
    const u32 px = I.prefix;
    if (px == PX_S && (root == R_WAITCNT || root == R_NOP || root == R_ENDPGM || root == R_BARRIER))
        return;
    if (px == PX_S && root == R_BRANCH)
        return;
    if (px == PX_S && (I.rflags & RF_CBRANCH)) {
        if (root == R_CBRANCH_SCC0 || root == R_CBRANCH_SCC1) {
            lv_mark(S, kRegIdScc, false);
        } else if (root == R_CBRANCH_VCCZ || root == R_CBRANCH_VCCNZ) {
            lv_mark(S, kRegIdVccLo, false);
            lv_mark(S, kRegIdVccHi, false);
        } else {
            lv_mark(S, kRegIdExecLo, false);
            lv_mark(S, kRegIdExecHi, false);
        }
        return;
    }
    if (px == PX_FLAT && (I.rflags & RF_STORE)) {
        for (u32 k = 0; k < n; ++k)
            add_operand_regs(o[k], S, false);
        return;
    }
    if (px == PX_S && (I.rflags & RF_CMP)) {
        for (u32 k = 0; k < n; ++k)
            add_operand_regs(o[k], S, false);
        lv_mark(S, kRegIdScc, true);
        return;
    }
    if (px == PX_S && root == R_AND_SAVEEXEC && n > 0) {
        add_operand_regs(o[0], S, true);
        for (u32 k = 1; k < n; ++k)
            add_operand_regs(o[k], S, false);
        lv_mark(S, kRegIdExecLo, false);
        lv_mark(S, kRegIdExecHi, false);
        lv_mark(S, kRegIdExecLo, true);
        lv_mark(S, kRegIdExecHi, true);
        return;
    }
    u32 ndefs = 1;
    if (px == PX_V && (root == R_ADD || root == R_SUB || root == R_SUBREV || root == R_ADDC) &&
        n >= 2 && (op_is_special(o[1], SP_VCC) || op_is_sreg_pair(o[1])))
        ndefs = 2;
    const bool reads_dst = (px == PX_S && (root == R_ADDK || root == R_MULK)) || (px == PX_V && root == R_MAC);
    for (u32 k = 0; k < n; ++k) {
        if (k < ndefs) {
            add_operand_regs(o[k], S, true);
            if (reads_dst && k == 0)
                add_operand_regs(o[k], S, false);
        } else {
            add_operand_regs(o[k], S, false);
        }
    }
    if (px == PX_S && n >= 1 &&
        (root == R_ADD || root == R_SUB || root == R_ADDK || root == R_MULK || root == R_AND ||
         root == R_OR || root == R_XOR || root == R_ANDN2 || root == R_LSHL || root == R_LSHR ||
         root == R_ASHR))
        lv_mark(S, kRegIdScc, true);
}

// live_in_sets  cfg.cpp:356-398, split across the warp (north star (4)):
// the per-block gen/kill sets are independent, one block per lane; the
// fixpoint is bitwise, so every live word converges on its own, one word per
// lane (the least fixpoint is unique: any order gives the reference's sets).
OD_NOINL bool liveness(KCtx &K) {
    const u32 nb = K.nblk;
    u32 *use = K.mem->get<u32>((u64)nb * kLiveWords);
    u32 *def = K.mem->get<u32>((u64)nb * kLiveWords);
    K.live_in = K.mem->get<u32>((u64)nb * kLiveWords);
    if (!use || !def || !K.live_in)
        return false;
    const u32 m = wmask(), r = wrank(m), nl = wsize(m);
    u32 any[kLiveWords]; // union of the use sets
    for (u32 w = 0; w < kLiveWords; ++w)
        any[w] = 0;
    LvSink S;
    for (u32 w = 0; w < kLiveWords; ++w)
        S.dd[w] = 0;
    S.touched = 0;
    const Block *__restrict__ blk = K.blk;
    const Ins *__restrict__ ins = K.ins;
    const u8 *__restrict__ supp = K.supp;
    u32 *__restrict__ live_in = K.live_in;
    for (u32 b = r; b < nb; b += nl) {
        for (u32 w = 0; w < kLiveWords; ++w) {
            S.U[w] = 0;
            S.D[w] = 0;
        }
        const u32 ib = blk[b].ib, ie = blk[b].ie;
        for (u32 i = ib; i < ie; ++i) {
            if (supp[i])
                continue;
            instruction_use_def(K, ins[i], S);
            lv_commit(S);
        }
        u32 *U = use + b * kLiveWords, *D = def + b * kLiveWords, *L = live_in + b * kLiveWords;
        for (u32 w = 0; w < kLiveWords; ++w) {
            U[w] = S.U[w];
            D[w] = S.D[w];
            L[w] = 0;
            any[w] |= S.U[w];
        }
    }
    for (u32 w = 0; w < kLiveWords; ++w)
        any[w] = wor(m, any[w]);
    wsync(m); // every lane sees every block's sets
    // Only words holding some use bit can ever become live (live_in is a
    // subset of the union of the use sets), so the fixpoint runs over those.
    u32 wl[kLiveWords];
    u32 nw = 0;
    for (u32 w = 0; w < kLiveWords; ++w)
        if (any[w])
            wl[nw++] = w;
    for (u32 k = r; k < nw; k += nl) {
        const u32 w = wl[k];
        bool changed = true;
        while (changed) {
            changed = false;
            for (u32 bi = nb; bi-- > 0;) {
                const u32 a0 = K.sx[2 * bi], a1 = K.sx[2 * bi + 1];
                u32 out = 0;
                if (a0 != kNoSucc)
                    out |= live_in[a0 * kLiveWords + w];
                if (a1 != kNoSucc)
                    out |= live_in[a1 * kLiveWords + w];
                const u32 in = use[bi * kLiveWords + w] | (out & ~def[bi * kLiveWords + w]);
                u32 &L = live_in[bi * kLiveWords + w];
                if (in != L) {
                    L = in;
                    changed = true;
                }
            }
        }
    }
    wsync(m); // the live sets are read by every lane from here on
    return true;
}

OD_INL bool lv_test(const u32 *set, u32 id) { return (set[id >> 5] >> (id & 31)) & 1; }

} // namespace od

#include "od_lower.cuh"
