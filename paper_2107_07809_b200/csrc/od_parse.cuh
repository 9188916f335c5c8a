// ocldec-b200: per-line front end (passes P1b-P1d).
//
// Line classification follows split_kernels/strip_comments/split_word
// (asm_frontend.cpp:26-75, 220-281); instruction decoding follows
// parse_text/parse_instruction/decompose_mnemonic/parse_operand/
// parse_register (asm_frontend.cpp:145-216, 375-521) and parse_type_suffix
// (type_recovery.cpp:50-73).  One thread decodes one line; the mnemonic root
// is resolved through a perfect hash over the dispatch set held in shared
// memory.
#pragma once

#include "od_base.cuh"

namespace od {

// ------------------------------------------------------------ line kinds
enum LineKind : u8 {
    LK_BLANK = 0,       // empty after comment strip + rtrim
    LK_KERNEL,          // ".kernel NAME"
    LK_KERNEL_NONAME,   // ".kernel" without a name: ParseError (asm_frontend.cpp:241)
    LK_DIR_CONFIG,      // ".config"
    LK_DIR_TEXT,        // ".text"
    LK_OTHER,           // anything else
};
// Role assigned by the section scan (split_kernels' mode machine).
enum LineRole : u8 { LR_NONE = 0, LR_CONFIG = 1, LR_TEXT = 2 };

// Per-line record produced by the front-end passes.
struct LineRec {
    u32 off;    // content offset (comment-stripped, right-trimmed; in aux for complex lines)
    u32 len;    // content length
    u8 kind;    // LineKind
    u8 role;    // LineRole
    u8 complex; // content needed /* */ removal and lives in the aux area
    u8 pad;
    u32 aux;    // scratch: materialized length for complex lines
};

// Decoded instruction line (parse_text + parse_instruction).
enum InsFlag : u8 { IF_HAS_INS = 1, IF_PARSE_FAILED = 2, IF_SYNTH = 4 };
struct LineIns {
    u32 src_off;   // Instruction::source_text
    u32 src_len;
    u32 op_start;  // first operand in the operand pool
    u32 lab_start; // first label in the label pool
    u16 root;      // Root
    u8 prefix;     // Prefix
    u8 rflags;     // RootFlag bits
    u16 nops;
    u16 nlabels;
    u8 flags;      // InsFlag
    u8 pad;
    u16 sfx[2];    // MnemonicParts::suffixes (0 = absent)
    u16 pad2;
};

struct Label {
    u32 off, len;
    u64 hash;
};

// ------------------------------------------------- comment strip / classify
// strip_comments (asm_frontend.cpp:44-66).  Returns the cut position for
// the simple case; *complex is set when a terminated /* */ must be removed
// from the middle (the content is then not a single span).
OD_NOINL u32 strip_scan(const u8 *p, u32 n, bool *complex) {
    bool inq = false;
    *complex = false;
    for (u32 i = 0; i < n; ++i) {
        u8 c = p[i];
        if (c == '"')
            inq = !inq;
        if (!inq) {
            if (c == '#' || c == ';')
                return i;
            if (c == '/' && i + 1 < n && p[i + 1] == '*') {
                // line.find("*/", i + 2)
                u32 close = n;
                for (u32 j = i + 2; j + 1 < n; ++j)
                    if (p[j] == '*' && p[j + 1] == '/') {
                        close = j;
                        break;
                    }
                if (close == n)
                    return i; // unterminated: drop the rest of the line
                *complex = true;
                i = close + 1;
                continue;
            }
        }
    }
    return n;
}

// Materializes strip_comments(line) into out (when non-null); returns length.
OD_NOINL u32 strip_materialize(const u8 *p, u32 n, u8 *out) {
    bool inq = false;
    u32 k = 0;
    for (u32 i = 0; i < n; ++i) {
        u8 c = p[i];
        if (c == '"')
            inq = !inq;
        if (!inq) {
            if (c == '#' || c == ';')
                break;
            if (c == '/' && i + 1 < n && p[i + 1] == '*') {
                u32 close = n;
                for (u32 j = i + 2; j + 1 < n; ++j)
                    if (p[j] == '*' && p[j + 1] == '/') {
                        close = j;
                        break;
                    }
                if (close == n)
                    break;
                i = close + 1;
                continue;
            }
        }
        if (out)
            out[k] = c;
        ++k;
    }
    return k;
}

OD_INL u32 rtrim_len(const u8 *p, u32 n) {
    while (n > 0 && c_space(p[n - 1]))
        --n;
    return n;
}

// split_word: first whitespace-delimited word of s (after ltrim).
OD_INL void split_word(const u8 *t, Span s, Span *word, Span *rest) {
    u32 b = s.off, e = s.off + s.len;
    while (b < e && c_space(t[b]))
        ++b;
    u32 w = b;
    while (w < e && !c_space(t[w]))
        ++w;
    word->off = b;
    word->len = w - b;
    u32 r = w;
    while (r < e && c_space(t[r]))
        ++r;
    rest->off = r;
    rest->len = e - r;
}

// Kind of a non-blank content line (split_kernels' first-word dispatch,
// asm_frontend.cpp:235-262).
OD_NOINL u8 classify_content(const u8 *t, Span c) {
    if (c.len == 0)
        return LK_BLANK;
    Span w, rest;
    split_word(t, c, &w, &rest);
    if (span_eq(t, w, ".kernel")) {
        Span name, extra;
        split_word(t, rest, &name, &extra);
        return name.len ? LK_KERNEL : LK_KERNEL_NONAME;
    }
    if (span_eq(t, w, ".config"))
        return LK_DIR_CONFIG;
    if (span_eq(t, w, ".text"))
        return LK_DIR_TEXT;
    return LK_OTHER;
}

// ------------------------------------------------------ mnemonic decoding
struct RootTable {
    u16 slot[128];      // perfect-hash slot -> Root id (0 = empty)
    char str[R_COUNT][16]; // root strings for verification
};

#define OD_ROOT_HASH_SEED 3731u

OD_INL u32 root_hash_slot(const u8 *p, u32 n) {
    u32 h = 2166136261u;
    for (u32 i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 16777619u;
    }
    return (h * OD_ROOT_HASH_SEED) >> 25;
}

// Fills the perfect-hash table (host or device; 128 slots, collision-free
// for the dispatch set by construction of the seed).
OD_NOINL void build_root_table(RootTable *rt) {
    const char *names[R_COUNT] = {OD_ROOT_STRINGS};
    for (u32 i = 0; i < 128; ++i)
        rt->slot[i] = 0;
    for (u32 i = 0; i < R_COUNT; ++i) {
        u32 n = 0;
        while (names[i][n]) {
            rt->str[i][n] = names[i][n];
            ++n;
        }
        for (u32 k = n; k < 16; ++k)
            rt->str[i][k] = 0;
        if (i)
            rt->slot[root_hash_slot((const u8 *)names[i], n)] = (u16)i;
    }
}

// parse_type_suffix  type_recovery.cpp:50-73
OD_INL u32 parse_sfx(const u8 *p, u32 n) {
    if (n < 2 || n > 3)
        return 0;
    u32 b;
    switch (p[0]) {
    case 'i': b = SB_I; break;
    case 'u': b = SB_U; break;
    case 'f': b = SB_F; break;
    case 'b': b = SB_B; break;
    default: return 0;
    }
    u32 w = 0;
    for (u32 i = 1; i < n; ++i) {
        if (!c_digit(p[i]))
            return 0;
        w = w * 10 + (p[i] - '0');
    }
    if (w == 8 || w == 16 || w == 24 || w == 32 || w == 64)
        return (b << 8) | w;
    return 0;
}

OD_INL bool starts_with(const u8 *p, u32 n, const char *lit) {
    u32 i = 0;
    for (; lit[i]; ++i)
        if (i >= n || p[i] != (u8)lit[i])
            return false;
    return true;
}

struct Mnem {
    u8 prefix;
    u8 rflags;
    u16 root;
    u16 sfx[2];
};

// decompose_mnemonic  asm_frontend.cpp:375-423
OD_NOINL Mnem decompose(const u8 *t, Span m, const RootTable *rt) {
    Mnem r;
    r.prefix = PX_OTHER;
    r.rflags = 0;
    r.root = R_UNKNOWN;
    r.sfx[0] = r.sfx[1] = 0;
    const u8 *p = t + m.off;
    u32 n = m.len;
    // one pass over the word: the first '_' (prefix end), the number of '_'
    // after it, and the last two of those (suffix token boundaries)
    u32 us = n, nus = 0;
    i32 u1 = -1, u2 = -1;
    for (u32 i = 0; i < n; ++i) {
        if (p[i] != '_')
            continue;
        if (us == n) {
            us = i;
        } else {
            ++nus;
            u2 = u1;
            u1 = (i32)i;
        }
    }
    if (us == n)
        return r;
    u8 px = PX_OTHER;
    if (us == 1 && p[0] == 's')
        px = PX_S;
    else if (us == 1 && p[0] == 'v')
        px = PX_V;
    else if (us == 2 && p[0] == 'd' && p[1] == 's')
        px = PX_DS;
    else if (us == 4 && p[0] == 'f' && p[1] == 'l' && p[2] == 'a' && p[3] == 't')
        px = PX_FLAT;
    if (px == PX_OTHER)
        return r;
    r.prefix = px;
    const u8 *rest = p + us + 1;
    const u32 rn = n - us - 1;
    // tokens of rest split on '_' (an empty rest has none); peel at most two
    // suffix tokens off the tail keeping >= 1 token
    const u32 ntok = rn > 0 ? nus + 1 : 0;
    const i32 off = (i32)us + 1; // rest-relative '_' positions: u - off
    u32 root_len = rn;
    u32 npeel = 0;
    u32 peeled[2];
    if (ntok > 1) {
        const u32 s1 = (u32)(u1 - off) + 1;
        const u32 sf = parse_sfx(rest + s1, root_len - s1);
        if (sf) {
            peeled[npeel++] = sf;
            root_len = s1 - 1;
            if (ntok > 2) {
                const u32 s2 = (u32)(u2 - off) + 1;
                const u32 sf2 = parse_sfx(rest + s2, root_len - s2);
                if (sf2) {
                    peeled[npeel++] = sf2;
                    root_len = s2 - 1;
                }
            }
        }
    }
    if (npeel == 1)
        r.sfx[0] = (u16)peeled[0];
    else if (npeel == 2) {
        r.sfx[0] = (u16)peeled[1];
        r.sfx[1] = (u16)peeled[0];
    }
    if (ntok == 0)
        root_len = 0;
    // root flags (rfind(x, 0) == 0 tests)
    // (the five prefixes differ in their first byte or, for c, the second)
    switch (root_len ? rest[0] : 0) {
    case 'c':
        if (starts_with(rest, root_len, "cbranch_"))
            r.rflags |= RF_CBRANCH;
        else if (starts_with(rest, root_len, "cmp_"))
            r.rflags |= RF_CMP;
        break;
    case 's':
        if (starts_with(rest, root_len, "store"))
            r.rflags |= RF_STORE;
        break;
    case 'l':
        if (starts_with(rest, root_len, "lshr"))
            r.rflags |= RF_LSHR;
        break;
    case 'a':
        if (starts_with(rest, root_len, "ashr"))
            r.rflags |= RF_ASHR;
        break;
    default: break;
    }
    // perfect-hash lookup + verification
    u32 slot = root_hash_slot(rest, root_len);
    u16 id = rt->slot[slot];
    if (id) {
        const char *s = rt->str[id];
        u32 i = 0;
        bool eq = true;
        for (; i < root_len; ++i)
            if (s[i] == 0 || (u8)s[i] != rest[i]) {
                eq = false;
                break;
            }
        if (eq && s[i] == 0)
            r.root = id;
    }
    return r;
}

// ------------------------------------------------------- operand parsing
// Result of one token: 0 ok, else the operand ParseError the reference throws
// (asm_frontend.cpp:159-183): 1 unbalanced bracket, 2 range without ':',
// 3 bad range, 4 negative index, 5 beyond the register file.
OD_NOINL int parse_register(const u8 *t, Span tok, Opnd *op, bool *is_reg) {
    *is_reg = false;
    const u8 *p = t + tok.off;
    u32 n = tok.len;
    if (n < 2 || (p[0] != 's' && p[0] != 'v'))
        return 0;
    const bool scalar = p[0] == 's';
    const u32 limit = scalar ? 104u : 256u;
    u32 first, count;
    const u8 *rest = p + 1;
    u32 rn = n - 1;
    if (rest[0] == '[') {
        if (rest[rn - 1] != ']')
            return 1; // unbalanced bracket
        // rest.substr(1, size-2): for "[" alone size-2 underflows -> npos
        // semantics give the whole tail; n>=2 and rest[0]=='[' and
        // rest.back()==']' means rn>=1; rn==1 is "[" == "]" impossible.
        const u8 *in = rest + 1;
        u32 inn = rn >= 2 ? rn - 2 : 0;
        u32 colon = 0;
        while (colon < inn && in[colon] != ':')
            ++colon;
        if (colon == inn)
            return 2; // no ':'
        i64 lo, hi;
        bool okl = parse_int(in, colon, &lo);
        bool okh = parse_int(in + colon + 1, inn - colon - 1, &hi);
        if (!okl || !okh || lo < 0 || hi < lo)
            return 3; // bad range
        first = (u32)lo;
        count = (u32)(hi - lo + 1);
    } else {
        i64 idx;
        if (!parse_int(rest, rn, &idx))
            return 0; // "saveexec" and other identifiers
        if (idx < 0)
            return 4; // negative index
        first = (u32)idx;
        count = 1;
    }
    if ((u32)(first + count) > limit)
        return 5; // exceeds the register file
    op->kind = scalar ? OK_SREG : OK_VREG;
    op->special = 0;
    op->count = count;
    op->r.a = first;
    op->r.b = 0;
    *is_reg = true;
    return 0;
}

// parse_operand  asm_frontend.cpp:188-216
OD_NOINL int parse_operand(const u8 *t, Span tok, Opnd *op) {
    const u8 *p = t + tok.off;
    u32 n = tok.len;
    int sp = -1;
    if (n == 4 && p[0] == 'e' && p[1] == 'x' && p[2] == 'e' && p[3] == 'c')
        sp = SP_EXEC;
    else if (n == 3 && p[0] == 'v' && p[1] == 'c' && p[2] == 'c')
        sp = SP_VCC;
    else if (n == 3 && p[0] == 's' && p[1] == 'c' && p[2] == 'c')
        sp = SP_SCC;
    else if (n == 2 && p[0] == 'm' && p[1] == '0')
        sp = SP_M0;
    else if (n == 7 && p[0] == 'e' && p[1] == 'x' && p[2] == 'e' && p[3] == 'c' && p[4] == '_' &&
             p[5] == 'l' && p[6] == 'o')
        sp = SP_EXEC_LO;
    else if (n == 7 && p[0] == 'e' && p[1] == 'x' && p[2] == 'e' && p[3] == 'c' && p[4] == '_' &&
             p[5] == 'h' && p[6] == 'i')
        sp = SP_EXEC_HI;
    else if (n == 6 && p[0] == 'v' && p[1] == 'c' && p[2] == 'c' && p[3] == '_' && p[4] == 'l' &&
             p[5] == 'o')
        sp = SP_VCC_LO;
    else if (n == 6 && p[0] == 'v' && p[1] == 'c' && p[2] == 'c' && p[3] == '_' && p[4] == 'h' &&
             p[5] == 'i')
        sp = SP_VCC_HI;
    if (sp >= 0) {
        op->kind = OK_SPECIAL;
        op->special = (u8)sp;
        op->count = (sp == SP_EXEC || sp == SP_VCC) ? 2 : 1;
        op->value = 0;
        return 0;
    }
    bool is_reg;
    if (int err = parse_register(t, tok, op, &is_reg))
        return err;
    if (is_reg)
        return 0;
    i64 v;
    if (parse_int(p, n, &v)) {
        op->kind = OK_LITERAL;
        op->special = 0;
        op->count = 1;
        op->value = v;
        return 0;
    }
    bool plain = n > 0 && c_ident_start(p[0]);
    for (u32 i = 0; plain && i < n; ++i)
        if (!c_ident_char(p[i]))
            plain = false;
    op->kind = plain ? OK_SYMBOL : OK_ANNOT;
    op->special = 0;
    op->count = 1;
    op->r.a = tok.off;
    op->r.b = tok.len;
    return 0;
}

// Decodes one text line: label peeling (parse_text, asm_frontend.cpp:486-521)
// plus parse_instruction (:439-484).  When ops/labs are null only the
// counts are produced (sizing pass).  Returns 1 when an operand ParseError
// demoted the instruction to parse_failed.
OD_NOINL int decode_line(const u8 *t, Span content, const RootTable *rt, LineIns *out, Opnd *ops,
                         u32 ops_cap, Label *labs) {
    u32 b = content.off, e = content.off + content.len;
    while (b < e && c_space(t[b]))
        ++b;
    u32 nlab = 0;
    while (b < e && c_ident_start(t[b])) {
        u32 x = b;
        while (x < e && c_ident_char(t[x]))
            ++x;
        if (x >= e || t[x] != ':')
            break;
        if (labs) {
            labs[nlab].off = b;
            labs[nlab].len = x - b;
            labs[nlab].hash = fnv1a64(t + b, x - b);
        }
        ++nlab;
        b = x + 1;
        while (b < e && c_space(t[b]))
            ++b;
    }
    out->nlabels = (u16)(nlab > 65535 ? 65535 : nlab);
    out->flags = 0;
    out->nops = 0;
    out->root = R_UNKNOWN;
    out->prefix = PX_OTHER;
    out->rflags = 0;
    out->sfx[0] = out->sfx[1] = 0;
    out->src_off = b;
    out->src_len = e - b; // content is right-trimmed already
    if (b == e)
        return 0; // label-only line
    out->flags = IF_HAS_INS;
    Span src = {b, e - b};
    Span word, rest;
    split_word(t, src, &word, &rest);
    Mnem m = decompose(t, word, rt);
    out->prefix = m.prefix;
    out->rflags = m.rflags;
    out->root = m.root;
    out->sfx[0] = m.sfx[0];
    out->sfx[1] = m.sfx[1];

    if (span_eq(t, word, "s_waitcnt")) {
        if (rest.len) {
            if (ops && ops_cap > 0) {
                ops[0].kind = OK_ANNOT;
                ops[0].special = 0;
                ops[0].count = 1;
                ops[0].r.a = rest.off;
                ops[0].r.b = rest.len;
            }
            out->nops = 1;
        }
        return 0;
    }
    // split_fields (asm_frontend.cpp:80-107) + per-field split_word tokens.
    u32 nops = 0;
    int depth = 0;
    bool inq = false;
    u32 fstart = rest.off;
    const u32 rend = rest.off + rest.len;
    for (u32 i = rest.off; i <= rend; ++i) {
        bool cut = false;
        if (i == rend) {
            cut = true;
        } else {
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
        // field [fstart, i): trim, then split into tokens
        u32 fb = fstart, fe = i;
        while (fb < fe && c_space(t[fb]))
            ++fb;
        while (fe > fb && c_space(t[fe - 1]))
            --fe;
        bool first_tok = true;
        u32 q = fb;
        while (q < fe) {
            u32 te = q;
            while (te < fe && !c_space(t[te]))
                ++te;
            Span tok = {q, te - q};
            Opnd tmp;
            if (int err = parse_operand(t, tok, &tmp)) {
                // the failing token goes to the line's first operand slot
                // (diagnostics); the instruction itself has no operands
                if (ops && ops_cap > 0) {
                    ops[0].kind = OK_ANNOT;
                    ops[0].special = (u8)err;
                    ops[0].pad = 0;
                    ops[0].count = 1;
                    ops[0].r.a = tok.off;
                    ops[0].r.b = tok.len;
                }
                out->flags |= IF_PARSE_FAILED;
                out->prefix = PX_OTHER;
                out->rflags = 0;
                out->root = R_UNKNOWN;
                out->sfx[0] = out->sfx[1] = 0;
                out->nops = 0;
                return 1;
            }
            if (!first_tok && tmp.kind == OK_SYMBOL)
                tmp.kind = OK_ANNOT;
            if (ops && nops < ops_cap) // a later ParseError leaves the sized slot empty
                ops[nops] = tmp;
            ++nops;
            first_tok = false;
            q = te;
            while (q < fe && c_space(t[q]))
                ++q;
        }
        fstart = i + 1;
    }
    out->nops = (u16)nops;
    return 0;
}

} // namespace od
