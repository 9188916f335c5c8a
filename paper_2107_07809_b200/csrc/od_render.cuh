// ocldec-b200: builtin folds (builtin_detector.cpp) and the streaming
// OpenCL renderer (codegen.cpp, type_recovery.cpp:171-212).
#pragma once

#include "od_expr.cuh"

namespace od {

struct KArg {
    Span name;     // raw name (signature)
    DT type;
    u32 name_id;   // canonical id of the sanitized name ('.' -> '_')
    u8 implicit;
    u8 pad[3];
};

struct KConfig {
    Span name;
    u32 dims;
    u32 cws[3];
    u32 useargs;
    KArg *args;
    u32 nargs;
    u32 fold_local_size;
};

struct FoldScratch {
    U32Stack st;    // traversal stack
    U32Stack terms; // collected add terms
};

// match_builtin  builtin_detector.cpp:22-29
OD_INL bool match_builtin(const EArena &E, u32 e, u32 fn, u32 dim) {
    while (e && E.n[e].kind == E_UNARY && (E.n[e].op == U_LO32 || E.n[e].op == U_CAST))
        e = E.n[e].a;
    return e && E.n[e].kind == E_BUILTIN && E.n[e].op == fn && E.n[e].x == dim;
}

OD_INL bool is_const_value(const EArena &E, u32 e, u64 v) {
    return e && E.n[e].kind == E_CONST && (E.cval(e) & 0xffffffffu) == (v & 0xffffffffu);
}

OD_INL u32 cfg_local_size(const KConfig &c, int dim) {
    if (dim < 0 || dim > 2)
        return 1;
    return c.cws[dim];
}

// match_group_product  builtin_detector.cpp:39-59
OD_NOINL bool match_group_product(const EArena &E, u32 e, const KConfig &cfg, u32 dim) {
    u32 cws = cfg_local_size(cfg, (int)dim);
    if (cws == 1 && match_builtin(E, e, F_GROUP_ID, dim))
        return true;
    if (!e || E.n[e].kind != E_BINARY)
        return false;
    const ENode &x = E.n[e];
    if (x.op == O_SHL) {
        return match_builtin(E, x.a, F_GROUP_ID, dim) && x.b && E.n[x.b].kind == E_CONST &&
               E.cval(x.b) < 32 && (1u << E.cval(x.b)) == cws;
    }
    if (x.op != O_MUL)
        return false;
    bool fa = is_const_value(E, x.b, cws) || match_builtin(E, x.b, F_LOCAL_SIZE, dim);
    if (match_builtin(E, x.a, F_GROUP_ID, dim) && fa)
        return true;
    bool fb = is_const_value(E, x.a, cws) || match_builtin(E, x.a, F_LOCAL_SIZE, dim);
    if (match_builtin(E, x.b, F_GROUP_ID, dim) && fb)
        return true;
    return false;
}

// fold_global_id  builtin_detector.cpp:86-124
OD_NOINL u32 fold_global_id(EArena &E, u32 e, const KConfig &cfg, FoldScratch &s) {
    if (!e || E.n[e].kind != E_BINARY || E.n[e].op != O_ADD || dt_bits(E.n[e].type) != 32)
        return 0;
    u32 tb = s.terms.top;
    collect_add_terms(E, e, s.st, s.terms);
    u32 nt = s.terms.top - tb;
    u32 *terms = s.terms.p + tb;
    u32 result = 0;
    if (nt >= 2 && !s.terms.oom) {
        for (u32 dim = 0; dim < cfg.dims && !result; ++dim) {
            int product = -1, local = -1, offset = -1;
            for (u32 i = 0; i < nt; ++i) {
                if (product < 0 && match_group_product(E, terms[i], cfg, dim))
                    product = (int)i;
                else if (local < 0 && match_builtin(E, terms[i], F_LOCAL_ID, dim))
                    local = (int)i;
                else if (offset < 0 && match_builtin(E, terms[i], F_GLOBAL_OFFSET, dim))
                    offset = (int)i;
            }
            if (product < 0 || local < 0)
                continue;
            u32 gid = E.builtin(F_GLOBAL_ID, dim, DT_U32);
            u32 core = offset >= 0
                           ? gid
                           : E.binary(O_SUB, gid, E.builtin(F_GLOBAL_OFFSET, dim, DT_U32), DT_U32);
            DT t = E.n[e].type;
            u32 sum = core;
            for (u32 i = 0; i < nt; ++i)
                if ((int)i != product && (int)i != local && (int)i != offset)
                    sum = sum ? E.binary(O_ADD, sum, terms[i], t) : terms[i];
            result = sum;
        }
    }
    s.terms.top = tb;
    return result;
}

// fold_num_groups  builtin_detector.cpp:126-143
OD_NOINL u32 fold_num_groups(EArena &E, u32 e, const KConfig &cfg) {
    if (!e || E.n[e].kind != E_BINARY)
        return 0;
    const ENode x = E.n[e];
    for (u32 dim = 0; dim < cfg.dims; ++dim) {
        if (!match_builtin(E, x.a, F_GLOBAL_SIZE, dim))
            continue;
        u32 cws = cfg_local_size(cfg, (int)dim);
        bool hit = false;
        if (x.op == O_DIV && is_const_value(E, x.b, cws))
            hit = true;
        else if (x.op == O_LSHR && x.b && E.n[x.b].kind == E_CONST && E.cval(x.b) < 32 &&
                 (1u << E.cval(x.b)) == cws)
            hit = true;
        if (hit)
            return E.builtin(F_NUM_GROUPS, dim, DT_U32);
    }
    return 0;
}

// fold_local_size  builtin_detector.cpp:145-169
OD_NOINL u32 fold_local_size(EArena &E, u32 e, const KConfig &cfg) {
    if (!e || E.n[e].kind != E_BINARY || E.n[e].op != O_MUL)
        return 0;
    const ENode x = E.n[e];
    for (u32 dim = 0; dim < cfg.dims; ++dim) {
        u32 cws = cfg_local_size(cfg, (int)dim);
        if (cws == 1)
            continue;
        u32 group, other;
        if (match_builtin(E, x.a, F_GROUP_ID, dim)) {
            group = x.a;
            other = x.b;
        } else if (match_builtin(E, x.b, F_GROUP_ID, dim)) {
            group = x.b;
            other = x.a;
        } else {
            continue;
        }
        if (is_const_value(E, other, cws))
            return E.binary(O_MUL, group, E.builtin(F_LOCAL_SIZE, dim, DT_U32), x.type);
    }
    return 0;
}

enum : u32 { kMemoNull = 0xffffffffu };

// fold_expr  builtin_detector.cpp:171-209.  Pure in its argument, so the
// result is memoized per node (the reference re-walks shared sub-DAGs).
OD_NOINL u32 fold_expr(EArena &E, u32 root, const KConfig &cfg, FoldScratch &s) {
    if (!root)
        return 0;
    if (E.n[root].memo)
        return E.n[root].memo == kMemoNull ? 0 : E.n[root].memo;
    U32Stack &st = s.st;
    u32 base = st.top;
    st.push(root);
    while (st.top > base && !st.oom && !E.oom) {
        u32 e = st.p[st.top - 1];
        const ENode &x = E.n[e];
        if (x.memo) {
            st.top--;
            continue;
        }
        // children first
        u32 ch[3] = {0, 0, 0};
        u32 nch = 0;
        if (x.kind == E_UNARY || x.kind == E_DEREF) {
            ch[0] = x.a;
            nch = 1;
        } else if (x.kind == E_BINARY) {
            ch[0] = x.a;
            ch[1] = x.b;
            nch = 2;
        } else if (x.kind == E_TERNARY) {
            ch[0] = x.a;
            ch[1] = x.b;
            ch[2] = x.c;
            nch = 3;
        }
        bool pending = false;
        for (u32 k = 0; k < nch; ++k)
            if (ch[k] && !E.n[ch[k]].memo) {
                st.push(ch[k]);
                pending = true;
            }
        if (pending)
            continue;
        st.top--;
        u32 f[3];
        for (u32 k = 0; k < 3; ++k)
            f[k] = ch[k] ? (E.n[ch[k]].memo == kMemoNull ? 0 : E.n[ch[k]].memo) : 0;
        u32 cur = e;
        const ENode xe = E.n[e];
        if ((nch >= 1 && f[0] != ch[0]) || (nch >= 2 && f[1] != ch[1]) ||
            (nch >= 3 && f[2] != ch[2])) {
            switch (xe.kind) {
            case E_UNARY: cur = E.unary(xe.op, f[0], xe.type); break;
            case E_BINARY: cur = E.binary(xe.op, f[0], f[1], xe.type); break;
            case E_TERNARY: cur = E.ternary(f[0], f[1], f[2], xe.type); break;
            case E_DEREF: cur = E.deref(f[0], xe.type, dt_space(xe.type)); break;
            default: break;
            }
        }
        for (;;) {
            u32 next = fold_global_id(E, cur, cfg, s);
            if (!next)
                next = fold_num_groups(E, cur, cfg);
            if (!next && cfg.fold_local_size)
                next = fold_local_size(E, cur, cfg);
            if (!next)
                break;
            cur = next;
        }
        E.n[e].memo = cur ? cur : kMemoNull;
    }
    st.top = base;
    return E.n[root].memo == kMemoNull ? 0 : E.n[root].memo;
}

// ------------------------------------------------------------- rendering
// render_type  type_recovery.cpp:171-212
OD_INL void render_scalar_type(Writer &w, DT t) {
    u32 bits = dt_bits(t) == 24 ? 32 : dt_bits(t);
    u32 base = dt_base(t);
    if (base == B_BINARY || base == B_UNKNOWN)
        base = B_UNSIGNED;
    switch (base) {
    case B_VOID: w.lit("void"); return;
    case B_FLOAT: w.puts(bits == 64 ? "double" : "float"); return;
    case B_SIGNED:
        w.puts(bits == 8 ? "char" : bits == 16 ? "short" : bits == 64 ? "long" : "int");
        return;
    default:
        w.puts(bits == 8 ? "uchar" : bits == 16 ? "ushort" : bits == 64 ? "ulong" : "uint");
        return;
    }
}

OD_INL void render_space_prefix(Writer &w, u32 space) {
    switch (space) {
    case AS_GLOBAL: w.lit("__global "); break;
    case AS_LOCAL: w.lit("__local "); break;
    case AS_CONSTANT: w.lit("__constant "); break;
    case AS_PRIVATE: w.lit("__private "); break;
    default: break;
    }
}

// Pointer types recurse on pointee(): each level prints the space prefix,
// then the pointee, ' ', and its own depth in stars.
OD_NOINL void render_type(Writer &w, DT t) {
    u32 d = dt_depth(t);
    if (d == 0) {
        render_scalar_type(w, t);
        return;
    }
    // levels d, d-1, ..., 1: prefixes outermost first
    DT cur = t;
    for (u32 k = d; k >= 1; --k) {
        render_space_prefix(w, dt_space(cur));
        cur = dt_pointee(cur);
    }
    render_scalar_type(w, cur);
    for (u32 k = 1; k <= d; ++k) {
        w.put(' ');
        for (u32 s = 0; s < k; ++s)
            w.put('*');
    }
}

// render_type(...) ends in '*' iff it is a pointer.
OD_INL bool type_ends_star(DT t) { return dt_depth(t) > 0; }

OD_INL const char *builtin_name(u32 fn) {
    switch (fn) {
    case F_GLOBAL_ID: return "get_global_id";
    case F_LOCAL_ID: return "get_local_id";
    case F_GROUP_ID: return "get_group_id";
    case F_GLOBAL_SIZE: return "get_global_size";
    case F_LOCAL_SIZE: return "get_local_size";
    case F_NUM_GROUPS: return "get_num_groups";
    case F_GLOBAL_OFFSET: return "get_global_offset";
    default: return "get_work_dim";
    }
}

// register name class (physical slot) -> reg_id_name
OD_INL void put_reg_name(Writer &w, u32 cls) {
    if (cls < 104) {
        w.put('s');
        w.put_u64(cls);
    } else if (cls < 360) {
        w.put('v');
        w.put_u64(cls - 104);
    } else if (cls == 360) {
        w.lit("exec");
    } else if (cls == 361) {
        w.lit("vcc");
    } else if (cls == 362) {
        w.lit("scc");
    } else {
        w.lit("m0");
    }
}

OD_INL void put_var_name(Writer &w, u32 cls, u32 num) {
    put_reg_name(w, cls);
    w.put('_');
    w.put_u64(num);
}

// render_const  codegen.cpp:106-136
OD_NOINL void render_const(Writer &w, const EArena &E, u32 e) {
    DT t = E.n[e].type;
    u64 v = E.cval(e);
    if (dt_is_float(t) && dt_bits(t) == 32) {
        u32 bits = (u32)v;
        float f;
        memcpy(&f, &bits, 4);
        if (isfinite(f) && f == floorf(f) && fabsf(f) < 1e6f) {
            w.put_i64((long long)f);
            w.lit(".0f");
            return;
        }
        w.lit("as_float(0x");
        w.put_hex(bits);
        w.lit("u)");
        return;
    }
    if (dt_is_signed(t) && dt_bits(t) == 32 && (v >> 31) == 1) {
        w.put_i64((i64)(i32)(u32)v);
        return;
    }
    if (v < 4096) {
        w.put_u64(v);
    } else {
        w.lit("0x");
        w.put_hex(v);
    }
    if (dt_bits(t) == 64 && v > 0xffffffffull)
        w.lit("ul");
}

enum { kPrimary = 16, kUnary = 14 };

OD_INL int binop_prec(u32 op) {
    switch (op) {
    case O_MUL:
    case O_DIV: return 13;
    case O_ADD:
    case O_SUB: return 12;
    case O_SHL:
    case O_LSHR:
    case O_ASHR: return 11;
    case O_CMPLT:
    case O_CMPLE:
    case O_CMPGT:
    case O_CMPGE:
    case O_CMPLTU:
    case O_CMPLEU:
    case O_CMPGTU:
    case O_CMPGEU: return 9;
    case O_CMPEQ:
    case O_CMPNE: return 8;
    case O_AND: return 7;
    case O_XOR: return 6;
    case O_OR: return 5;
    default: return kPrimary;
    }
}

OD_INL const char *binop_text(u32 op) {
    switch (op) {
    case O_ADD: return " + ";
    case O_SUB: return " - ";
    case O_MUL: return " * ";
    case O_DIV: return " / ";
    case O_AND: return " & ";
    case O_OR: return " | ";
    case O_XOR: return " ^ ";
    case O_SHL: return " << ";
    case O_LSHR:
    case O_ASHR: return " >> ";
    case O_CMPEQ: return " == ";
    case O_CMPNE: return " != ";
    case O_CMPLT:
    case O_CMPLTU: return " < ";
    case O_CMPLE:
    case O_CMPLEU: return " <= ";
    case O_CMPGT:
    case O_CMPGTU: return " > ";
    case O_CMPGE:
    case O_CMPGEU: return " >= ";
    default: return " ? ";
    }
}

OD_INL bool op_wants_unsigned(u32 op) {
    return op == O_CMPLTU || op == O_CMPLEU || op == O_CMPGTU || op == O_CMPGEU ||
           op == O_LSHR || op == O_MULHI;
}
OD_INL bool op_wants_signed(u32 op) {
    return op == O_CMPLT || op == O_CMPLE || op == O_CMPGT || op == O_CMPGE || op == O_ASHR ||
           op == O_MULHIS;
}

// is_bit_reinterpret  codegen.cpp:158-161
OD_INL bool is_bit_reinterpret(DT from, DT to) {
    return dt_bits(from) == dt_bits(to) && dt_is_float(from) != dt_is_float(to) &&
           !dt_is_pointer(from) && !dt_is_pointer(to);
}

// cast_name  codegen.cpp:163-167
OD_INL const char *cast_name(DT to) {
    if (dt_is_float(to))
        return dt_bits(to) == 64 ? "as_double" : "as_float";
    return dt_bits(to) == 64 ? "as_ulong" : (dt_is_signed(to) ? "as_int" : "as_uint");
}

// Render tasks (explicit stack, 64-bit entries: kind | arg<<8 | node<<32).
enum RTask : u32 { RT_NODE = 0, RT_SA, RT_CHAR, RT_STR, RT_NAME };
enum RStr : u32 { S_COMMA = 0, S_SHR32, S_QMARK, S_COLON, S_BINOP_BASE = 16 };

OD_INL const char *rstr(u32 id) {
    switch (id) {
    case S_COMMA: return ", ";
    case S_SHR32: return " >> 32)";
    case S_QMARK: return " ? ";
    case S_COLON: return " : ";
    default: return binop_text(id - S_BINOP_BASE);
    }
}

struct TaskStack {
    u64 *p;
    u32 top, cap, hw;
    bool oom;
    OD_INL void push(u32 kind, u32 arg, u32 node) {
        if (top < cap) {
            p[top++] = (u64)kind | ((u64)arg << 8) | ((u64)node << 32);
            if (top > hw)
                hw = top;
        } else {
            oom = true;
        }
    }
};

struct RenderCtx {
    EArena *E;
    const KConfig *cfg;
    const u8 *text;       // listing bytes (argument names)
    const Span *arg_sname; // sanitized-name id -> raw span (print with '.'->'_')
    TaskStack ts;
    FoldScratch fs;       // term scratch for render_indexed
};

OD_INL void put_arg_name(Writer &w, const RenderCtx &rc, u32 name_id) {
    Span s = rc.arg_sname[name_id];
    for (u32 i = 0; i < s.len; ++i) {
        u8 c = rc.text[s.off + i];
        w.put(c == '.' ? '_' : c);
    }
}

OD_INL const ENode *strip_casts(const EArena &E, u32 &e) {
    while (e && E.n[e].kind == E_UNARY && E.n[e].op == U_CAST)
        e = E.n[e].a;
    return e ? &E.n[e] : nullptr;
}

// unscale_term  codegen.cpp:172-192 (allocates scratch nodes)
OD_INL u32 unscale_term(EArena &E, u32 term, u32 size) {
    if (size == 1)
        return term;
    // A Cast returns its inner result when that succeeds; a Cast node itself
    // is neither const nor binary, so otherwise the level fails.  Hence the
    // answer is the one for the innermost non-Cast node of the chain (or a
    // Cast with a null operand, which fails).
    u32 cur = term;
    while (cur && E.n[cur].kind == E_UNARY && E.n[cur].op == U_CAST && E.n[cur].a)
        cur = E.n[cur].a;
    if (!cur)
        return 0;
    const ENode x = E.n[cur];
    if (x.kind == E_CONST && E.cval(cur) % size == 0)
        return E.constant(E.cval(cur) / size, x.type);
    if (x.kind != E_BINARY)
        return 0;
    if (x.op == O_SHL && x.b && E.n[x.b].kind == E_CONST && E.cval(x.b) < 32 &&
        (1ull << E.cval(x.b)) == size)
        return x.a;
    if (x.op == O_MUL) {
        if (x.b && E.n[x.b].kind == E_CONST && E.cval(x.b) == size)
            return x.a;
        if (x.a && E.n[x.a].kind == E_CONST && E.cval(x.a) == size)
            return x.b;
    }
    return 0;
}

// render_indexed  codegen.cpp:202-234: returns true and pushes the tasks
// for "name[index]" when the address splits into pointer-arg base + scaled
// index terms.
OD_NOINL bool render_indexed(Writer &w, RenderCtx &rc, u32 addr, DT elem) {
    EArena &E = *rc.E;
    U32Stack &terms = rc.fs.terms;
    u32 tb = terms.top;
    collect_add_terms(E, addr, rc.fs.st, terms);
    u32 nt = terms.top - tb;
    u32 *tv = terms.p + tb;
    int base = -1;
    u32 esz = dt_byte_size(elem);
    for (u32 i = 0; i < nt; ++i) {
        u32 b = tv[i];
        const ENode *bare = strip_casts(E, b);
        if (base < 0 && bare && bare->kind == E_ARG && dt_is_pointer(bare->type) &&
            dt_byte_size(dt_pointee(bare->type)) == esz) {
            base = (int)i;
        }
    }
    bool ok = base >= 0 && !terms.oom;
    u32 index = 0;
    if (ok) {
        for (u32 i = 0; i < nt; ++i) {
            if ((int)i == base)
                continue;
            u32 part = unscale_term(E, tv[i], esz);
            if (!part) {
                ok = false;
                break;
            }
            index = index ? E.binary(O_ADD, index, part, E.n[part].type) : part;
        }
    }
    if (ok) {
        u32 b = tv[base];
        const ENode *bare = strip_casts(E, b);
        put_arg_name(w, rc, bare->a);
        w.put('[');
        rc.ts.push(RT_CHAR, ']', 0);
        if (index)
            rc.ts.push(RT_NODE, 0, index);
        else
            rc.ts.push(RT_CHAR, '0', 0);
    }
    terms.top = tb;
    return ok;
}

OD_NOINL void render_deref(Writer &w, RenderCtx &rc, u32 addr, DT elem) {
    if (render_indexed(w, rc, addr, elem))
        return;
    w.lit("*((");
    switch (dt_space(elem)) {
    case AS_GLOBAL: w.lit("__global "); break;
    case AS_LOCAL: w.lit("__local "); break;
    case AS_CONSTANT: w.lit("__constant "); break;
    default: break;
    }
    render_type(w, dt_with_space(elem, AS_NONE));
    w.lit(" *)");
    rc.ts.push(RT_CHAR, ')', 0);
    rc.ts.push(RT_NODE, kUnary, addr);
}

// render(e, min_prec)  codegen.cpp:260-352, streamed through the task stack.
OD_NOINL void render_expr(Writer &w, RenderCtx &rc, u32 root, int min_prec = 0) {
    EArena &E = *rc.E;
    TaskStack &ts = rc.ts;
    u32 base = ts.top;
    ts.push(RT_NODE, (u32)min_prec, root);
    while (ts.top > base && !ts.oom) {
        u64 tk = ts.p[--ts.top];
        u32 kind = (u32)(tk & 0xff);
        u32 arg = (u32)((tk >> 8) & 0xffffff);
        u32 e = (u32)(tk >> 32);
        if (kind == RT_CHAR) {
            w.put((u8)arg);
            continue;
        }
        if (kind == RT_STR) {
            w.puts(rstr(arg));
            continue;
        }
        if (kind == RT_SA) {
            // render_sign_aware  codegen.cpp:141-154; arg = op | min_prec<<8
            u32 op = arg & 0xff;
            u32 mp = arg >> 8;
            if (!e) {
                ts.push(RT_NODE, mp, 0);
                continue;
            }
            DT ct = E.n[e].type;
            bool cu = op_wants_unsigned(op) && dt_is_signed(ct);
            bool cs = op_wants_signed(op) && !dt_is_signed(ct) && !dt_is_float(ct);
            if (!cu && !cs) {
                ts.push(RT_NODE, mp, e);
                continue;
            }
            w.put('(');
            if (cu)
                w.puts(dt_bits(ct) == 64 ? "ulong" : "uint");
            else
                w.puts(dt_bits(ct) == 64 ? "long" : "int");
            w.put(')');
            ts.push(RT_NODE, kUnary, e);
            continue;
        }
        // RT_NODE
        int mp = (int)arg;
        if (!e) {
            w.lit("0 /* missing */");
            continue;
        }
        const ENode x = E.n[e];
        switch (x.kind) {
        case E_CONST: render_const(w, E, e); break;
        case E_BUILTIN:
            w.puts(builtin_name(x.op));
            w.put('(');
            if (x.op != F_WORK_DIM)
                w.put_u64(x.x);
            w.put(')');
            break;
        case E_ARG: put_arg_name(w, rc, x.a); break;
        case E_VAR: put_var_name(w, x.x, x.a); break;
        case E_KBASE: w.lit("__settings_base"); break;
        case E_UNARY:
            switch (x.op) {
            case U_LNOT:
                w.put('!');
                ts.push(RT_NODE, kUnary, x.a);
                break;
            case U_BITNOT:
                w.put('~');
                ts.push(RT_NODE, kUnary, x.a);
                break;
            case U_NEG:
                w.put('-');
                ts.push(RT_NODE, kUnary, x.a);
                break;
            case U_LO32:
                w.lit("(uint)");
                ts.push(RT_NODE, kUnary, x.a);
                break;
            case U_HI32:
                w.lit("(uint)(");
                ts.push(RT_STR, S_SHR32, 0);
                ts.push(RT_NODE, 11, x.a);
                break;
            default: // U_CAST
                if (x.a && is_bit_reinterpret(E.n[x.a].type, x.type)) {
                    w.puts(cast_name(x.type));
                    w.put('(');
                    ts.push(RT_CHAR, ')', 0);
                    ts.push(RT_NODE, 0, x.a);
                } else {
                    w.put('(');
                    render_type(w, dt_with_space(x.type, AS_NONE));
                    w.put(')');
                    ts.push(RT_NODE, kUnary, x.a);
                }
                break;
            }
            break;
        case E_BINARY: {
            if (x.op == O_MULHI || x.op == O_MULHIS) {
                w.lit("mul_hi(");
                ts.push(RT_CHAR, ')', 0);
                ts.push(RT_SA, x.op, x.b);
                ts.push(RT_STR, S_COMMA, 0);
                ts.push(RT_SA, x.op, x.a);
                break;
            }
            if (x.op == O_CONCAT64) {
                w.lit("upsample(");
                ts.push(RT_CHAR, ')', 0);
                ts.push(RT_NODE, 0, x.a);
                ts.push(RT_STR, S_COMMA, 0);
                ts.push(RT_NODE, 0, x.b);
                break;
            }
            int prec = binop_prec(x.op);
            bool paren = prec < mp;
            if (paren) {
                w.put('(');
                ts.push(RT_CHAR, ')', 0);
            }
            ts.push(RT_SA, x.op | ((u32)(prec + 1) << 8), x.b);
            ts.push(RT_STR, S_BINOP_BASE + x.op, 0);
            ts.push(RT_SA, x.op | ((u32)prec << 8), x.a);
            break;
        }
        case E_TERNARY: {
            bool paren = 3 < mp;
            if (paren) {
                w.put('(');
                ts.push(RT_CHAR, ')', 0);
            }
            ts.push(RT_NODE, 3, x.c);
            ts.push(RT_STR, S_COLON, 0);
            ts.push(RT_NODE, 3, x.b);
            ts.push(RT_STR, S_QMARK, 0);
            ts.push(RT_NODE, 4, x.a);
            break;
        }
        case E_DEREF: render_deref(w, rc, x.a, x.type); break;
        default: break;
        }
    }
    ts.top = base;
}

} // namespace od
