// ocldec-b200: expression arena, peephole factories, builtin folds and the
// streaming OpenCL renderer (one thread per kernel, explicit stacks).
//
//   factories / expr_equal / negate_condition   expr.cpp:40-228
//   fold_expr and the builtin folds             builtin_detector.cpp:20-209
//   render / render_const / render_indexed      codegen.cpp:19-352
//   render_type                                 type_recovery.cpp:171-212
//
// Nodes are 24-byte records addressed by u32 ids (0 = null).  Identity of an
// id is the identity of the reference's shared_ptr: factories allocate
// exactly where the reference calls make_shared and return existing ids
// where it returns existing pointers (no hash-consing), because
// read_pair_ids/dissolve_pair compare pointers (sym_state.cpp:110,129).
#pragma once

#include <math.h>

#include "od_base.cuh"

namespace od {

enum EKind : u8 { E_NULL = 0, E_CONST, E_BUILTIN, E_ARG, E_KBASE, E_VAR, E_UNARY, E_BINARY,
                  E_TERNARY, E_DEREF };
enum UOp : u8 { U_LNOT = 0, U_BITNOT, U_NEG, U_LO32, U_HI32, U_CAST };
enum BOp : u8 { O_ADD = 0, O_SUB, O_MUL, O_MULHI, O_MULHIS, O_DIV, O_AND, O_OR, O_XOR, O_SHL,
                O_LSHR, O_ASHR, O_CONCAT64, O_CMPEQ, O_CMPNE, O_CMPLT, O_CMPLE, O_CMPGT, O_CMPGE,
                O_CMPLTU, O_CMPLEU, O_CMPGTU, O_CMPGEU };
enum BFn : u8 { F_GLOBAL_ID = 0, F_LOCAL_ID, F_GROUP_ID, F_GLOBAL_SIZE, F_LOCAL_SIZE,
                F_NUM_GROUPS, F_GLOBAL_OFFSET, F_WORK_DIM };

struct alignas(8) ENode {
    u8 kind;
    u8 op;   // UOp/BOp; BFn for builtins
    u16 x;   // builtin dim; var name class (physical register slot)
    DT type;
    u32 a, b, c; // children; const value = a | b<<32; var number = a; arg name id = a
    u32 memo;    // fold_expr cache (0 = not folded yet)
};

static_assert(sizeof(ENode) == 24, "EArena::put writes a node as three 8-byte words");

struct KConfig; // od_kernel.cuh

// Per-kernel expression arena.
struct EArena {
    ENode *n;
    u32 top, cap;
    bool oom;

    OD_INL u32 alloc() {
        if (top >= cap) {
            oom = true;
            return 0; // degrade to null; the kernel is retried with more memory
        }
        return top++;
    }
    OD_INL const ENode &operator[](u32 i) const { return n[i]; }
    // A node in three 8-byte stores (ENode is 24 bytes, the pool 16-byte aligned).
    OD_INL void put(u32 i, u8 kind, u8 op, u16 x, DT t, u32 a, u32 b, u32 c) {
        u64 *q = reinterpret_cast<u64 *>(&n[i]);
        q[0] = (u64)kind | ((u64)op << 8) | ((u64)x << 16) | ((u64)t << 32);
        q[1] = (u64)a | ((u64)b << 32);
        q[2] = (u64)c; // memo = 0
    }
    OD_INL u64 cval(u32 i) const { return (u64)n[i].a | ((u64)n[i].b << 32); }
    OD_INL bool is_const(u32 i) const { return i && n[i].kind == E_CONST; }
    OD_INL bool is_const_v(u32 i, u64 v) const { return is_const(i) && cval(i) == v; }

    // Expr::constant  expr.cpp:40-44
    OD_HOT u32 constant(u64 v, DT t) {
        u32 bits = dt_bits(t) ? dt_bits(t) : 64;
        u64 mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
        v &= mask;
        u32 i = alloc();
        if (!i)
            return 0;
        put(i, E_CONST, 0, 0, t, (u32)v, (u32)(v >> 32), 0);
        return i;
    }
    OD_HOT u32 leaf(u8 kind, u8 op, u16 x, DT t, u32 a) {
        u32 i = alloc();
        if (!i)
            return 0;
        put(i, kind, op, x, t, a, 0, 0);
        return i;
    }
    OD_INL u32 builtin(u32 fn, u32 dim, DT t) { return leaf(E_BUILTIN, (u8)fn, (u16)dim, t, 0); }
    OD_INL u32 arg(u32 name_id, DT t) { return leaf(E_ARG, 0, 0, t, name_id); }
    OD_INL u32 kbase() { return leaf(E_KBASE, 0, 0, DT_U64, 0); }
    OD_INL u32 var(u32 cls, u32 num, DT t) { return leaf(E_VAR, 0, (u16)cls, t, num); }

    // Expr::unary  expr.cpp:71-93
    OD_HOT u32 unary(u32 op, u32 a, DT t) {
        if (a) {
            const ENode &x = n[a];
            if (op == U_LO32 && x.kind == E_BINARY && x.op == O_CONCAT64)
                return x.a;
            if (op == U_HI32 && x.kind == E_BINARY && x.op == O_CONCAT64)
                return x.b;
            if (x.kind == E_CONST) {
                u64 v = cval(a);
                switch (op) {
                case U_LO32: return constant((u32)v, t);
                case U_HI32: return constant((u32)(v >> 32), t);
                case U_BITNOT: return constant(~v, t);
                case U_NEG: return constant(~v + 1, t);
                default: break;
                }
            }
        }
        u32 i = alloc();
        if (!i)
            return 0;
        put(i, E_UNARY, (u8)op, 0, t, a, 0, 0);
        return i;
    }

    // Expr::binary  expr.cpp:95-132
    OD_HOT u32 binary(u32 op, u32 a, u32 b, DT t) {
        if (a && b && is_const(a) && is_const(b) && !dt_is_float(t) && dt_bits(t) <= 32) {
            u32 x = (u32)cval(a), y = (u32)cval(b);
            bool folded = true;
            u32 v = 0;
            switch (op) {
            case O_ADD: v = x + y; break;
            case O_SUB: v = x - y; break;
            case O_MUL: v = x * y; break;
            case O_AND: v = x & y; break;
            case O_OR: v = x | y; break;
            case O_XOR: v = x ^ y; break;
            case O_SHL: v = y >= 32 ? 0 : x << y; break;
            case O_LSHR: v = y >= 32 ? 0 : x >> y; break;
            default: folded = false; break;
            }
            if (folded)
                return constant(v, t);
        }
        if (a && b && is_const_v(b, 0) &&
            (op == O_ADD || op == O_SUB || op == O_OR || op == O_XOR || op == O_SHL ||
             op == O_LSHR || op == O_ASHR))
            return a;
        if (a && b && is_const_v(a, 0) && (op == O_ADD || op == O_OR))
            return b;
        if (a && b && op == O_MUL) {
            if (is_const_v(b, 1))
                return a;
            if (is_const_v(a, 1))
                return b;
        }
        u32 i = alloc();
        if (!i)
            return 0;
        put(i, E_BINARY, (u8)op, 0, t, a, b, 0);
        return i;
    }

    // Expr::ternary  expr.cpp:134-140
    OD_NOINL u32 ternary(u32 cond, u32 a, u32 b, DT t) {
        if (cond && is_const(cond))
            return cval(cond) ? a : b;
        u32 i = alloc();
        if (!i)
            return 0;
        put(i, E_TERNARY, 0, 0, t, cond, a, b);
        return i;
    }

    // Expr::deref  expr.cpp:142-148
    OD_NOINL u32 deref(u32 addr, DT pointee, u32 space) {
        u32 i = alloc();
        if (!i)
            return 0;
        put(i, E_DEREF, 0, 0, dt_with_space(pointee, space), addr, 0, 0);
        return i;
    }
};

OD_INL bool is_cmp(u32 op) { return op >= O_CMPEQ && op <= O_CMPGEU; }

// Scratch stack of u32 carved from the arena (explicit recursion stacks).
struct U32Stack {
    u32 *p;
    u32 top, cap, hw;
    bool oom;
    OD_INL void push(u32 v) {
        if (top < cap) {
            p[top++] = v;
            if (top > hw)
                hw = top;
        } else {
            oom = true;
        }
    }
    OD_INL u32 pop() { return p[--top]; }
    OD_INL bool empty() const { return top == 0; }
};

// expr_equal  expr.cpp:152-177 (iterative; pointer equality short-cuts)
OD_NOINL bool expr_equal(const EArena &E, u32 a, u32 b, U32Stack &st) {
    u32 base = st.top;
    st.push(a);
    st.push(b);
    bool ok = true;
    while (st.top > base && !st.oom) {
        u32 y = st.pop(), x = st.pop();
        if (x == y)
            continue;
        if (!x || !y || E.n[x].kind != E.n[y].kind) {
            ok = false;
            break;
        }
        const ENode &p = E.n[x], &q = E.n[y];
        switch (p.kind) {
        case E_CONST:
            if (!(p.a == q.a && p.b == q.b && dt_bits(p.type) == dt_bits(q.type)))
                ok = false;
            break;
        case E_BUILTIN:
            if (!(p.op == q.op && p.x == q.x))
                ok = false;
            break;
        case E_ARG:
            if (p.a != q.a)
                ok = false;
            break;
        case E_VAR:
            if (!(p.x == q.x && p.a == q.a))
                ok = false;
            break;
        case E_KBASE:
            break;
        case E_UNARY:
            if (p.op != q.op)
                ok = false;
            else {
                st.push(p.a);
                st.push(q.a);
            }
            break;
        case E_BINARY:
            if (p.op != q.op)
                ok = false;
            else {
                st.push(p.b);
                st.push(q.b);
                st.push(p.a);
                st.push(q.a);
            }
            break;
        case E_TERNARY:
            st.push(p.c);
            st.push(q.c);
            st.push(p.b);
            st.push(q.b);
            st.push(p.a);
            st.push(q.a);
            break;
        case E_DEREF:
            if (p.type != q.type)
                ok = false;
            else {
                st.push(p.a);
                st.push(q.a);
            }
            break;
        }
        if (!ok)
            break;
    }
    st.top = base;
    return ok;
}

// negate_condition  expr.cpp:206-228
OD_NOINL u32 negate_condition(EArena &E, u32 e) {
    if (e && E.n[e].kind == E_BINARY) {
        u32 op = E.n[e].op, f = op;
        switch (op) {
        case O_CMPEQ: f = O_CMPNE; break;
        case O_CMPNE: f = O_CMPEQ; break;
        case O_CMPLT: f = O_CMPGE; break;
        case O_CMPGE: f = O_CMPLT; break;
        case O_CMPGT: f = O_CMPLE; break;
        case O_CMPLE: f = O_CMPGT; break;
        case O_CMPLTU: f = O_CMPGEU; break;
        case O_CMPGEU: f = O_CMPLTU; break;
        case O_CMPGTU: f = O_CMPLEU; break;
        case O_CMPLEU: f = O_CMPGTU; break;
        default: break;
        }
        if (f != op) {
            const ENode x = E.n[e];
            return E.binary(f, x.a, x.b, x.type);
        }
    }
    if (e && E.n[e].kind == E_UNARY && E.n[e].op == U_LNOT)
        return E.n[e].a;
    return E.unary(U_LNOT, e, DT_I32);
}

// collect_add_terms  expr.cpp:179-186: appends the in-order leaves of the
// Add tree rooted at e to out (left to right).
OD_NOINL void collect_add_terms(const EArena &E, u32 e, U32Stack &st, U32Stack &out) {
    u32 base = st.top;
    st.push(e);
    while (st.top > base && !st.oom) {
        u32 x = st.pop();
        if (x && E.n[x].kind == E_BINARY && E.n[x].op == O_ADD) {
            st.push(E.n[x].b);
            st.push(E.n[x].a);
        } else {
            out.push(x);
        }
    }
    st.top = base;
}

} // namespace od
