// ocldec-b200: symbolic lowering (sym_state.cpp, lower.cpp), decl hoisting
// (decompiler.cpp:37-53) and kernel emission (codegen.cpp:358-467).
//
// RegisterFile copies at if-splits (lower.cpp:143-147) are replaced by an
// undo log: the then arm runs in place, its touched slots are saved as a
// sorted delta and rolled back, the else arm runs, and the merge visits only
// the union of touched slots in ascending register id (the order of
// merge_at_join's 0..365 loop, sym_state.cpp:876).
#pragma once

namespace od {

// ------------------------------------------------------- register file
OD_INL u32 dense_of_phys(u32 p) {
    if (p < 360)
        return p;
    switch (p) {
    case 360: return kRegIdExecLo;
    case 361: return kRegIdVccLo;
    case 362: return kRegIdScc;
    default: return kRegIdM0;
    }
}

OD_INL void log_slot(KCtx &K, u32 p) {
    K.dirty[p >> 5] |= 1u << (p & 31);
    if (!K.log_depth)
        return;
    if (K.nlog >= K.log_cap) {
        K.oom = true;
        return;
    }
    const uint4 v = *reinterpret_cast<const uint4 *>(&K.regs[p]);
    *reinterpret_cast<uint4 *>(&K.log[K.nlog++]) = make_uint4(v.x, v.y, v.z, (v.w & 0xffu) | (p << 8));
    if (K.nlog > K.log_hw)
        K.log_hw = K.nlog;
}

OD_INL void undo_to(KCtx &K, u32 pos) {
    while (K.nlog > pos) {
        const uint4 v = *reinterpret_cast<const uint4 *>(&K.log[--K.nlog]);
        *reinterpret_cast<uint4 *>(&K.regs[v.w >> 8]) = make_uint4(v.x, v.y, v.z, v.w & 0xffu);
    }
}

OD_INL void record_fresh(KCtx &K, u32 cls, u32 num, DT t) {
    if (K.nfresh >= K.fresh_cap) {
        K.oom = true;
        return;
    }
    Fresh &f = K.fresh[K.nfresh++];
    f.cls = cls;
    f.num = num;
    f.type = t;
}

// bind_fresh  sym_state.cpp:63-78
OD_HOT u32 bind_fresh(KCtx &K, u32 p, DT t = DT_B32) {
    Slot &s = K.regs[p];
    if (!s.expr) {
        log_slot(K, p);
        if (dt_is_unknown(s.type))
            s.type = t;
        s.expr = K.E.var(p, s.version, s.type);
        s.integ = IN_ENTIRE;
        record_fresh(K, p, s.version, s.type);
        K.pool.insert(p, s.version);
    }
    return s.expr;
}

// read_slot32  sym_state.cpp:82-94
OD_INL u32 read_slot32(KCtx &K, u32 id) {
    u32 p = phys_of(id);
    bind_fresh(K, p);
    const Slot &s = K.regs[p];
    if (s.integ == IN_LOW)
        return K.E.unary(U_LO32, s.expr, DT_B32);
    if (s.integ == IN_HIGH)
        return K.E.unary(U_HI32, s.expr, DT_B32);
    return s.expr;
}

// concat64  sym_state.cpp:96-105
OD_NOINL u32 concat64(KCtx &K, u32 lo, u32 hi) {
    EArena &E = K.E;
    if (E.is_const_v(hi, 0))
        return E.unary(U_CAST, lo, DT_U64);
    if (lo && hi && E.n[lo].kind == E_UNARY && E.n[lo].op == U_LO32 && E.n[hi].kind == E_UNARY &&
        E.n[hi].op == U_HI32 && expr_equal(E, E.n[lo].a, E.n[hi].a, K.eqst))
        return E.n[lo].a;
    return E.binary(O_CONCAT64, lo, hi, DT_B64);
}

// read_pair_ids  sym_state.cpp:107-114.  The two read_slot32 calls are
// arguments of one call; GCC (the oracle's compiler) evaluates them right to
// left, which fixes the order fresh variables are recorded in.
OD_NOINL u32 read_pair_ids(KCtx &K, u32 lo_id) {
    const Slot &lo = K.regs[phys_of(lo_id)];
    const Slot &hi = K.regs[phys_of(lo_id + 1)];
    if (lo.expr && lo.expr == hi.expr && lo.integ == IN_LOW && hi.integ == IN_HIGH)
        return lo.expr;
    u32 h = read_slot32(K, lo_id + 1);
    u32 l = read_slot32(K, lo_id);
    return concat64(K, l, h);
}

// dissolve_pair  sym_state.cpp:118-135
OD_HOT void dissolve_pair(KCtx &K, u32 id) {
    u32 p = phys_of(id);
    Slot &s = K.regs[p];
    if (s.integ == IN_ENTIRE || !s.expr)
        return;
    const bool is_low = s.integ == IN_LOW;
    if (id >= kRegIdExecLo) {
        log_slot(K, p);
        s.integ = IN_ENTIRE;
        return;
    }
    u32 pid = is_low ? id + 1 : id - 1;
    if (pid >= kRegIdExecLo) { // out of the reference's std::array range
        K.oom = true;
        return;
    }
    Slot &q = K.regs[pid];
    if (q.expr == s.expr) {
        log_slot(K, pid);
        q.expr = K.E.unary(is_low ? U_HI32 : U_LO32, s.expr, DT_B32);
        q.integ = IN_ENTIRE;
        q.type = DT_B32;
    }
    log_slot(K, p);
    s.integ = IN_ENTIRE;
}

OD_HOT void write_slot32(KCtx &K, u32 id, u32 value, DT t) {
    if (id >= kNumRegIds) {
        K.oom = true;
        return;
    }
    dissolve_pair(K, id);
    u32 p = phys_of(id);
    log_slot(K, p);
    Slot &s = K.regs[p];
    s.version += 1;
    s.expr = value;
    s.type = t;
    s.integ = IN_ENTIRE;
}

OD_NOINL void write_pair_ids(KCtx &K, u32 lo_id, u32 value, DT t) {
    if (lo_id >= kRegIdExecLo) {
        if (lo_id >= kNumRegIds) {
            K.oom = true;
            return;
        }
        u32 p = phys_of(lo_id);
        log_slot(K, p);
        Slot &s = K.regs[p];
        s.version += 1;
        s.expr = value;
        s.type = t;
        s.integ = IN_ENTIRE;
        return;
    }
    if (lo_id + 1 >= kRegIdExecLo) {
        K.oom = true;
        return;
    }
    dissolve_pair(K, lo_id);
    dissolve_pair(K, lo_id + 1);
    log_slot(K, lo_id);
    log_slot(K, lo_id + 1);
    Slot &lo = K.regs[lo_id];
    Slot &hi = K.regs[lo_id + 1];
    lo.version += 1;
    hi.version += 1;
    lo.expr = value;
    hi.expr = value;
    lo.type = t;
    hi.type = t;
    lo.integ = IN_LOW;
    hi.integ = IN_HIGH;
}

// invalidate_slot  sym_state.cpp:169-180
OD_NOINL void invalidate_slot(KCtx &K, u32 id, u32 count) {
    for (u32 i = 0; i < count; ++i) {
        if (id + i >= kNumRegIds) {
            K.oom = true; // std::array::at would throw in the reference
            return;
        }
        dissolve_pair(K, id + i);
        u32 p = phys_of(id + i);
        log_slot(K, p);
        Slot &s = K.regs[p];
        s.version += 1;
        s.expr = 0;
        s.type = DT_UNKNOWN;
        s.integ = IN_ENTIRE;
        if (id + i >= kRegIdExecLo)
            break;
    }
}

OD_INL u32 operand_reg_id(const Opnd &o) {
    switch (o.kind) {
    case OK_SREG: return o.r.a;
    case OK_VREG: return kRegIdVgpr0 + o.r.a;
    case OK_SPECIAL:
        switch (o.special) {
        case SP_EXEC:
        case SP_EXEC_LO: return kRegIdExecLo;
        case SP_EXEC_HI: return kRegIdExecHi;
        case SP_VCC:
        case SP_VCC_LO: return kRegIdVccLo;
        case SP_VCC_HI: return kRegIdVccHi;
        case SP_SCC: return kRegIdScc;
        default: return kRegIdM0;
        }
    default: return kNumRegIds;
    }
}

OD_INL u32 read_pair(KCtx &K, const Opnd &o);

// read_operand  sym_state.cpp:205-227
OD_HOT u32 read_operand(KCtx &K, const Opnd &o) {
    switch (o.kind) {
    case OK_LITERAL: return K.E.constant((u64)o.value & 0xffffffffull, DT_B32);
    case OK_SREG:
    case OK_VREG: {
        if (o.count >= 2)
            return read_pair(K, o);
        u32 id = operand_reg_id(o);
        if (id >= kNumRegIds) {
            K.oom = true;
            return 0;
        }
        return read_slot32(K, id);
    }
    case OK_SPECIAL: {
        u32 id = operand_reg_id(o);
        DT t = (o.special == SP_EXEC || o.special == SP_VCC) ? DT_B64 : DT_B32;
        return bind_fresh(K, phys_of(id), t);
    }
    default: return 0;
    }
}

// read_pair  sym_state.cpp:229-240
OD_INL u32 read_pair(KCtx &K, const Opnd &o) {
    if (o.kind == OK_LITERAL)
        return K.E.constant((u64)o.value, DT_B64);
    if (o.kind == OK_SPECIAL)
        return read_operand(K, o);
    if (o.kind == OK_SREG || o.kind == OK_VREG) {
        u32 id = operand_reg_id(o);
        if (id + 1 >= kNumRegIds) {
            K.oom = true;
            return 0;
        }
        if (o.count < 2)
            return read_slot32(K, id);
        return read_pair_ids(K, id);
    }
    return 0;
}

// ------------------------------------------------------- statements
OD_INL u32 new_stmt(KCtx &K, u8 kind) {
    if (K.nst >= K.st_cap) {
        K.oom = true;
        return 0; // stmt 0 is a scratch sink
    }
    u32 i = K.nst++;
    Stmt &s = K.st[i];
    s.kind = kind;
    s.pad = 0;
    s.cls = 0;
    s.next = 0;
    s.a = s.b = s.c = s.d = 0;
    return i;
}

OD_INL u32 new_list(KCtx &K) {
    if (K.nlists >= K.lists_cap) {
        K.oom = true;
        return 0;
    }
    u32 i = K.nlists++;
    K.lists[i].head = K.lists[i].tail = 0;
    return i;
}

OD_INL void list_append(KCtx &K, u32 l, u32 s) {
    if (!s)
        return;
    SList &L = K.lists[l];
    if (L.tail)
        K.st[L.tail].next = s;
    else
        L.head = s;
    L.tail = s;
}

OD_INL u32 fold(KCtx &K, u32 e) { return fold_expr(K.E, e, K.cfg, K.fs); }

// Clears a name set (16-byte stores; cap is a power of two >= 1024).
OD_INL void name_set_clear(NameSet &ns) {
    uint4 z = {0, 0, 0, 0};
    uint4 *p = reinterpret_cast<uint4 *>(ns.keys);
    for (u32 i = 0; i < ns.cap / 2; ++i)
        p[i] = z;
    ns.count = 0;
}

// ------------------------------------------------------------ stepper
struct Step {
    KCtx &K;
    const Ins &I;
    u32 out;        // statement list
    const Opnd *o;  // the instruction's operands (K.in->ops + I.op_start)
    u32 nn_;        // operand count (0 for the synthetic s_endpgm)

    OD_INL const Opnd &op(u32 k) const { return o[k]; }
    OD_INL u32 n() const { return nn_; }
    OD_INL u32 read(const Opnd &o) { return read_operand(K, o); }
    OD_INL u32 read64(const Opnd &o) { return read_pair(K, o); }
    OD_INL DT ty(u32 e) const { return K.E.n[e].type; }

    OD_HOT void write(const Opnd &o, u32 value, DT t) {
        u32 id = operand_reg_id(o);
        if (id >= kNumRegIds)
            return;
        const bool pair = o.count >= 2 || (o.kind == OK_SPECIAL && (o.special == SP_EXEC || o.special == SP_VCC));
        if (pair)
            write_pair_ids(K, id, value, t);
        else
            write_slot32(K, id, value, t);
    }

    // Stepper::fallback  sym_state.cpp:273-288
    OD_NOINL void fallback() {
        u32 s = new_stmt(K, SK_RAW);
        K.st[s].a = I.src.off;
        K.st[s].b = I.src.len;
        list_append(K, out, s);
        K.fallbacks++;
        u32 nn = (I.flags & IF_PARSE_FAILED) ? 0 : n();
        for (u32 k = 0; k < nn; ++k) {
            u32 id = operand_reg_id(op(k));
            if (id < kNumRegIds) {
                invalidate_slot(K, id, op(k).count);
                break;
            }
        }
        K.pend.valid = 0;
        K.pend.base64 = K.pend.addend = 0;
        K.pend.lo_vgpr = K.pend.lo_version = 0;
    }

    // Stepper::coerce  sym_state.cpp:300-310
    OD_HOT u32 coerce(u32 e, DT want) {
        if (!e)
            return e;
        DT et = ty(e);
        if (dt_base(et) == dt_base(want) && dt_bits(et) == dt_bits(want))
            return e;
        if (K.E.is_const(e))
            return K.E.constant(K.E.cval(e), want);
        if (dt_is_float(want) != dt_is_float(et))
            return K.E.unary(U_CAST, e, want);
        return e;
    }

    // Shared handler tails (one out-of-line copy instead of one per handler:
    // the lowering pass is bound by instruction fetch).  Reads happen in the
    // order of the arguments, as in the handlers they replace.
    OD_NOINL u32 rd(u32 k, DT t) { return coerce(read(op(k)), t); }
    OD_NOINL void bin(u32 o, DT t, u32 ka, u32 kb) {
        u32 a = rd(ka, t);
        u32 b = rd(kb, t);
        write(op(0), K.E.binary(o, a, b, t), t);
    }

    OD_NOINL void push_store(u32 addr, u32 value, DT et) {
        u32 s = new_stmt(K, SK_STORE);
        // lower_block folds store address and value (lower.cpp:37-39); the
        // fold runs in its own pass (dk_fold)
        K.st[s].a = addr; // folded by dk_fold
        K.st[s].b = value;
        K.st[s].c = et;
        list_append(K, out, s);
    }

    // do_scalar_load  sym_state.cpp:348-405
    OD_NOINL void scalar_load(u32 dwords) {
        if (n() < 2 || !op_is_sreg(op(0)))
            return fallback();
        const Opnd &dst = op(0);
        const Opnd &base_op = op(1);
        u64 offset = 0;
        if (n() >= 3 && op(2).kind == OK_LITERAL)
            offset = (u64)op(2).value;
        u32 base = read64(base_op);
        if (base && K.E.n[base].kind == E_KBASE) {
            if (dwords <= 2) {
                u32 v = match_settings_load(K, (u32)offset, dwords);
                if (v) {
                    if (dwords == 2)
                        write_pair_ids(K, dst.r.a, v, ty(v));
                    else
                        write_slot32(K, dst.r.a, v, ty(v));
                    return;
                }
            }
            bool all_known = true;
            for (u32 i = 0; i < dwords && all_known; ++i) {
                bool second;
                all_known = abi_find_dword(K, (u32)offset + 4 * i, &second) != nullptr;
            }
            if (all_known) {
                for (u32 i = 0; i < dwords;) {
                    bool second;
                    const AbiEntry *e = abi_find_dword(K, (u32)offset + 4 * i, &second);
                    u32 v = match_settings_load(K, e->offset, e->dwords);
                    if (e->dwords == 2 && !second && i + 1 < dwords) {
                        write_pair_ids(K, dst.r.a + i, v, v ? ty(v) : DT_UNKNOWN);
                        i += 2;
                    } else {
                        u32 half = e->dwords == 2 ? K.E.unary(second ? U_HI32 : U_LO32, v, DT_B32) : v;
                        write_slot32(K, dst.r.a + i, half, half ? ty(half) : DT_UNKNOWN);
                        i += 1;
                    }
                }
                return;
            }
            diag(K, DG_SLOAD_UNMAPPED, I.line);
        }
        for (u32 i = 0; i < dwords; ++i) {
            u32 addr = K.E.binary(O_ADD, base, K.E.constant(offset + 4 * i, DT_U64), DT_U64);
            u32 v = K.E.deref(addr, DT_B32, AS_GLOBAL);
            write_slot32(K, dst.r.a + i, v, ty(v));
        }
    }

    // do_compare  sym_state.cpp:407-460
    OD_NOINL bool compare(bool vector_side) {
        DT ct = suffix_type0(I, DT_I32);
        const bool uns = dt_base(ct) == B_UNSIGNED;
        u32 cop;
        switch (I.root) {
        case R_CMP_EQ: cop = O_CMPEQ; break;
        case R_CMP_NE:
        case R_CMP_LG:
        case R_CMP_NEQ: cop = O_CMPNE; break;
        case R_CMP_LT: cop = uns ? O_CMPLTU : O_CMPLT; break;
        case R_CMP_LE: cop = uns ? O_CMPLEU : O_CMPLE; break;
        case R_CMP_GT: cop = uns ? O_CMPGTU : O_CMPGT; break;
        case R_CMP_GE: cop = uns ? O_CMPGEU : O_CMPGE; break;
        default: return false;
        }
        u32 fs = vector_side ? 1 : 0;
        if (n() < fs + 2)
            return false;
        u32 a = read(op(fs));
        u32 b = read(op(fs + 1));
        if (dt_is_float(ct)) {
            a = coerce(a, ct);
            b = coerce(b, ct);
        } else if (a && K.E.is_const(a)) {
            a = K.E.constant(K.E.cval(a), ct);
        }
        if (!dt_is_float(ct) && b && K.E.is_const(b))
            b = K.E.constant(K.E.cval(b), ct);
        u32 cmp = K.E.binary(cop, a, b, DT_I32);
        if (vector_side) {
            write(op(0), cmp, DT_B64);
        } else {
            log_slot(K, 362);
            Slot &scc = K.regs[362];
            scc.version += 1;
            scc.expr = cmp;
            scc.type = DT_I32;
            scc.integ = IN_ENTIRE;
        }
        return true;
    }

    // handle_scalar  sym_state.cpp:462-555
    OD_NOINL bool scalar() {
        const u32 r = I.root;
        const u32 nn = n();
        if (nn > 0 && op(0).kind == OK_SPECIAL &&
            (op(0).special == SP_EXEC || op(0).special == SP_EXEC_LO || op(0).special == SP_EXEC_HI))
            return false;
        switch (r) { // one jump table (instruction fetch)
        case R_LOAD_DWORD: return scalar_load(1), true;
        case R_LOAD_DWORDX2: return scalar_load(2), true;
        case R_LOAD_DWORDX4: return scalar_load(4), true;
        case R_MOV:
            if (nn < 2)
                return false;
            {
            DT t = suffix_type0(I, DT_B32);
            u32 v = dt_bits(t) == 64 ? read64(op(1)) : read(op(1));
            write(op(0), v, v ? ty(v) : DT_UNKNOWN);
            return true;
        }
        case R_ADD:
        case R_SUB:
        case R_MUL:
        case R_ADDK:
        case R_MULK:
            if (nn < 2)
                return false;
            {
            const bool k = r == R_ADDK || r == R_MULK;
            if (!k && nn < 3)
                return false;
            u32 o = O_ADD;
            if (r == R_SUB)
                o = O_SUB;
            else if (r == R_MUL || r == R_MULK)
                o = O_MUL;
            bin(o, suffix_type0(I, DT_I32), k ? 0 : 1, k ? 1 : 2);
            invalidate_slot(K, kRegIdScc, 1);
            return true;
        }
        case R_AND:
        case R_OR:
        case R_XOR:
        case R_ANDN2:
            if (nn < 3)
                return false;
            {
            DT t = suffix_type0(I, DT_B32);
            const bool wide = dt_bits(t) == 64;
            u32 a = wide ? read64(op(1)) : read(op(1));
            u32 b = wide ? read64(op(2)) : read(op(2));
            u32 v;
            if (r == R_ANDN2)
                v = K.E.binary(O_AND, a, K.E.unary(U_BITNOT, b, t), t);
            else if (r == R_AND)
                v = K.E.binary(O_AND, a, b, t);
            else if (r == R_OR)
                v = K.E.binary(O_OR, a, b, t);
            else
                v = K.E.binary(O_XOR, a, b, t);
            write(op(0), v, t);
            invalidate_slot(K, kRegIdScc, 1);
            return true;
        }
        case R_LSHL:
        case R_LSHR:
        case R_ASHR:
            if (nn < 3)
                return false;
            {
            DT t = suffix_type0(I, DT_B32);
            const bool wide = dt_bits(t) == 64;
            u32 a = wide ? read64(op(1)) : read(op(1));
            u32 b = read(op(2));
            u32 o = r == R_LSHL ? O_SHL : (r == R_LSHR ? O_LSHR : O_ASHR);
            write(op(0), K.E.binary(o, a, b, t), t);
            invalidate_slot(K, kRegIdScc, 1);
            return true;
        }
        default:
            break;
        }
        if (I.rflags & RF_CMP)
            return compare(false);
        if (r == R_AND_SAVEEXEC)
            return false;
        if (r == R_WAITCNT || r == R_NOP || r == R_ENDPGM || r == R_BRANCH || (I.rflags & RF_CBRANCH))
            return true;
        return false;
    }

    OD_INL u32 mask24(u32 e) {
        return K.E.binary(O_AND, e, K.E.constant(0xffffff, DT_U32), DT_U32);
    }

    // src24_kind  sym_state.cpp:563-568: 0 none, 1 unsigned, 2 signed
    OD_INL u32 src24() const {
        for (u32 k = 0; k < 2; ++k) {
            u32 s = I.sfx[k];
            if (!s)
                break;
            if (sfx_bits(s) == 24)
                return sfx_base(s) == SB_I ? 2 : 1;
        }
        return 0;
    }

    // handle_vector  sym_state.cpp:577-769
    OD_NOINL bool vector() {
        const u32 r = I.root;
        const u32 nn = n();
        // one jump table instead of a chain of tests spread over the handlers
        // (the lowering pass is bound by instruction fetch)
        switch (r) {
        case R_MOV:
            if (nn < 2)
                return false;
            {
            u32 v = read(op(1));
            write(op(0), v, v ? ty(v) : DT_B32);
            return true;
        }
        case R_CNDMASK:
            if ((I.flags & IF_PARSE_FAILED) || nn < 4 || !op_is_vreg(op(0)))
                return false;
            {
            u32 cond = read(op(3));
            u32 a = read(op(1));
            u32 b = read(op(2));
            DT t = b ? ty(b) : DT_B32;
            write(op(0), K.E.ternary(cond, b, a, t), t);
            return true;
        }
        case R_ADD:
        case R_SUB:
        case R_SUBREV:
            if (nn < 3)
                return false;
            {
            u32 src0 = 1;
            bool carry = false;
            if (op_is_special(op(1), SP_VCC) || op_is_sreg_pair(op(1))) {
                src0 = 2;
                carry = true;
            }
            if (nn < src0 + 2)
                return false;
            DT t = suffix_type0(I, DT_U32);
            u32 a = rd(src0, t);
            u32 b = rd(src0 + 1, t);
            if (r == R_SUBREV) {
                u32 x = a;
                a = b;
                b = x;
            }
            u32 o = r == R_ADD ? O_ADD : O_SUB;
            u32 value = K.E.binary(o, a, b, t);
            Pending pd;
            pd.valid = 0;
            pd.lo_vgpr = pd.lo_version = 0;
            pd.base64 = pd.addend = 0;
            if (r == R_ADD && carry && op_is_vreg(op(0))) {
                u32 lo = 0, other = 0;
                if (a && K.E.n[a].kind == E_UNARY && K.E.n[a].op == U_LO32) {
                    lo = a;
                    other = b;
                } else if (b && K.E.n[b].kind == E_UNARY && K.E.n[b].op == U_LO32) {
                    lo = b;
                    other = a;
                }
                if (lo) {
                    pd.valid = 1;
                    pd.lo_vgpr = op(0).r.a;
                    pd.base64 = K.E.n[lo].a;
                    pd.addend = other;
                }
            }
            write(op(0), value, t);
            if (carry)
                invalidate_slot(K, operand_reg_id(op(1)), op(1).count);
            K.pend = pd;
            if (pd.valid)
                K.pend.lo_version = K.regs[kRegIdVgpr0 + pd.lo_vgpr].version;
            return true;
        }
        case R_ADDC:
            if (nn < 5)
                return false;
            {
            const Pending pd = K.pend;
            K.pend.valid = 0;
            K.pend.base64 = K.pend.addend = 0;
            K.pend.lo_vgpr = K.pend.lo_version = 0;
            DT t = suffix_type0(I, DT_U32);
            u32 x = read(op(2));
            u32 y = read(op(3));
            const bool cin_vcc = op_is_special(op(4), SP_VCC);
            if (pd.valid && cin_vcc && op_is_vreg(op(0)) && op(0).r.a == pd.lo_vgpr + 1 &&
                K.regs[kRegIdVgpr0 + pd.lo_vgpr].version == pd.lo_version) {
                u32 hi = 0, zero = 0;
                if (x && K.E.n[x].kind == E_UNARY && K.E.n[x].op == U_HI32 &&
                    expr_equal(K.E, K.E.n[x].a, pd.base64, K.eqst)) {
                    hi = x;
                    zero = y;
                } else if (y && K.E.n[y].kind == E_UNARY && K.E.n[y].op == U_HI32 &&
                           expr_equal(K.E, K.E.n[y].a, pd.base64, K.eqst)) {
                    hi = y;
                    zero = x;
                }
                if (hi && zero && K.E.is_const_v(zero, 0)) {
                    u32 add64 = K.E.unary(U_CAST, pd.addend, DT_U64);
                    u32 joint = K.E.binary(O_ADD, pd.base64, add64, DT_U64);
                    u32 lo_id = kRegIdVgpr0 + pd.lo_vgpr;
                    if (lo_id + 1 >= kRegIdExecLo) {
                        K.oom = true;
                        return true;
                    }
                    log_slot(K, lo_id);
                    Slot &lo = K.regs[lo_id];
                    lo.expr = joint;
                    lo.integ = IN_LOW;
                    lo.type = DT_U64;
                    log_slot(K, lo_id + 1);
                    Slot &hs = K.regs[lo_id + 1];
                    hs.version += 1;
                    hs.expr = joint;
                    hs.integ = IN_HIGH;
                    hs.type = DT_U64;
                    invalidate_slot(K, operand_reg_id(op(1)), op(1).count);
                    return true;
                }
            }
            diag(K, DG_ADDC, I.line);
            u32 v = K.E.binary(O_ADD, coerce(x, t), coerce(y, t), t);
            write(op(0), v, t);
            invalidate_slot(K, operand_reg_id(op(1)), op(1).count);
            return true;
        }
        case R_MUL:
        case R_MUL_LO:
        case R_MUL_HI:
            if (nn < 3)
                return false;
            {
            const u32 narrow = src24();
            if (narrow == 2)
                return false;
            DT t = suffix_type0(I, DT_U32);
            u32 o = O_MUL;
            if (r == R_MUL_HI)
                o = dt_is_signed(t) ? O_MULHIS : O_MULHI;
            if (narrow != 1) {
                bin(o, t, 1, 2);
                return true;
            }
            u32 a = rd(1, t);
            u32 b = rd(2, t);
            a = mask24(a);
            b = mask24(b);
            write(op(0), K.E.binary(o, a, b, t), t);
            return true;
        }
        case R_MAC:
            if (nn < 3)
                return false;
            {
            DT t = suffix_type0(I, DT_F32);
            u32 a = rd(1, t);
            u32 b = rd(2, t);
            u32 d = rd(0, t);
            u32 v = K.E.binary(O_ADD, K.E.binary(O_MUL, a, b, t), d, t);
            write(op(0), v, t);
            return true;
        }
        case R_MAD:
            if (nn < 4)
                return false;
            {
            const u32 narrow = src24();
            if (narrow == 2)
                return false;
            DT t = suffix_type0(I, DT_F32);
            u32 a = rd(1, t);
            u32 b = rd(2, t);
            u32 c = rd(3, t);
            if (narrow == 1) {
                a = mask24(a);
                b = mask24(b);
            }
            u32 v = K.E.binary(O_ADD, K.E.binary(O_MUL, a, b, t), c, t);
            write(op(0), v, t);
            return true;
        }
        case R_LSHLREV:
        case R_LSHRREV:
        case R_ASHRREV:
        case R_LSHL:
        case R_LSHR:
        case R_ASHR:
            if (nn < 3)
                return false;
            {
            const bool rev = r == R_LSHLREV || r == R_LSHRREV || r == R_ASHRREV;
            u32 shift = read(op(rev ? 1 : 2));
            u32 value = read(op(rev ? 2 : 1));
            DT t = (r == R_ASHR || r == R_ASHRREV) ? DT_I32 : suffix_type0(I, DT_B32);
            u32 o = O_SHL;
            if (I.rflags & RF_LSHR)
                o = O_LSHR;
            else if (I.rflags & RF_ASHR)
                o = O_ASHR;
            write(op(0), K.E.binary(o, coerce(value, t), shift, t), t);
            return true;
        }
        case R_AND:
        case R_OR:
        case R_XOR:
            if (nn < 3)
                return false;
            {
            bin(r == R_AND ? O_AND : r == R_OR ? O_OR : O_XOR, suffix_type0(I, DT_B32), 1, 2);
            return true;
        }
        default:
            break;
        }
        if (I.rflags & RF_CMP)
            return compare(true);
        return false;
    }

    // pointer_base  sym_state.cpp:323-340 (pre-order, left first)
    OD_NOINL DT pointee_of(u32 addr) {
        U32Stack &st = K.eqst;
        u32 base = st.top;
        st.push(addr);
        u32 hit = 0;
        while (st.top > base && !st.oom) {
            u32 e = st.pop();
            if (!e)
                continue;
            const ENode &x = K.E.n[e];
            if (x.kind == E_ARG && dt_is_pointer(x.type)) {
                hit = e;
                break;
            }
            if (x.kind == E_BINARY && x.op == O_ADD) {
                st.push(x.b);
                st.push(x.a);
            } else if (x.kind == E_UNARY && x.op == U_CAST) {
                st.push(x.a);
            }
        }
        st.top = base;
        return hit ? dt_pointee(K.E.n[hit].type) : DT_B32;
    }

    // do_flat_load  sym_state.cpp:771-792
    OD_NOINL void flat_load(u32 dwords) {
        if (n() < 2)
            return fallback();
        const Opnd &dst = op(0);
        u32 addr = read64(op(1));
        DT elem = pointee_of(addr);
        if (dwords == 2 && dt_byte_size(elem) == 8) {
            u32 v = K.E.deref(addr, elem, AS_GLOBAL);
            write_pair_ids(K, kRegIdVgpr0 + dst.r.a, v, elem);
            return;
        }
        DT e32 = dt_byte_size(elem) == 4 ? elem : DT_B32;
        for (u32 i = 0; i < dwords; ++i) {
            u32 a = i == 0 ? addr : K.E.binary(O_ADD, addr, K.E.constant(4 * i, DT_U64), DT_U64);
            u32 v = K.E.deref(a, e32, AS_GLOBAL);
            write_slot32(K, kRegIdVgpr0 + dst.r.a + i, v, e32);
        }
    }

    // do_flat_store  sym_state.cpp:794-827
    OD_NOINL void flat_store(u32 dwords) {
        if (n() < 2)
            return fallback();
        u32 addr = read64(op(0));
        const Opnd data = op(1);
        DT elem = pointee_of(addr);
        if (dwords == 2 && dt_byte_size(elem) == 8 && data.count >= 2) {
            push_store(addr, read64(data), elem);
            return;
        }
        DT e32 = dt_byte_size(elem) == 4 ? elem : DT_B32;
        for (u32 i = 0; i < dwords; ++i) {
            u32 a = i == 0 ? addr : K.E.binary(O_ADD, addr, K.E.constant(4 * i, DT_U64), DT_U64);
            Opnd piece = data;
            if (piece.kind == OK_SREG || piece.kind == OK_VREG)
                piece.r.a = data.r.a + i;
            piece.count = 1;
            push_store(a, read(piece), e32);
        }
    }

    OD_NOINL bool flat() {
        switch (I.root) {
        case R_LOAD_DWORD: return flat_load(1), true;
        case R_LOAD_DWORDX2: return flat_load(2), true;
        case R_STORE_DWORD: return flat_store(1), true;
        case R_STORE_DWORDX2: return flat_store(2), true;
        default: return false;
        }
    }

    // step  sym_state.cpp:840-864
    OD_INL void run() {
        if (I.flags & IF_PARSE_FAILED) {
            fallback();
            return;
        }
        bool handled = false;
        if (I.prefix == PX_S)
            handled = scalar();
        else if (I.prefix == PX_V)
            handled = vector();
        else if (I.prefix == PX_FLAT)
            handled = flat();
        if (!handled)
            fallback();
        if (!(I.prefix == PX_V && (I.root == R_ADD || I.root == R_ADDC))) {
            K.pend.valid = 0;
            K.pend.base64 = K.pend.addend = 0;
            K.pend.lo_vgpr = K.pend.lo_version = 0;
        }
    }
};

// lower_block  lower.cpp:29-49
OD_NOINL void lower_block(KCtx &K, u32 b, u32 out) {
    const Block &B = K.blk[b];
    for (u32 i = B.ib; i < B.ie && !K.oom && !K.E.oom; ++i) {
        if (K.supp[i])
            continue;
        const Ins &I = K.ins[i];
        Step s{K, I, out, K.in->ops + I.op_start, (I.flags & IF_SYNTH) ? 0u : (u32)I.nops};
        s.run();
    }
}

// taken_cond  lower.cpp:53-87
OD_NOINL u32 taken_cond(KCtx &K, u32 cc, const Opnd &ms) {
    switch (cc) {
    case C_SCC0:
    case C_SCC1: {
        u32 e = K.regs[362].expr;
        if (!e)
            e = bind_fresh(K, 362, DT_B32);
        return cc == C_SCC1 ? e : negate_condition(K.E, e);
    }
    case C_VCCZ:
    case C_VCCNZ: {
        u32 e = bind_fresh(K, 361, DT_B64);
        return cc == C_VCCNZ ? e : negate_condition(K.E, e);
    }
    case C_MASKED: {
        u32 src = (ms.count >= 2 || ms.kind == OK_SPECIAL) ? read_pair(K, ms) : read_operand(K, ms);
        return negate_condition(K.E, src);
    }
    default: return 0;
    }
}

OD_INL void reset_slot(Slot &s) {
    s.version = 0;
    s.expr = 0;
    s.type = DT_UNKNOWN;
    s.integ = IN_ENTIRE;
}

// Every slot to the RegisterFile default (once per kernel, at pool carving).
OD_INL void full_register_init(KCtx &K) {
    for (u32 p = 0; p < kPhysSlots; ++p)
        reset_slot(K.regs[p]);
    for (u32 w = 0; w < kLiveWords; ++w)
        K.dirty[w] = 0;
}

// A default RegisterFile: only the slots written since the last reset (every
// write goes through log_slot, which marks them) are cleared — lower_goto
// restarts from this state at every block (lower.cpp:204-206).
OD_INL void initial_register_state(KCtx &K) {
    for (u32 w = 0; w < kLiveWords; ++w) {
        u32 m = K.dirty[w];
        K.dirty[w] = 0;
        while (m) {
            u32 b = ctz32(m);
            m &= m - 1;
            reset_slot(K.regs[w * 32 + b]);
        }
    }
    K.pend.valid = 0;
    K.pend.base64 = K.pend.addend = 0;
    K.pend.lo_vgpr = K.pend.lo_version = 0;
}

OD_INL void mark_dirty(KCtx &K, u32 p) { K.dirty[p >> 5] |= 1u << (p & 31); }

// initial_register_state  abi_model.cpp:253-281
OD_NOINL void abi_entry_state(KCtx &K) {
    initial_register_state(K);
    u32 base = K.E.kbase();
    K.regs[4].expr = base;
    K.regs[4].integ = IN_LOW;
    K.regs[4].type = DT_U64;
    K.regs[5].expr = base;
    K.regs[5].integ = IN_HIGH;
    K.regs[5].type = DT_U64;
    for (u32 d = 0; d < K.cfg.dims; ++d) {
        K.regs[kRegIdVgpr0 + d].expr = K.E.builtin(F_LOCAL_ID, d, DT_U32);
        K.regs[kRegIdVgpr0 + d].type = DT_U32;
        K.regs[6 + d].expr = K.E.builtin(F_GROUP_ID, d, DT_U32);
        K.regs[6 + d].type = DT_U32;
    }
    K.regs[360].expr = K.E.constant(~0ull, DT_B64);
    K.regs[360].type = DT_B64;
    mark_dirty(K, 4);
    mark_dirty(K, 5);
    mark_dirty(K, 360);
    for (u32 d = 0; d < K.cfg.dims; ++d) {
        mark_dirty(K, kRegIdVgpr0 + d);
        mark_dirty(K, 6 + d);
    }
}

// Collects the slots touched since log position p0 as a sorted delta on the
// delta stack; returns (start, count).
// collect_delta on a lone lane (the lowering of most kernels).
OD_NOINL void collect_delta_seq(KCtx &K, u32 p0, u32 *start, u32 *count) {
    u32 bm[kLiveWords];
    for (u32 w = 0; w < kLiveWords; ++w)
        bm[w] = 0;
    for (u32 i = p0; i < K.nlog; ++i) {
        u32 p = K.log[i].phys();
        bm[p >> 5] |= 1u << (p & 31);
    }
    *start = K.ndstk;
    for (u32 w = 0; w < kLiveWords; ++w) {
        u32 m = bm[w];
        while (m) {
            u32 bit = ctz32(m);
            m &= m - 1;
            u32 p = w * 32 + bit;
            if (K.ndstk >= K.dstk_cap) {
                K.oom = true;
                *count = K.ndstk - *start;
                return;
            }
            K.dstk_id[K.ndstk] = p;
            K.dstk[K.ndstk] = K.regs[p];
            K.ndstk++;
            if (K.ndstk > K.dstk_hw)
                K.dstk_hw = K.ndstk;
        }
    }
    *count = K.ndstk - *start;
}


// The slots an arm touched (its undo-log entries from p0), ascending, with
// their current values, pushed on the delta stack.  Split across the lanes
// executing it: the log entries into per-lane slot bitmaps (OR-reduced), then
// one lane per bitmap word writes that word's entries at their prefix rank.
OD_NOINL void collect_delta(KCtx &K, u32 p0, u32 *start, u32 *count) {
    const u32 m = wmask(), r = wrank(m), nl = wsize(m);
    if (nl == 1) {
        collect_delta_seq(K, p0, start, count);
        return;
    }
    u32 bm[kLiveWords];
    for (u32 w = 0; w < kLiveWords; ++w)
        bm[w] = 0;
    for (u32 i = p0 + r; i < K.nlog; i += nl) {
        const u32 p = K.log[i].phys();
        bm[p >> 5] |= 1u << (p & 31);
    }
    u32 total = 0;
    for (u32 w = 0; w < kLiveWords; ++w) {
        bm[w] = wor(m, bm[w]);
        total += popc32(bm[w]);
    }
    *start = K.ndstk;
    const u32 room = K.dstk_cap > K.ndstk ? K.dstk_cap - K.ndstk : 0;
    const u32 n = total < room ? total : room;
    for (u32 w = r; w < kLiveWords; w += nl) {
        u32 q = 0;
        for (u32 v = 0; v < w; ++v)
            q += popc32(bm[v]);
        for (u32 bits = bm[w]; bits && q < n; bits &= bits - 1, ++q) {
            const u32 p = w * 32 + ctz32(bits);
            K.dstk_id[K.ndstk + q] = p;
            K.dstk[K.ndstk + q] = K.regs[p];
        }
    }
    wsync(m);
    if (n < total)
        K.oom = true; // the kernel is re-run with a larger arena
    K.ndstk += n;
    if (K.ndstk > K.dstk_hw)
        K.dstk_hw = K.ndstk;
    *count = n;
}

OD_INL u32 half_view(KCtx &K, const Slot &s) {
    if (s.integ == IN_LOW)
        return K.E.unary(U_LO32, s.expr, DT_B32);
    if (s.integ == IN_HIGH)
        return K.E.unary(U_HI32, s.expr, DT_B32);
    return s.expr;
}

// merge_join on a lone lane: one pass in slot order.
OD_NOINL void merge_join_seq(KCtx &K, const Frame &F, u32 td, u32 tn, u32 ed, u32 en, bool has_else,
                       const u32 *live) {
    u32 i = 0, j = 0;
    while (i < tn || j < en) {
        u32 pt = i < tn ? K.dstk_id[td + i] : 0xffffffffu;
        u32 pe = j < en ? K.dstk_id[ed + j] : 0xffffffffu;
        u32 p = pt < pe ? pt : pe;
        Slot a = K.regs[p], b = K.regs[p];
        if (pt == p) {
            a = K.dstk[td + i];
            ++i;
        }
        if (pe == p) {
            b = K.dstk[ed + j];
            ++j;
        }
        Slot m = a; // merged starts as the then state
        if (p == 360) {
            // exec halves are skipped: the then side passes through
        } else if (a.version == b.version &&
                   (!a.expr || !b.expr || expr_equal(K.E, a.expr, b.expr, K.eqst))) {
            if (!a.expr && b.expr)
                m = b;
        } else {
            u32 top = a.version > b.version ? a.version : b.version;
            u32 id = dense_of_phys(p);
            if (!lv_test(live, id)) {
                m.version = top;
                m.expr = 0;
                m.type = DT_UNKNOWN;
                m.integ = IN_ENTIRE;
            } else {
                u32 tv, ev;
                if (p >= 361) { // vcc, scc, m0: raw slot expressions
                    tv = a.expr;
                    ev = b.expr;
                } else {
                    tv = a.expr ? half_view(K, a) : 0;
                    ev = b.expr ? half_view(K, b) : 0;
                }
                DT vt = DT_B32;
                if (tv && ev)
                    vt = dt_unify(K.E.n[tv].type, K.E.n[ev].type);
                else if (tv)
                    vt = K.E.n[tv].type;
                else if (ev)
                    vt = K.E.n[ev].type;
                if (dt_is_unknown(vt) || dt_is_pointer(vt))
                    vt = dt_bits(vt) == 64 ? DT_B64 : DT_B32;
                u32 serial = top + 1;
                while (!K.pool.insert(p, serial))
                    ++serial;
                // emit_join for this fixup
                u32 d = new_stmt(K, SK_DECL);
                K.st[d].cls = (u16)p;
                K.st[d].a = serial;
                K.st[d].c = vt;
                if (!has_else && ev)
                    K.st[d].b = ev;
                list_append(K, F.out, d);
                if (tv) {
                    u32 s = new_stmt(K, SK_ASSIGN);
                    K.st[s].cls = (u16)p;
                    K.st[s].a = serial;
                    K.st[s].b = tv;
                    list_append(K, F.then_l, s);
                }
                if (has_else && ev) {
                    u32 s = new_stmt(K, SK_ASSIGN);
                    K.st[s].cls = (u16)p;
                    K.st[s].a = serial;
                    K.st[s].b = ev;
                    list_append(K, F.else_l, s);
                }
                m.version = top + 1;
                m.expr = K.E.var(p, serial, vt);
                m.type = vt;
                m.integ = IN_ENTIRE;
            }
        }
        log_slot(K, p);
        K.regs[p] = m;
    }
}


// The undo record of slot p at log position at (log_slot's record).
OD_INL void log_at(KCtx &K, u32 at, u32 p) {
    const uint4 v = *reinterpret_cast<const uint4 *>(&K.regs[p]);
    *reinterpret_cast<uint4 *>(&K.log[at]) = make_uint4(v.x, v.y, v.z, (v.w & 0xffu) | (p << 8));
}

// merge_at_join (sym_state.cpp:866-957) + emit_join (lower.cpp:89-121) for
// the union of touched slots.  regs must hold the split state S0.
// Split across the lanes executing it (north star (4)): the union of the two
// arms' sorted delta lists is a bitmap; each lane takes bitmap words, finds a
// slot's then / else values at its rank in each list, and settles the slots
// that pass through or die (not live at the join) itself.  The live joins,
// which mint names, statements and expressions in slot order, are then
// settled in ascending slot order as the reference does.  Undo records go
// to the log at each slot's rank in the union, the reference's order.
OD_NOINL void merge_join(KCtx &K, const Frame &F, u32 td, u32 tn, u32 ed, u32 en, bool has_else,
                         const u32 *live) {
    const u32 m = wmask(), r = wrank(m), nl = wsize(m);
    if (nl == 1) {
        merge_join_seq(K, F, td, tn, ed, en, has_else, live);
        return;
    }
    u32 Tm[kLiveWords], Em[kLiveWords], Jm[kLiveWords];
    for (u32 w = 0; w < kLiveWords; ++w)
        Tm[w] = Em[w] = Jm[w] = 0;
    for (u32 i = r; i < tn; i += nl) {
        const u32 p = K.dstk_id[td + i];
        Tm[p >> 5] |= 1u << (p & 31);
    }
    for (u32 j = r; j < en; j += nl) {
        const u32 p = K.dstk_id[ed + j];
        Em[p >> 5] |= 1u << (p & 31);
    }
    u32 nu = 0;
    for (u32 w = 0; w < kLiveWords; ++w) {
        Tm[w] = wor(m, Tm[w]);
        Em[w] = wor(m, Em[w]);
        nu += popc32(Tm[w] | Em[w]);
    }
    const u32 log0 = K.nlog;
    const bool logging = K.log_depth != 0;
    if (logging && log0 + nu > K.log_cap)
        K.oom = true; // the kernel is re-run with a larger arena
    const bool rec = logging && !K.oom;
    auto sides = [&](u32 w, u32 bit, u32 rt, u32 re, Slot *a, Slot *b) {
        const u32 p = w * 32 + bit, below = (1u << bit) - 1;
        *a = (Tm[w] >> bit) & 1 ? K.dstk[td + rt + popc32(Tm[w] & below)] : K.regs[p];
        *b = (Em[w] >> bit) & 1 ? K.dstk[ed + re + popc32(Em[w] & below)] : K.regs[p];
    };
    for (u32 w = r; w < kLiveWords; w += nl) {
        u32 rt = 0, re = 0, ru = 0; // list ranks before this word
        for (u32 v = 0; v < w; ++v) {
            rt += popc32(Tm[v]);
            re += popc32(Em[v]);
            ru += popc32(Tm[v] | Em[v]);
        }
        const u32 U = Tm[w] | Em[w];
        u32 jm = 0;
        for (u32 bits = U; bits; bits &= bits - 1) {
            const u32 bit = ctz32(bits), p = w * 32 + bit;
            Slot a, b;
            sides(w, bit, rt, re, &a, &b);
            Slot mg = a; // merged starts as the then state
            if (p == 360) {
                // exec halves are skipped: the then side passes through
            } else if (a.version == b.version && (!a.expr || !b.expr || a.expr == b.expr)) {
                if (!a.expr && b.expr)
                    mg = b;
            } else if (a.version == b.version) {
                jm |= 1u << bit; // structural comparison (one shared scratch stack): settled below
                continue;
            } else {
                const u32 top = a.version > b.version ? a.version : b.version;
                if (lv_test(live, dense_of_phys(p))) {
                    jm |= 1u << bit; // live: settled below, in slot order
                    continue;
                }
                mg.version = top;
                mg.expr = 0;
                mg.type = DT_UNKNOWN;
                mg.integ = IN_ENTIRE;
            }
            if (rec)
                log_at(K, log0 + ru + popc32(U & ((1u << bit) - 1)), p);
            K.regs[p] = mg;
        }
        Jm[w] = jm;
    }
    for (u32 w = 0; w < kLiveWords; ++w) {
        Jm[w] = wor(m, Jm[w]);
        K.dirty[w] |= Tm[w] | Em[w];
    }
    wsync(m);
    // the live joins and the structural comparisons, ascending (names,
    // statements and expressions are minted in this order)
    u32 rt = 0, re = 0, ru = 0;
    for (u32 w = 0; w < kLiveWords; ++w) {
        const u32 U = Tm[w] | Em[w];
        for (u32 bits = Jm[w]; bits; bits &= bits - 1) {
            const u32 bit = ctz32(bits), p = w * 32 + bit;
            Slot a, b;
            sides(w, bit, rt, re, &a, &b);
            Slot mg = a;
            const u32 top = a.version > b.version ? a.version : b.version;
            const u32 at = log0 + ru + popc32(U & ((1u << bit) - 1));
            if (a.version == b.version) {
                if (expr_equal(K.E, a.expr, b.expr, K.eqst)) { // pass-through
                    if (rec)
                        log_at(K, at, p);
                    K.regs[p] = mg;
                    continue;
                }
                if (!lv_test(live, dense_of_phys(p))) { // dies at the join
                    mg.version = top;
                    mg.expr = 0;
                    mg.type = DT_UNKNOWN;
                    mg.integ = IN_ENTIRE;
                    if (rec)
                        log_at(K, at, p);
                    K.regs[p] = mg;
                    continue;
                }
            }
            u32 tv, ev;
            if (p >= 361) { // vcc, scc, m0: raw slot expressions
                tv = a.expr;
                ev = b.expr;
            } else {
                tv = a.expr ? half_view(K, a) : 0;
                ev = b.expr ? half_view(K, b) : 0;
            }
            DT vt = DT_B32;
            if (tv && ev)
                vt = dt_unify(K.E.n[tv].type, K.E.n[ev].type);
            else if (tv)
                vt = K.E.n[tv].type;
            else if (ev)
                vt = K.E.n[ev].type;
            if (dt_is_unknown(vt) || dt_is_pointer(vt))
                vt = dt_bits(vt) == 64 ? DT_B64 : DT_B32;
            u32 serial = top + 1;
            while (!K.pool.insert(p, serial))
                ++serial;
            // emit_join for this fixup
            u32 d = new_stmt(K, SK_DECL);
            K.st[d].cls = (u16)p;
            K.st[d].a = serial;
            K.st[d].c = vt;
            if (!has_else && ev)
                K.st[d].b = ev;
            list_append(K, F.out, d);
            if (tv) {
                u32 st = new_stmt(K, SK_ASSIGN);
                K.st[st].cls = (u16)p;
                K.st[st].a = serial;
                K.st[st].b = tv;
                list_append(K, F.then_l, st);
            }
            if (has_else && ev) {
                u32 st = new_stmt(K, SK_ASSIGN);
                K.st[st].cls = (u16)p;
                K.st[st].a = serial;
                K.st[st].b = ev;
                list_append(K, F.else_l, st);
            }
            mg.version = top + 1;
            mg.expr = K.E.var(p, serial, vt);
            mg.type = vt;
            mg.integ = IN_ENTIRE;
            if (rec)
                log_at(K, at, p);
            K.regs[p] = mg;
        }
        rt += popc32(Tm[w]);
        re += popc32(Em[w]);
        ru += popc32(U);
    }
    if (rec) {
        K.nlog = log0 + nu;
        if (K.nlog > K.log_hw)
            K.log_hw = K.nlog;
    }
}

OD_INL u32 push_frame(KCtx &K, u32 region, u32 out) {
    if (K.nframes >= K.frames_cap) {
        K.oom = true;
        return 0;
    }
    Frame &F = K.frames[K.nframes++];
    F.region = region;
    F.phase = 0;
    F.out = out;
    F.then_l = F.else_l = 0;
    F.cond = 0;
    F.child = 0;
    F.then_d = F.then_n = 0;
    return 1;
}

// lower_region  lower.cpp:123-172, iterative.
OD_NOINL void lower_structured(KCtx &K, u32 root, u32 out) {
    abi_entry_state(K);
    K.nframes = 0;
    push_frame(K, root, out);
    while (K.nframes && !K.oom && !K.E.oom) {
        Frame &F = K.frames[K.nframes - 1];
        const Region &R = K.rg[F.region];
        if (R.kind == RK_BLOCK) {
            u32 o = F.out;
            K.nframes--;
            lower_block(K, (u32)R.block_id, o);
            continue;
        }
        if (R.kind == RK_LINEAR) {
            if (F.child < R.ch_n) {
                u32 c = K.child[R.ch_b + F.child++];
                push_frame(K, c, F.out);
            } else {
                K.nframes--;
            }
            continue;
        }
        const bool has_else = R.kind == RK_IFELSE;
        if (F.phase == 0) {
            F.phase = 1;
            push_frame(K, K.child[R.ch_b], F.out);
            continue;
        }
        if (F.phase == 1) {
            u32 taken = taken_cond(K, R.cc, R.mask_source);
            u32 cond = R.then_is_taken ? taken : negate_condition(K.E, taken);
            F.cond = cond;
            F.log_p0 = K.nlog;
            F.pend = K.pend;
            F.dstk_p0 = K.ndstk;
            F.then_l = new_list(K);
            F.else_l = new_list(K);
            K.log_depth++;
            F.phase = 2;
            push_frame(K, K.child[R.ch_b + 1], F.then_l);
            continue;
        }
        if (F.phase == 2) {
            collect_delta(K, F.log_p0, &F.then_d, &F.then_n);
            undo_to(K, F.log_p0);
            K.pend = F.pend;
            F.phase = 3;
            if (has_else) {
                push_frame(K, K.child[R.ch_b + 2], F.else_l);
                continue;
            }
        }
        // phase 3: both arms lowered
        u32 ed, en;
        collect_delta(K, F.log_p0, &ed, &en);
        undo_to(K, F.log_p0);
        K.log_depth--;
        const u32 *live = K.live_in + (u32)R.join_block * kLiveWords;
        merge_join(K, F, F.then_d, F.then_n, ed, en, has_else, live);
        K.pend.valid = 0;
        K.pend.base64 = K.pend.addend = 0;
        K.pend.lo_vgpr = K.pend.lo_version = 0;
        u32 s = new_stmt(K, SK_IF);
        K.st[s].a = F.cond;
        K.st[s].b = K.lists[F.then_l].head;
        K.st[s].c = K.lists[F.else_l].head;
        list_append(K, F.out, s);
        K.ndstk = F.dstk_p0;
        u32 out2 = F.out;
        u32 join = R.join_absorbed ? K.child[R.ch_b + R.ch_n - 1] : 0;
        K.nframes--;
        if (join)
            push_frame(K, join, out2);
    }
}

// lower_goto_form  lower.cpp:187-250
OD_NOINL void lower_goto(KCtx &K, u32 out) {
    diag(K, DG_GOTO, 0);
    for (u32 k = 0; k < K.nblk && !K.oom && !K.E.oom; ++k) {
        u32 id = k;
        if (k > 0 && (!blk_reach(K, id) || K.blk[id].absorbed))
            continue;
        const Block &B = K.blk[id];
        u32 l = new_stmt(K, SK_LABEL);
        K.st[l].a = id;
        list_append(K, out, l);
        if (id == 0)
            abi_entry_state(K);
        else
            initial_register_state(K);
        lower_block(K, id, out);
        const Term &t = B.term;
        if (t.kind == T_FALL || t.kind == T_UNCOND) {
            u32 g = new_stmt(K, SK_GOTO);
            K.st[g].c = (u32)t.taken;
            list_append(K, out, g);
        } else if (t.kind == T_COND) {
            u32 cond = taken_cond(K, t.cc, t.mask_source);
            if (!cond) {
                diag(K, DG_EXEC_BRANCH, t.line);
                const Ins &last = K.ins[B.ie - 1];
                u32 r = new_stmt(K, SK_RAW);
                K.st[r].a = last.src.off;
                K.st[r].b = last.src.len;
                list_append(K, out, r);
                K.fallbacks++;
            } else {
                u32 g = new_stmt(K, SK_GOTO);
                K.st[g].a = cond;
                K.st[g].c = (u32)t.taken;
                list_append(K, out, g);
            }
            u32 g2 = new_stmt(K, SK_GOTO);
            K.st[g2].c = (u32)(t.not_taken >= 0 ? t.not_taken : t.taken);
            list_append(K, out, g2);
        }
    }
}

// ------------------------------------------------------------ emission
OD_INL void put_block_label(KCtx &K, Writer &w, u32 b) {
    const Block &B = K.blk[b];
    if (B.lab_n) {
        const Label &L = klabel(K, B.lab_b);
        w.putn(K.in->t + L.off, L.len);
    } else {
        w.lit("bb");
        w.put_u64(b);
    }
}

// ----------------------------------------------------- body export (step -3)
// DecompiledKernel::body (LoweredBody, lower.hpp:20-41) as text, for callers
// that need the statement tree itself (the drop-in binding rebuilds it;
// acceptance_main.cpp's differential gate evaluates it).  Expression nodes
// are printed once each, children first, and referenced by their 1-based
// export number (0 = null); every statement follows the nodes it uses:
//   N kind op x type a b c [len name]   (kind/op/x/type as ExprKind+1 / op /
//        builtin dim / DataType base|bits<<8|depth<<16|space<<24; a b c are
//        child numbers, or a const's low / high words; Var / KernelArg carry
//        their rendered name)
//   A len name value | D len name type value | W addr value elem_type
//   R len text | I cond ... E ... F | L len label | G cond len label
OD_INL void exp_name(DotSink &o, const u8 *b, u32 n) {
    o.u(n);
    o.c(' ');
    o.m(b, n);
}

// Exports the node DAG under root; returns its export number.
OD_NOINL u32 exp_node(KCtx &K, DotSink &o, u32 root, u32 tag, u32 *nid) {
    const u32 kMask = 0x3fffffffu, kTags = 0xc0000000u;
    EArena &E = K.E;
    if (!root)
        return 0;
    if ((E.n[root].memo & kTags) == tag)
        return E.n[root].memo & kMask;
    TaskStack &ts = K.rc.ts;
    const u32 base = ts.top;
    ts.push(0, 0, root);
    while (ts.top > base && !ts.oom) {
        u64 &tk = ts.p[ts.top - 1];
        const u32 e = (u32)(tk >> 32), st = (u32)(tk & 0xff);
        const ENode x = E.n[e];
        u32 ch[3] = {0, 0, 0}, nch = 0;
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
        if (st < nch) {
            tk = (tk & ~0xffull) | (st + 1);
            const u32 c = ch[st];
            if (c && (E.n[c].memo & kTags) != tag)
                ts.push(0, 0, c);
            continue;
        }
        ts.top--;
        if ((E.n[e].memo & kTags) == tag) // reached twice through the stack
            continue;
        u32 cid[3] = {0, 0, 0};
        for (u32 k = 0; k < nch; ++k)
            cid[k] = ch[k] ? (E.n[ch[k]].memo & kMask) : 0;
        o.c('N');
        o.c(' ');
        o.u(x.kind);
        o.c(' ');
        o.u(x.op);
        o.c(' ');
        o.u(x.x);
        o.c(' ');
        o.u(x.type);
        o.c(' ');
        if (x.kind == E_CONST) {
            o.u(x.a);
            o.c(' ');
            o.u(x.b);
            o.c(' ');
            o.u(0);
        } else {
            o.u(nch > 0 ? cid[0] : x.a);
            o.c(' ');
            o.u(cid[1]);
            o.c(' ');
            o.u(cid[2]);
        }
        if (x.kind == E_VAR || x.kind == E_ARG) {
            u8 buf[64];
            Writer w{buf, 0, sizeof buf, false};
            if (x.kind == E_VAR)
                put_var_name(w, x.x, x.a);
            else
                put_arg_name(w, K.rc, x.a);
            o.c(' ');
            exp_name(o, buf, w.n < sizeof buf ? w.n : (u32)sizeof buf);
        }
        o.c('\n');
        E.n[e].memo = tag | ++*nid;
    }
    ts.top = base;
    return E.n[root].memo & kMask;
}

OD_NOINL void body_text(KCtx &K, DotSink &o) {
    const u32 tag = (K.exp_pass++ & 1) ? 0x80000000u : 0x40000000u;
    u32 nid = 0;
    TaskStack &ts = K.rc.ts;
    const u32 base = ts.top;
    for (u32 li = 0; li < 2; ++li) {
        // statement frames: (stmt, state) with state 0 new, 1 then done, 2 else done
        ts.push(0, 0, K.lists[K.exp_lists[li]].head);
        const u32 lbase = ts.top - 1;
        while (ts.top > lbase && !ts.oom) {
            u64 &fr = ts.p[ts.top - 1];
            const u32 si = (u32)(fr >> 32), state = (u32)(fr & 0xff);
            if (!si) {
                ts.top--;
                continue;
            }
            const Stmt S = K.st[si];
            u8 buf[64];
            Writer w{buf, 0, sizeof buf, false};
            if (S.kind == SK_IF) {
                if (state == 0) {
                    const u32 c = exp_node(K, o, S.a, tag, &nid);
                    o.s("I ");
                    o.u(c);
                    o.c('\n');
                    fr = (fr & ~0xffull) | 1;
                    ts.push(0, 0, S.b);
                } else if (state == 1 && S.c) {
                    o.s("E\n");
                    fr = (fr & ~0xffull) | 2;
                    ts.push(0, 0, S.c);
                } else {
                    o.s("F\n");
                    fr = ((u64)S.next << 32);
                }
                continue;
            }
            switch (S.kind) {
            case SK_ASSIGN: {
                const u32 v = exp_node(K, o, S.b, tag, &nid);
                put_var_name(w, S.cls, S.a);
                o.s("A ");
                exp_name(o, buf, w.n);
                o.c(' ');
                o.u(v);
                break;
            }
            case SK_DECL: {
                const u32 v = exp_node(K, o, S.b, tag, &nid);
                put_var_name(w, S.cls, S.a);
                o.s("D ");
                exp_name(o, buf, w.n);
                o.c(' ');
                o.u(dt_with_space(S.c, AS_NONE));
                o.c(' ');
                o.u(v);
                break;
            }
            case SK_STORE: {
                const u32 ad = exp_node(K, o, S.a, tag, &nid);
                const u32 v = exp_node(K, o, S.b, tag, &nid);
                o.s("W ");
                o.u(ad);
                o.c(' ');
                o.u(v);
                o.c(' ');
                o.u(S.c);
                break;
            }
            case SK_RAW: {
                const u8 *p = K.in->t + S.a;
                u32 b = 0, e = S.b;
                while (b < e && (p[b] == ' ' || p[b] == '\t'))
                    ++b;
                while (e > b && (p[e - 1] == ' ' || p[e - 1] == '\t'))
                    --e;
                o.s("R ");
                exp_name(o, p + b, e - b);
                break;
            }
            case SK_LABEL:
                put_block_label(K, w, S.a);
                o.s("L ");
                exp_name(o, buf, w.n);
                break;
            case SK_GOTO: {
                const u32 c = exp_node(K, o, S.a, tag, &nid);
                put_block_label(K, w, S.c);
                o.s("G ");
                o.u(c);
                o.c(' ');
                exp_name(o, buf, w.n);
                break;
            }
            default: break;
            }
            o.c('\n');
            fr = ((u64)S.next << 32);
        }
    }
    if (ts.oom)
        K.oom = true;
    ts.top = base;
}

// emit_statement  codegen.cpp:393-442 (one statement, no If bodies)
OD_NOINL void emit_simple(KCtx &K, Writer &w, const Stmt &s, u32 depth) {
    RenderCtx &rc = K.rc;
    u32 mark = K.E.top; // scratch nodes from render_indexed are discarded
    switch (s.kind) {
    case SK_ASSIGN:
        w.spaces(depth * 4);
        put_var_name(w, s.cls, s.a);
        w.lit(" = ");
        render_expr(w, rc, s.b, 0);
        w.lit(";\n");
        break;
    case SK_DECL:
        w.spaces(depth * 4);
        render_type(w, dt_with_space(s.c, AS_NONE));
        w.put(' ');
        put_var_name(w, s.cls, s.a);
        if (s.b) {
            w.lit(" = ");
            render_expr(w, rc, s.b, 0);
        }
        w.lit(";\n");
        break;
    case SK_STORE: {
        w.spaces(depth * 4);
        u32 target = K.E.deref(s.a, s.c, AS_GLOBAL);
        render_expr(w, rc, target, 0);
        w.lit(" = ");
        u32 v = s.b;
        if (v && is_bit_reinterpret(K.E.n[v].type, s.c)) {
            w.puts(cast_name(s.c));
            w.put('(');
            render_expr(w, rc, v, 0);
            w.put(')');
        } else {
            render_expr(w, rc, v, 0);
        }
        w.lit(";\n");
        break;
    }
    case SK_RAW: {
        w.spaces(depth * 4);
        w.lit("__asm volatile (\"");
        const u8 *p = K.in->t + s.a;
        u32 b = 0, e = s.b;
        while (b < e && (p[b] == ' ' || p[b] == '\t'))
            ++b;
        while (e > b && (p[e - 1] == ' ' || p[e - 1] == '\t'))
            --e;
        w.putn(p + b, e - b);
        w.lit("\");\n");
        break;
    }
    case SK_LABEL:
        put_block_label(K, w, s.a);
        w.lit(":;\n");
        break;
    case SK_GOTO:
        w.spaces(depth * 4);
        if (s.a) {
            w.lit("if (");
            render_expr(w, rc, s.a, 0);
            w.lit(") goto ");
        } else {
            w.lit("goto ");
        }
        put_block_label(K, w, s.c);
        w.lit(";\n");
        break;
    default: break;
    }
    K.E.top = mark;
}

// emit_body  codegen.cpp:378-381, iterative over nested If bodies.
OD_NOINL void emit_list(KCtx &K, Writer &w, u32 head, u32 depth, u32 *stk, u32 stk_cap) {
    // stack entries: (stmt, depth, state) triples
    u32 sp = 0;
    stk[0] = head;
    stk[1] = depth;
    stk[2] = 0;
    sp = 1;
    while (sp) {
        u32 *e = stk + 3 * (sp - 1);
        u32 s = e[0];
        if (!s) {
            --sp;
            continue;
        }
        const Stmt &S = K.st[s];
        u32 dp = e[1];
        if (S.kind != SK_IF) {
            emit_simple(K, w, S, dp);
            e[0] = S.next;
            continue;
        }
        if (e[2] == 0) {
            w.spaces(dp * 4);
            w.lit("if (");
            u32 mark = K.E.top;
            render_expr(w, K.rc, S.a, 0);
            K.E.top = mark;
            w.lit(") {\n");
            e[2] = 1;
            if (3 * (sp + 1) > stk_cap) {
                K.oom = true;
                return;
            }
            u32 *n = stk + 3 * sp;
            n[0] = S.b;
            n[1] = dp + 1;
            n[2] = 0;
            ++sp;
            continue;
        }
        if (e[2] == 1 && S.c) {
            w.spaces(dp * 4);
            w.lit("} else {\n");
            e[2] = 2;
            if (3 * (sp + 1) > stk_cap) {
                K.oom = true;
                return;
            }
            u32 *n = stk + 3 * sp;
            n[0] = S.c;
            n[1] = dp + 1;
            n[2] = 0;
            ++sp;
            continue;
        }
        w.spaces(dp * 4);
        w.lit("}\n");
        e[0] = S.next;
        e[2] = 0;
    }
}

// ------------------------------------------------------------ budgets
// Capacities of the dynamic pools for a kernel section of n lines, scaled by
// s on retry.  Measured high-water marks per line on the synthetic shapes
// (tools/devhost OD_USAGE): nodes <= 3, stmts <= 0.6, log <= 0.6,
// deltas <= 0.3, fresh <= 0.34, output <= 30 bytes.
struct PoolCaps {
    u32 nodes, stmts, log, dstk, fresh, names, stack, tasks, out;
};

OD_INL PoolCaps pool_caps(u32 n, u32 s) {
    PoolCaps c;
    c.nodes = s * (4 * n + 1024);
    c.stmts = s * (n + 256);
    c.log = s * (2 * n + 1024);
    c.dstk = s * (n + 1024);
    c.fresh = s * (n / 2 + 256);
    u32 want = 2 * (c.fresh + c.log / 2);
    u32 pw = 1024;
    while (pw < want)
        pw <<= 1;
    c.names = pw;
    c.stack = s * (n + 256);
    c.tasks = s * (n + 256);
    u64 out = (u64)s * (48ull * n + 8192);
    c.out = out > 0xfffff000ull ? 0xfffff000u : (u32)out;
    return c;
}

// Upper bound of the arena decompile_kernel needs for a kernel of sizes z at
// scale s (every allocation it makes, in order; regions <= 2 * blocks + 4).
// At s > 1 (a retry) the block bound falls back to one block per
// instruction.
// Diagnostics of one kernel: at most one per config line, two per
// instruction (operand / stepper warnings), two per block (unreachable note,
// mask or goto warning) and a few kernel-level ones.
OD_INL u32 diag_cap_of(u32 ncfg, u32 nins, u32 nb, u32 s) { return (ncfg + 2 * (nins + 1) + 2 * nb + 16) * (s ? s : 1); }
OD_INL u32 diag_cap(const KIn &in) {
    const u32 nb = in.nblk_cap ? in.nblk_cap : in.nins + 3;
    return diag_cap_of(in.ncfg, in.nins, nb, in.scale);
}

OD_INL u64 arena_budget(const KSize &z, u32 s) {
    const u64 ni = z.nins + 1;                                // + synthetic s_endpgm
    u64 b = ni + 2;                                           // blocks (build_cfg's cap)
    if (s <= 1 && z.nb < b)
        b = z.nb;
    const u64 r = 2 * b + 4;                                  // regions (build_regions' cap)
    u64 t = 0;
    t += (z.ncfg + 1) * (sizeof(KArg) + sizeof(Span));       // config
    t += (ni + 1) * sizeof(Ins) + (z.nlab + 1) * 4;           // instructions, labels
    t += (8 + z.ncfg + z.novr) * sizeof(AbiEntry);           // ABI map
    t += b * (sizeof(Block) + 4) + (2 * b + 4) * 4 + (ni + 1) + b * 8 + (b / 32 + 1) * 4; // blocks, stamps, work, supp, sx, rbits
    u64 lc = 16;
    while (lc < 2 * ((u64)z.nlab + 1))
        lc <<= 1;
    t += 2 * lc * 4;                                          // label map
    t += (r + 1) * sizeof(Region) + (4 * r + 8) * 4 + 9 * (r + 1) * 4 + (r / 64 + 2) * 8 +
         (2 * r + 4) * 4 * 3 + (b + 1) * 4;                   // regions, pred edge lists
    t += 3 * b * kLiveWords * 4;                              // liveness
    t += kPhysSlots * sizeof(Slot);
    const PoolCaps c = pool_caps(z.n, s);
    t += (u64)c.nodes * sizeof(ENode) + (u64)c.stmts * sizeof(Stmt) + (2 * r + 4) * sizeof(SList) +
         (2 * r + 8) * sizeof(Frame) + (u64)c.log * sizeof(UndoRec) + (u64)c.dstk * (sizeof(Slot) + 4) +
         (u64)c.fresh * sizeof(Fresh) + (u64)c.names * 8 + 3ull * c.stack * 4 + (u64)c.tasks * 8 +
         3 * (r + 8) * 4 + c.out;
    t += (u64)diag_cap_of(z.ncfg, z.nins, s <= 1 ? z.nb : z.nins + 3, s) * sizeof(Diag); // diagnostics
    t += 64 * 16; // per-allocation alignment
    return (t + 255) & ~255ull;
}

// ------------------------------------------------------------ driver
// decompile_section (decompiler.cpp:55-101) for one kernel, split into three
// phases so each device launch runs one phase's code (the instruction cache
// holds one phase, not the whole pipeline):
//   dk_front  parse_config .. liveness, pool carving
//   dk_lower  lower_kernel + hoist_fresh_decls
//   dk_emit   emit_kernel
// The per-kernel state persists between launches in a KState at the base of
// the kernel's arena slice; each phase copies it to local memory, re-points
// the self-references (kstate_fix) and writes it back.
#ifdef __CUDA_ARCH__
#define OD_CLK() clock64()
#define OD_PROF(i, t0)                                                                             \
    do {                                                                                           \
        if (in.prof) {                                                                             \
            long long t1_ = clock64();                                                             \
            if (wleader(wmask()))                                                                  \
                atomicAdd((unsigned long long *)&in.prof[i], (unsigned long long)(t1_ - t0));      \
            t0 = t1_;                                                                              \
        }                                                                                          \
    } while (0)
#else
#define OD_CLK() 0
#define OD_PROF(i, t0) (void)t0
#endif

struct KState {
    KIn in;
    Bump mem;
    KCtx K;
    KOut out;
    Writer w;
    u32 *estk;
    u32 ecap, body, hoist;
    u32 done; // out.status is final
};

OD_INL void kstate_fix(KState &S) {
    S.K.in = &S.in;
    S.K.mem = &S.mem;
    S.K.rc.E = &S.K.E;
    S.K.rc.cfg = &S.K.cfg;
}

// Initializes S for one kernel; mem must be the kernel's whole arena slice.
OD_INL void kstate_init(KState &S, const KIn &in, const Bump &mem) {
    memset(&S, 0, sizeof(S));
    S.in = in;
    S.mem = mem;
    S.out.status = KS_OK;
    kstate_fix(S);
}

OD_NOINL void dk_front(KState &S) {
    const KIn &in = S.in;
    Bump &mem = S.mem;
    KCtx &K = S.K;
    KOut &out = S.out;
    long long tp = OD_CLK();
#define OD_CHECK(x)                                                                                \
    do {                                                                                           \
        if (!(x) || mem.oom) {                                                                     \
            out.status = KS_OOM;                                                                   \
            S.done = 1;                                                                            \
            return;                                                                                \
        }                                                                                          \
    } while (0)
    OD_CHECK(collect_alloc(K)); // first in the arena (k_front's warp may have filled them)
    {
        const u32 cap = diag_cap(in);
        K.dg = mem.get<Diag>(cap);
        K.dg_cap = cap;
        K.ndg = 0;
        OD_CHECK(K.dg);
    }
    OD_CHECK(parse_config(K));
    if (in.collected)
        collect_finish(K, Collected{in.c_nins, in.c_nkl, in.c_pend_b, in.c_last_line, in.c_any_failed});
    else
        collect_finish(K, collect_fill(K));
    out.ninstr = K.nins_real;
    OD_CHECK(build_abi(K));
    OD_PROF(0, tp);
    OD_CHECK(build_cfg(K));
    if (K.failed) {
        out.status = KS_FAILED;
        S.done = 1;
        return;
    }
    OD_PROF(1, tp);
    normalize(K);
    OD_CHECK(!K.oom);
    OD_PROF(2, tp);
    if (in.dump && (in.dump->flags & DUMP_CFG))
        dump_emit(K, -1);
    if (in.dump && (in.dump->flags & DUMP_BODY))
        dump_emit(K, -4);
    OD_CHECK(build_regions(K));
    reduce(K);
    if (K.oom) {
        out.status = KS_OOM;
        S.done = 1;
        return;
    }
    if (in.dump && (in.dump->flags & DUMP_MERGES))
        dump_emit(K, -2);
    if (K.dump_full) { // grow the dump pool and run the kernel again
        out.status = KS_STAGE_FULL;
        S.done = 1;
        return;
    }
    OD_PROF(3, tp);
    out.structured = K.reduced ? 1 : 0;
    // live_in_sets is only read at if-joins (merge_at_join, lower.cpp:143-157):
    // kernels whose region tree has no if (straight-line, or goto form) skip it.
    if (K.reduced && K.nif)
        OD_CHECK(liveness(K));
    else
        K.live_in = nullptr;
    OD_PROF(4, tp);

    // Carve the remaining arena into the dynamic pools.
    out.u_fixed = (u32)mem.top;
    out.u_regions = K.nrg;
    K.regs = mem.get<Slot>(kPhysSlots);
    OD_CHECK(K.regs);
    if (in.names_zeroed_by_caller) { // k_front's warp writes the default slots
        for (u32 w = 0; w < kLiveWords; ++w)
            K.dirty[w] = 0;
    } else {
        full_register_init(K);
    }
    const PoolCaps pc = pool_caps(in.lend - in.lbeg, in.scale ? in.scale : 1);
    K.E.cap = pc.nodes;
    K.E.n = mem.get<ENode>(K.E.cap);
    K.st_cap = pc.stmts;
    K.st = mem.get<Stmt>(K.st_cap);
    K.lists_cap = 2 * K.nrg + 4;
    K.lists = mem.get<SList>(K.lists_cap);
    K.frames_cap = 2 * K.nrg + 8;
    K.frames = mem.get<Frame>(K.frames_cap);
    K.log_cap = pc.log;
    K.log = mem.get<UndoRec>(K.log_cap);
    K.dstk_cap = pc.dstk;
    K.dstk = mem.get<Slot>(K.dstk_cap);
    K.dstk_id = mem.get<u32>(K.dstk_cap);
    K.fresh_cap = pc.fresh;
    K.fresh = mem.get<Fresh>(K.fresh_cap);
    K.pool.cap = pc.names;
    K.pool.keys = mem.get<u64>(pc.names);
    K.pool.count = 0;
    K.pool.oom = false;
    const u32 scap = pc.stack;
    K.fs.st.p = mem.get<u32>(scap);
    K.fs.st.cap = scap;
    K.fs.terms.p = mem.get<u32>(scap);
    K.fs.terms.cap = scap;
    K.eqst.p = mem.get<u32>(scap);
    K.eqst.cap = scap;
    const u32 tcap = pc.tasks;
    K.rc.ts.p = mem.get<u64>(tcap);
    K.rc.ts.cap = tcap;
    S.ecap = 3 * (K.nrg + 8);
    S.estk = mem.get<u32>(S.ecap);
    Writer &w = S.w;
    w.cap = pc.out;
    w.p = mem.get<u8>(w.cap);
    w.n = 0;
    w.overflow = false;
    OD_CHECK(K.E.n && K.st && K.lists && K.frames && K.log && K.dstk && K.dstk_id && K.fresh &&
             K.pool.keys && K.fs.st.p && K.fs.terms.p && K.eqst.p && K.rc.ts.p && S.estk && w.p);
    if (!in.names_zeroed_by_caller) // (k_front: the whole warp zeroes it, coalesced)
        name_set_clear(K.pool);
    memset(&K.E.n[0], 0, sizeof(ENode));
    K.E.top = 1; // node 0 = null
    K.E.oom = false;
    K.nst = 1;   // stmt 0 = sink
    K.st[0].kind = SK_RAW;
    K.st[0].next = 0;
    K.nlists = 0;
    S.body = new_list(K);
    K.rc.text = in.t;
    K.rc.arg_sname = K.arg_sname;
    K.rc.fs = K.fs;
    OD_PROF(5, tp);
#undef OD_CHECK
}

OD_NOINL void dk_lower(KState &S) {
    const KIn &in = S.in;
    KCtx &K = S.K;
    KOut &out = S.out;
    long long tp = OD_CLK();
    if (K.reduced)
        lower_structured(K, K.root_r, S.body);
    else
        lower_goto(K, S.body);
    OD_PROF(6, tp);
    if (K.oom || K.E.oom || K.pool.oom || K.eqst.oom || K.fs.st.oom || K.fs.terms.oom) {
        out.status = KS_OOM;
        S.done = 1;
        return;
    }
    out.fallbacks = K.fallbacks;

    // hoist_fresh_decls: first occurrence per name, in record order.
    S.hoist = new_list(K);
    for (u32 i = 0; i < K.nfresh; ++i) {
        const Fresh &f = K.fresh[i];
        if (!K.pool.mark(f.cls, f.num))
            continue;
        u32 d = new_stmt(K, SK_DECL);
        K.st[d].cls = (u16)f.cls;
        K.st[d].a = f.num;
        K.st[d].c = f.type;
        list_append(K, S.hoist, d);
    }
    if (K.oom || K.pool.oom) {
        out.status = KS_OOM;
        S.done = 1;
    }
}

// The fold_expr calls of lower_block / taken_cond / emit_join (lower.cpp:37-39,
// 89-121, 139-141, 225-240) as one pass over the statement pool.  Folded
// trees only ever land in statements (never in register slots, whose
// identity read_pair_ids/dissolve_pair compare), and fold_expr is a pure
// function of its subtree, so folding after lowering gives the same text.
OD_NOINL void dk_fold(KState &S) {
    const KIn &in = S.in;
    KCtx &K = S.K;
    long long tp = OD_CLK();
    for (u32 i = 1; i < K.nst && !K.E.oom; ++i) {
        Stmt &st = K.st[i];
        switch (st.kind) {
        case SK_STORE:
            st.a = fold(K, st.a);
            st.b = fold(K, st.b);
            break;
        case SK_DECL:
        case SK_ASSIGN:
            if (st.b)
                st.b = fold(K, st.b);
            break;
        case SK_IF:
        case SK_GOTO:
            if (st.a)
                st.a = fold(K, st.a);
            break;
        default: break;
        }
    }
    OD_PROF(8, tp);
    if (K.E.oom || K.fs.st.oom || K.fs.terms.oom) {
        S.out.status = KS_OOM;
        S.done = 1;
    }
}

// emit_kernel  codegen.cpp:446-467
// The lowered statement tree as a step -3 dump (k_export, after k_emit, only
// when DUMP_BODY is requested).  Returns false when the dump pool is full.
OD_NOINL bool dk_export(KState &S) {
    KCtx &K = S.K;
    K.rc.fs = K.fs;
    K.exp_lists[0] = S.hoist;
    K.exp_lists[1] = S.body;
    K.exp_pass = 0;
    K.dump_full = false;
    dump_emit(K, -3);
    return !K.dump_full;
}

OD_NOINL void dk_emit(KState &S) {
    const KIn &in = S.in;
    KCtx &K = S.K;
    KOut &out = S.out;
    Writer &w = S.w;
    long long tp = OD_CLK();
    K.rc.fs = K.fs;
    const u8 *t = in.t;
    w.lit("__kernel void ");
    w.putn(t + K.cfg.name.off, K.cfg.name.len);
    w.put('(');
    bool first = true;
    for (u32 i = 0; i < K.cfg.nargs; ++i) {
        const KArg &a = K.cfg.args[i];
        if (a.implicit)
            continue;
        if (!first)
            w.lit(", ");
        first = false;
        render_type(w, a.type);
        if (!type_ends_star(a.type))
            w.put(' ');
        w.putn(t + a.name.off, a.name.len);
    }
    w.lit(") {\n");
    emit_list(K, w, K.lists[S.hoist].head, 1, S.estk, S.ecap);
    emit_list(K, w, K.lists[S.body].head, 1, S.estk, S.ecap);
    w.lit("}\n");
    S.done = 1;
    if (K.oom || K.E.oom || K.rc.ts.oom || w.overflow || K.rc.fs.terms.oom || K.rc.fs.st.oom) {
        out.status = KS_OOM;
        return;
    }
    OD_PROF(7, tp);
    out.out_len = w.n;
    out.u_nodes = K.E.top;
    out.u_stmts = K.nst;
    out.u_log = K.log_hw;
    out.u_dstk = K.dstk_hw;
    out.u_fresh = K.nfresh;
    out.u_names = K.pool.count;
    {
        u32 h = K.fs.st.hw;
        if (K.fs.terms.hw > h) h = K.fs.terms.hw;
        if (K.eqst.hw > h) h = K.eqst.hw;
        if (K.rc.fs.st.hw > h) h = K.rc.fs.st.hw;
        if (K.rc.fs.terms.hw > h) h = K.rc.fs.terms.hw;
        out.u_stack = h;
    }
    out.u_tasks = K.rc.ts.hw;
}

// Arena slice of a kernel of n lines at scale s on the device: the KState
// plus everything dk_front/dk_lower/dk_emit allocate.
OD_INL u64 kernel_budget(const KSize &z, u32 s) { return arena_budget(z, s) + ((sizeof(KState) + 255) & ~255ull); }

// All three phases back to back (host harness and single-launch use).
// Returns the status; on KS_OK the OpenCL source is at *src.
OD_INL KOut decompile_kernel(const KIn &in, Bump &mem, const u8 **src) {
    // The state moves between phases as it does between device launches,
    // so a stale self-reference shows up here too.
    KState A, B;
    kstate_init(A, in, mem);
    dk_front(A);
    B = A;
    memset(&A, 0xA5, sizeof(A));
    kstate_fix(B);
    if (!B.done)
        dk_lower(B);
    if (!B.done)
        dk_fold(B);
    A = B;
    memset(&B, 0x5A, sizeof(B));
    kstate_fix(A);
    if (!A.done)
        dk_emit(A);
    *src = A.w.p;
    return A.out;
}

} // namespace od
