// ocldec-b200: the batched semantic check -- the
// reference's differential backend (core/src/oracle.cpp) restated on the
// device: a single-lane interpreter of the kernel's instructions
// (interpret_asm, oracle.cpp:106-625) and an evaluator of the body the
// pipeline lowered (evaluate_decompiled, oracle.cpp:627-842), run side by
// side for sampled environments (od_semenv.cuh).  Equal write traces in
// every environment say the emitted OpenCL computes what the assembly does.
//
// One kernel per warp, one environment per lane (k_semcheck, od_phases.cu).
// Each lane's memory overlays, variables and evaluation stack live in a
// fixed slice of a scratch pool; a kernel that outgrows it is reported as
// SEM_CAPACITY rather than compared.
#pragma once

#include "od_semenv.cuh"

namespace od {

constexpr u64 kSemSettingsBase = 0xf000000000000000ull; // oracle.cpp:17-20
constexpr u32 kSemMemCap = 256;    // stores per side and environment (the trace log)
constexpr u32 kSemMemSlots = 512;  // the overlay's open-addressing table (power of two, load <= 1/2)
constexpr u32 kSemVarCap = 512;    // variable slots (open addressing, power of two)
constexpr u32 kSemStackCap = 512;  // evaluation stack entries
constexpr u64 kSemMemBytes = kSemMemCap * 12ull + kSemMemSlots * 12ull;
constexpr u64 kSemLaneBytes = 2 * kSemMemBytes + kSemVarCap * 16 + kSemStackCap * 16;
constexpr u32 kSemEnvs = 8;        // environments (lanes) per kernel
constexpr long kSemFuel = 1 << 20; // interpreter steps (oracle.cpp:121)
constexpr u32 kSemDeferCap = 1u << 16; // deferred kernels per chunk (k_semcheck's list)
constexpr u32 kSemDeferKB = 256u << 10; // their estimated listing bytes per chunk, in KB (256 MB)
constexpr u64 kSemDeferRunKB = 1u << 20; // ... and per run (1 GiB of host memory at most)
constexpr u32 kSemBatch = 2048;    // warps of a k_semcheck launch (scratch per wave stream: kSemBatch x kSemEnvs lanes)

// Memory  oracle.cpp:41-56: a pristine hash overlaid by this run's writes;
// the writes in order are the trace.  The overlay is an open-addressing
// table (one or two probes per access; key 0 = empty, address 0 kept aside),
// the ordered log only feeds the debug dumps (OD_SEM_DEBUG, tools/devhost).
struct SemMem {
    u64 *addr; // log, kSemMemCap
    u32 *val;
    u64 *tkey; // overlay, kSemMemSlots
    u32 *tval;
    u32 n;
    u64 seed;
    u64 hash;
    u32 count; // trace length (every store, also past the log's room)
    bool full;
    bool zset; // address 0 written
    u32 zval;
    // Carves this memory's arrays from base (advancing it) and clears it.
    OD_INL void init(u8 *&base, u64 mem_seed) {
        addr = reinterpret_cast<u64 *>(base);
        tkey = addr + kSemMemCap;
        val = reinterpret_cast<u32 *>(tkey + kSemMemSlots);
        tval = val + kSemMemCap;
        base += kSemMemBytes;
        for (u32 i = 0; i < kSemMemSlots; ++i)
            tkey[i] = 0;
        n = 0;
        seed = mem_seed;
        hash = kSemTraceSeed;
        count = 0;
        full = false;
        zset = false;
        zval = 0;
    }
    static OD_INL u32 slot(u64 a) { return (u32)((a * 0x9e3779b97f4a7c15ull) >> 55) & (kSemMemSlots - 1); }
    OD_INL u32 load(u64 a) const {
        if (!a)
            return zset ? zval : sem_initial_memory(seed, a);
        for (u32 i = slot(a);; i = (i + 1) & (kSemMemSlots - 1)) {
            const u64 k = tkey[i];
            if (k == a)
                return tval[i];
            if (!k)
                return sem_initial_memory(seed, a);
        }
    }
    OD_INL void store(u64 a, u32 v) {
        hash = sem_trace_step(hash, a, v);
        ++count;
        if (n >= kSemMemCap) {
            full = true;
            return;
        }
        addr[n] = a;
        val[n] = v;
        ++n;
        if (!a) {
            zset = true;
            zval = v;
            return;
        }
        for (u32 i = slot(a);; i = (i + 1) & (kSemMemSlots - 1)) {
            const u64 k = tkey[i];
            if (k == a || !k) { // at most kSemMemCap distinct addresses: always a free slot
                tkey[i] = a;
                tval[i] = v;
                return;
            }
        }
    }
};

// One k_semcheck launch (od_sem.cu).
struct SemArgs {
    u32 n;           // wave slots
    u32 *next;       // the wave's slot counter
    u8 *scratch;     // kSemBatch warps x kSemEnvs lanes x kSemLaneBytes
    SemResult *out;  // per chunk kernel
    u64 seed, kbase; // environment seed; listing ordinal of the chunk's kernel 0
    u64 *counts;     // kernels per SemStatus
    const u64 *kmap; // non-null: kernel k's listing ordinal is kmap[kbase + k] (deferred re-checks)
    long budget;     // steps per environment before a kernel is deferred: max(budget, 8 x its
                     // instructions); < 0: exactly -budget (tests); 0: never
    u32 *dlist;      // deferred kernels: [0] count, [1] estimated KB, then chunk kernel indices
    u32 dcap;
    u32 dkb;         // estimated listing KB the chunk may defer (the run's remaining allowance)
};

// What the kernel sees of one environment.
struct SemCtx {
    const KCtx *K;
    SemEnv env;
    u64 argv[32];  // per argument index: the value its sanitized name looks up (0 if none)
    bool unsupported;
    bool nan_choice; // an operation met two different NaN payloads (sem_nan)
};

OD_INL bool sem_name_matches(const u8 *t, Span raw, Span other) {
    // raw == other with '.' -> '_' applied to other (slot_value / KernelArg lookup)
    if (raw.len != other.len)
        return false;
    for (u32 i = 0; i < raw.len; ++i) {
        const u8 c = t[other.off + i];
        if (t[raw.off + i] != (c == '.' ? '_' : c))
            return false;
    }
    return true;
}

// Argument values: env.arg_values holds the non-implicit arguments by raw
// name (envgen.cpp:70-81); lookups go by the sanitized name of an argument
// (oracle.cpp:80-85, 655-658), last declaration winning.
OD_INL void sem_args(SemCtx &c, SemRng &r) {
    const KCtx &K = *c.K;
    const u32 na = K.cfg.nargs < 32 ? K.cfg.nargs : 32;
    u64 raw[32];
    for (u32 i = 0; i < na; ++i) {
        const KArg &a = K.cfg.args[i];
        raw[i] = a.implicit ? 0 : sem_arg(r, &c.env, dt_is_pointer(a.type), dt_is_float(a.type), dt_bits(a.type));
    }
    for (u32 j = 0; j < na; ++j) {
        c.argv[j] = 0;
        for (u32 i = 0; i < na; ++i)
            if (!K.cfg.args[i].implicit && sem_name_matches(K.in->t, K.cfg.args[i].name, K.cfg.args[j].name))
                c.argv[j] = raw[i];
    }
}

// slot_value  oracle.cpp:59-90
OD_INL u64 sem_slot_value(const SemCtx &c, const AbiEntry *e) {
    const SemEnv &v = c.env;
    if (e->has_builtin) {
        const u32 d = e->dim < 3 ? e->dim : 0;
        switch (e->fn) {
        case F_GLOBAL_OFFSET: return v.global_offset[d];
        case F_GLOBAL_SIZE: return (u64)(u32)(v.cws[d] * v.num_groups[d]);
        case F_WORK_DIM: return v.dims;
        case F_LOCAL_SIZE: return v.cws[d];
        case F_NUM_GROUPS: return v.num_groups[d];
        default: return 0;
        }
    }
    if (e->arg_index >= 0 && (u32)e->arg_index < c.K->cfg.nargs && e->arg_index < 32)
        return c.argv[e->arg_index];
    return 0;
}

// ------------------------------------------------------------ interpreter
// IEEE single arithmetic, round to nearest, never contracted into an FMA
// (the reference's host build does the multiply and the add separately).
// NaNs follow the host's SSE rules, not the GPU's canonical 0x7fffffff: a NaN
// operand propagates quieted, and an invalid operation yields the default NaN
// 0xffc00000.  When BOTH operands are NaNs with different payloads, IEEE 754
// leaves the choice open and the reference's result depends on how its
// compiler ordered the operands: the environment is then marked
// indeterminate (SEM_INDETERMINATE) instead of guessing.
OD_INL float sem_nan(SemCtx &c, float a, float b, float r) {
    u32 ua, ub;
    memcpy(&ua, &a, 4);
    memcpy(&ub, &b, 4);
    const bool na = (ua & 0x7fffffffu) > 0x7f800000u, nb = (ub & 0x7fffffffu) > 0x7f800000u;
    if (na && nb && (ua | 0x400000u) != (ub | 0x400000u))
        c.nan_choice = true;
#ifdef __CUDA_ARCH__
    if (!isnan(r))
        return r;
    if (na)
        return __uint_as_float(ua | 0x400000u);
    if (nb)
        return __uint_as_float(ub | 0x400000u);
    return __uint_as_float(0xffc00000u);
#else
    return r;
#endif
}
OD_INL float sem_fmul(SemCtx &c, float a, float b) {
#ifdef __CUDA_ARCH__
    return sem_nan(c, a, b, __fmul_rn(a, b));
#else
    return sem_nan(c, a, b, a * b);
#endif
}
OD_INL float sem_fadd(SemCtx &c, float a, float b) {
#ifdef __CUDA_ARCH__
    return sem_nan(c, a, b, __fadd_rn(a, b));
#else
    return sem_nan(c, a, b, a + b);
#endif
}
OD_INL float sem_fsub(SemCtx &c, float a, float b) {
#ifdef __CUDA_ARCH__
    return sem_nan(c, a, b, __fsub_rn(a, b));
#else
    return sem_nan(c, a, b, a - b);
#endif
}
OD_INL float sem_fdiv(SemCtx &c, float a, float b) {
#ifdef __CUDA_ARCH__
    return sem_nan(c, a, b, __fdiv_rn(a, b));
#else
    return sem_nan(c, a, b, a / b);
#endif
}

struct SemMachine {
    SemCtx &c;
    SemMem &mem;
    u32 s[kSgprCount];
    u32 v[kVgprCount];
    u64 exec, vcc;
    u32 scc, m0;
    bool bad; // OracleUnsupported
    long steps; // instructions executed (fuel used)
    u32 wm;     // device: the lanes (environments) of this kernel's warp, stepped in pc order
    u32 tc_key[16], tc_val[16]; // branch targets already resolved (pc + 1 -> instruction)

    const Opnd *opsp; // c.K->in->ops, held by run() (one load instead of a pointer chain per operand)
    const Ins *insp;  // c.K->ins
    OD_INL const Opnd &op(const Ins &I, u32 k) const { return opsp[I.op_start + k]; }
    OD_INL u32 nops(const Ins &I) const { return (I.flags & IF_SYNTH) ? 0 : I.nops; }
    OD_INL bool lane_on() const { return (exec & 1) != 0; }
    OD_INL u32 sget(u32 i) {
        if (i >= kSgprCount) {
            bad = true; // std::array::at
            return 0;
        }
        return s[i];
    }
    OD_INL void sset(u32 i, u32 x) {
        if (i >= kSgprCount)
            bad = true;
        else
            s[i] = x;
    }
    OD_INL u32 vget(u32 i) {
        if (i >= kVgprCount) {
            bad = true;
            return 0;
        }
        return v[i];
    }
    OD_INL void vset(u32 i, u32 x) {
        if (i >= kVgprCount)
            bad = true;
        else
            v[i] = x;
    }
    OD_HD u64 read64(const Opnd &o) {
        switch (o.kind) {
        case OK_SREG: return (u64)sget(o.r.a) | ((u64)sget(o.r.a + 1) << 32);
        case OK_VREG: return (u64)vget(o.r.a) | ((u64)vget(o.r.a + 1) << 32);
        case OK_LITERAL: return (u64)o.value;
        case OK_SPECIAL:
            if (o.special == SP_EXEC)
                return exec;
            if (o.special == SP_VCC)
                return vcc;
            break;
        default: break;
        }
        bad = true;
        return 0;
    }
    OD_HD u32 read32(const Opnd &o) {
        switch (o.kind) {
        case OK_SREG: return sget(o.r.a);
        case OK_VREG: return vget(o.r.a);
        case OK_LITERAL: return (u32)o.value;
        case OK_SPECIAL:
            switch (o.special) {
            case SP_EXEC_LO: return (u32)exec;
            case SP_EXEC_HI: return (u32)(exec >> 32);
            case SP_VCC_LO: return (u32)vcc;
            case SP_VCC_HI: return (u32)(vcc >> 32);
            case SP_SCC: return scc;
            case SP_M0: return m0;
            default: break;
            }
            break;
        default: break;
        }
        bad = true;
        return 0;
    }
    OD_HD void write_sdst32(const Opnd &o, u32 x) {
        if (o.kind == OK_SREG)
            sset(o.r.a, x);
        else if (o.kind == OK_SPECIAL && o.special == SP_M0)
            m0 = x;
        else
            bad = true;
    }
    OD_HD void write_sdst64(const Opnd &o, u64 x) {
        if (o.kind == OK_SREG) {
            sset(o.r.a, (u32)x);
            sset(o.r.a + 1, (u32)(x >> 32));
        } else if (o.kind == OK_SPECIAL && o.special == SP_EXEC) {
            exec = x;
        } else if (o.kind == OK_SPECIAL && o.special == SP_VCC) {
            vcc = x;
        } else {
            bad = true;
        }
    }
    OD_HD void write_vdst(const Opnd &o, u32 x) {
        if (o.kind != OK_VREG) {
            bad = true;
            return;
        }
        if (lane_on())
            vset(o.r.a, x);
    }
    OD_HD void write_carry(const Opnd &o, u64 bit) {
        const u64 masked = lane_on() ? bit : 0;
        if (op_is_special(o, SP_VCC))
            vcc = masked;
        else
            write_sdst64(o, masked);
    }
    OD_HD u32 settings_dword(u32 offset) {
        bool second = false;
        const AbiEntry *e = abi_find_dword(*c.K, offset, &second);
        if (!e)
            return sem_initial_memory(c.env.mem_seed, kSemSettingsBase + offset);
        const u64 x = sem_slot_value(c, e);
        return second ? (u32)(x >> 32) : (u32)x;
    }
    OD_HD u32 load_dword(u64 a) {
        if (a >= kSemSettingsBase && a < kSemSettingsBase + (1ull << 20))
            return settings_dword((u32)(a - kSemSettingsBase));
        return mem.load(a);
    }
    // compare  oracle.cpp:413-441: the op from the root, the type from the
    // first suffix (scalar default b32, vector default i32)
    OD_HD bool compare(const Ins &I, DT t, u32 a, u32 b) {
        const u32 r = I.root;
        if (dt_is_float(t)) {
            const float x = __uint_as_float_h(a), y = __uint_as_float_h(b);
            switch (r) {
            case R_CMP_EQ: return x == y;
            case R_CMP_NE:
            case R_CMP_LG:
            case R_CMP_NEQ: return x != y;
            case R_CMP_LT: return x < y;
            case R_CMP_LE: return x <= y;
            case R_CMP_GT: return x > y;
            case R_CMP_GE: return x >= y;
            default: break;
            }
        } else if (dt_base(t) == B_UNSIGNED || dt_base(t) == B_BINARY) {
            switch (r) {
            case R_CMP_EQ: return a == b;
            case R_CMP_NE:
            case R_CMP_LG: return a != b;
            case R_CMP_LT: return a < b;
            case R_CMP_LE: return a <= b;
            case R_CMP_GT: return a > b;
            case R_CMP_GE: return a >= b;
            default: break;
            }
        } else {
            const i32 x = (i32)a, y = (i32)b;
            switch (r) {
            case R_CMP_EQ: return x == y;
            case R_CMP_NE:
            case R_CMP_LG: return x != y;
            case R_CMP_LT: return x < y;
            case R_CMP_LE: return x <= y;
            case R_CMP_GT: return x > y;
            case R_CMP_GE: return x >= y;
            default: break;
            }
        }
        bad = true; // unknown comparison (e.g. "neq" on integers)
        return false;
    }
    static OD_INL float __uint_as_float_h(u32 b) {
        float f;
        memcpy(&f, &b, 4);
        return f;
    }
    static OD_INL u32 __float_as_uint_h(float f) {
        u32 b;
        memcpy(&b, &f, 4);
        return b;
    }
    OD_HD bool mul24(const Ins &I) {
        for (u32 k = 0; k < 2; ++k)
            if (I.sfx[k] && sfx_bits(I.sfx[k]) == 24) {
                if (sfx_base(I.sfx[k]) == SB_I)
                    bad = true; // signed 24-bit multiply
                return true;
            }
        return false;
    }
    // target  oracle.cpp:233-240: the instruction the label sits on
    OD_HD u32 target(const Ins &I) {
        const u32 pc = (u32)(&I - insp), h = pc & 15;
        if (tc_key[h] == pc + 1) // loops branch to the same labels over and over
            return tc_val[h];
        if (nops(I) == 0 || op(I, 0).kind != OK_SYMBOL) {
            bad = true;
            return 0;
        }
        const Opnd &o = op(I, 0);
        const int b = lmap_get(*c.K, Span{o.r.a, o.r.b});
        if (b < 0) {
            bad = true;
            return 0;
        }
        tc_key[h] = pc + 1;
        tc_val[h] = c.K->blk[b].ib;
        return tc_val[h];
    }

    // scalar  oracle.cpp:268-411; returns false on s_endpgm
    OD_HD bool scalar(const Ins &I, u32 &next) {
        const u32 r = I.root, n = nops(I);
        if (r == R_ENDPGM)
            return false;
        if (r == R_WAITCNT || r == R_NOP || r == R_BARRIER)
            return true;
        if (r == R_BRANCH) {
            next = target(I);
            return true;
        }
        if (I.rflags & RF_CBRANCH) {
            bool taken = false;
            switch (r) {
            case R_CBRANCH_SCC0: taken = scc == 0; break;
            case R_CBRANCH_SCC1: taken = scc != 0; break;
            case R_CBRANCH_VCCZ: taken = vcc == 0; break;
            case R_CBRANCH_VCCNZ: taken = vcc != 0; break;
            case R_CBRANCH_EXECZ: taken = exec == 0; break;
            case R_CBRANCH_EXECNZ: taken = exec != 0; break;
            default: bad = true; return true;
            }
            if (taken)
                next = target(I);
            return true;
        }
        if (r == R_LOAD_DWORD || r == R_LOAD_DWORDX2 || r == R_LOAD_DWORDX4) {
            const u32 dw = r == R_LOAD_DWORD ? 1 : r == R_LOAD_DWORDX2 ? 2 : 4;
            if (n < 2 || op(I, 0).kind != OK_SREG) {
                bad = true;
                return true;
            }
            const u64 base = read64(op(I, 1));
            const u64 off = n >= 3 && op(I, 2).kind == OK_LITERAL ? (u64)op(I, 2).value : 0;
            const u64 a = base + off;
            if (a >= kSemSettingsBase && a < kSemSettingsBase + (1ull << 20) && dw <= 2) {
                if (const AbiEntry *e = abi_find(*c.K, (u32)(a - kSemSettingsBase), dw)) {
                    const u64 x = sem_slot_value(c, e);
                    sset(op(I, 0).r.a, (u32)x);
                    if (dw == 2)
                        sset(op(I, 0).r.a + 1, (u32)(x >> 32));
                    return true;
                }
            }
            for (u32 k = 0; k < dw; ++k)
                sset(op(I, 0).r.a + k, load_dword(a + 4 * k));
            return true;
        }
        const DT t = suffix_type0(I, DT_B32);
        const bool wide = dt_bits(t) == 64;
        if (r == R_MOV && n >= 2) {
            if (wide)
                write_sdst64(op(I, 0), read64(op(I, 1)));
            else
                write_sdst32(op(I, 0), read32(op(I, 1)));
            return true;
        }
        if ((r == R_ADD || r == R_SUB) && n >= 3) {
            const u64 a = read32(op(I, 1)), b = read32(op(I, 2));
            const u64 x = r == R_ADD ? a + b : a - b;
            write_sdst32(op(I, 0), (u32)x);
            if (dt_is_signed(t)) {
                const i64 sr = r == R_ADD ? (i64)(i32)a + (i32)b : (i64)(i32)a - (i32)b;
                scc = sr != (i64)(i32)(u32)sr ? 1 : 0;
            } else {
                scc = (u32)((x >> 32) & 1);
            }
            return true;
        }
        if ((r == R_ADDK || r == R_MULK) && n >= 2) {
            const u32 a = read32(op(I, 0)), b = read32(op(I, 1));
            write_sdst32(op(I, 0), r == R_ADDK ? a + b : a * b);
            if (r == R_ADDK)
                scc = (((u64)a + b) >> 32) ? 1 : 0;
            return true;
        }
        if (r == R_MUL && n >= 3) {
            write_sdst32(op(I, 0), read32(op(I, 1)) * read32(op(I, 2)));
            return true;
        }
        if ((r == R_AND || r == R_OR || r == R_XOR || r == R_ANDN2) && n >= 3) {
            const u64 a = wide ? read64(op(I, 1)) : read32(op(I, 1));
            const u64 b = wide ? read64(op(I, 2)) : read32(op(I, 2));
            const u64 x = r == R_AND ? (a & b) : r == R_OR ? (a | b) : r == R_XOR ? (a ^ b) : (a & ~b);
            if (wide)
                write_sdst64(op(I, 0), x);
            else
                write_sdst32(op(I, 0), (u32)x);
            scc = x != 0;
            return true;
        }
        if ((r == R_LSHL || r == R_LSHR || r == R_ASHR) && n >= 3) {
            const u64 a = wide ? read64(op(I, 1)) : read32(op(I, 1));
            const u32 sh = read32(op(I, 2)) & (wide ? 63 : 31);
            u64 x;
            if (r == R_LSHL)
                x = a << sh;
            else if (r == R_LSHR)
                x = a >> sh;
            else
                x = wide ? (u64)((i64)a >> sh) : (u64)(u32)((i32)(u32)a >> sh);
            if (wide)
                write_sdst64(op(I, 0), x);
            else
                write_sdst32(op(I, 0), (u32)x);
            scc = x != 0;
            return true;
        }
        if (r == R_AND_SAVEEXEC && n >= 2) {
            const u64 old = exec;
            write_sdst64(op(I, 0), old);
            exec = old & read64(op(I, 1));
            scc = exec != 0;
            return true;
        }
        if ((I.rflags & RF_CMP) && n >= 2) {
            scc = compare(I, t, read32(op(I, 0)), read32(op(I, 1))) ? 1 : 0;
            return true;
        }
        bad = true;
        return true;
    }

    // vector  oracle.cpp:443-577
    OD_HD void vector(const Ins &I) {
        const u32 r = I.root, n = nops(I);
        const DT t = suffix_type0(I, DT_U32);
        if (r == R_MOV && n >= 2) {
            write_vdst(op(I, 0), read32(op(I, 1)));
            return;
        }
        if (r == R_CNDMASK && n >= 4) {
            const u64 cc = read64(op(I, 3));
            write_vdst(op(I, 0), (cc & 1) ? read32(op(I, 2)) : read32(op(I, 1)));
            return;
        }
        if ((r == R_ADD || r == R_SUB || r == R_SUBREV) && n >= 3) {
            u32 src0 = 1;
            const Opnd *carry = nullptr;
            if (op_is_special(op(I, 1), SP_VCC) || (op(I, 1).kind == OK_SREG && op(I, 1).count == 2)) {
                src0 = 2;
                carry = &op(I, 1);
            }
            if (n < src0 + 2) {
                bad = true;
                return;
            }
            u64 a = read32(op(I, src0)), b = read32(op(I, src0 + 1));
            if (r == R_SUBREV) {
                const u64 tmp = a;
                a = b;
                b = tmp;
            }
            if (dt_is_float(t)) {
                if (dt_bits(t) != 32 || carry) {
                    bad = true;
                    return;
                }
                const float x = __uint_as_float_h((u32)a), y = __uint_as_float_h((u32)b);
                write_vdst(op(I, 0), __float_as_uint_h(r == R_ADD ? sem_fadd(c, x, y) : sem_fsub(c, x, y)));
                return;
            }
            const u64 x = r == R_ADD ? a + b : a - b;
            write_vdst(op(I, 0), (u32)x);
            if (carry)
                write_carry(*carry, r == R_ADD ? (x >> 32) & 1 : (a < b ? 1 : 0));
            return;
        }
        if (r == R_ADDC && n >= 5) {
            const u64 cin = read64(op(I, 4)) & 1;
            const u64 x = (u64)read32(op(I, 2)) + read32(op(I, 3)) + cin;
            write_vdst(op(I, 0), (u32)x);
            write_carry(op(I, 1), (x >> 32) & 1);
            return;
        }
        if ((r == R_MUL || r == R_MUL_LO || r == R_MUL_HI) && n >= 3) {
            u64 a = read32(op(I, 1)), b = read32(op(I, 2));
            if (mul24(I)) {
                a &= 0xffffff;
                b &= 0xffffff;
            }
            if (r == R_MUL_HI) {
                const u64 prod = dt_is_signed(t) ? (u64)((i64)(i32)a * (i64)(i32)b) : a * b;
                write_vdst(op(I, 0), (u32)(prod >> 32));
            } else if (dt_is_float(t)) {
                write_vdst(op(I, 0), __float_as_uint_h(sem_fmul(c, __uint_as_float_h((u32)a), __uint_as_float_h((u32)b))));
            } else {
                write_vdst(op(I, 0), (u32)(a * b));
            }
            return;
        }
        if (r == R_MAC && n >= 3) {
            if (!dt_is_float(t)) {
                bad = true;
                return;
            }
            float x = sem_fmul(c, __uint_as_float_h(read32(op(I, 1))), __uint_as_float_h(read32(op(I, 2))));
            x = sem_fadd(c, x, __uint_as_float_h(read32(op(I, 0))));
            write_vdst(op(I, 0), __float_as_uint_h(x));
            return;
        }
        if (r == R_MAD && n >= 4) {
            if (dt_is_float(t)) {
                float x = sem_fmul(c, __uint_as_float_h(read32(op(I, 1))), __uint_as_float_h(read32(op(I, 2))));
                x = sem_fadd(c, x, __uint_as_float_h(read32(op(I, 3))));
                write_vdst(op(I, 0), __float_as_uint_h(x));
            } else {
                u32 a = read32(op(I, 1)), b = read32(op(I, 2));
                const u32 cc = read32(op(I, 3));
                if (mul24(I)) {
                    a &= 0xffffff;
                    b &= 0xffffff;
                }
                write_vdst(op(I, 0), a * b + cc);
            }
            return;
        }
        if ((r == R_LSHLREV || r == R_LSHRREV || r == R_ASHRREV || r == R_LSHL || r == R_LSHR || r == R_ASHR) &&
            n >= 3) {
            const bool rev = r == R_LSHLREV || r == R_LSHRREV || r == R_ASHRREV;
            const u32 sh = read32(op(I, rev ? 1 : 2)) & 31;
            const u32 a = read32(op(I, rev ? 2 : 1));
            u32 x;
            if (r == R_LSHLREV || r == R_LSHL)
                x = a << sh;
            else if (r == R_LSHRREV || r == R_LSHR)
                x = a >> sh;
            else
                x = (u32)((i32)a >> sh);
            write_vdst(op(I, 0), x);
            return;
        }
        if ((r == R_AND || r == R_OR || r == R_XOR) && n >= 3) {
            const u32 a = read32(op(I, 1)), b = read32(op(I, 2));
            write_vdst(op(I, 0), r == R_AND ? (a & b) : r == R_OR ? (a | b) : (a ^ b));
            return;
        }
        if ((I.rflags & RF_CMP) && n >= 3) {
            const bool x = compare(I, suffix_type0(I, DT_I32), read32(op(I, 1)), read32(op(I, 2)));
            const u64 bit = (lane_on() && x) ? 1 : 0;
            if (op_is_special(op(I, 0), SP_VCC))
                vcc = bit;
            else if (op(I, 0).kind == OK_SREG && op(I, 0).count == 2)
                write_sdst64(op(I, 0), bit);
            else
                bad = true;
            return;
        }
        bad = true;
    }

    // flat  oracle.cpp:585-611
    OD_HD void flat(const Ins &I) {
        const u32 r = I.root, n = nops(I);
        if (n < 2) {
            bad = true;
            return;
        }
        if (r == R_LOAD_DWORD || r == R_LOAD_DWORDX2) {
            const u64 a = read64(op(I, 1));
            const u32 dw = r == R_LOAD_DWORDX2 ? 2 : 1;
            for (u32 k = 0; k < dw; ++k)
                if (lane_on())
                    vset(op(I, 0).r.a + k, load_dword(a + 4 * k));
            return;
        }
        if (r == R_STORE_DWORD || r == R_STORE_DWORDX2) {
            const u64 a = read64(op(I, 0));
            const u32 dw = r == R_STORE_DWORDX2 ? 2 : 1;
            for (u32 k = 0; k < dw; ++k)
                if (lane_on())
                    mem.store(a + 4 * k, vget(op(I, 1).r.a + k));
            return;
        }
        bad = true;
    }

    // Machine::run  oracle.cpp:221-231
    // Machine::run  oracle.cpp:221-231, split so that a run can pause: run(limit)
    // steps until every lane has stopped or has executed `limit` steps (held),
    // and a later run(larger limit) continues from the same state.
    u32 pc;
    bool stop;
    bool held; // this lane reached the step limit of the last run() unfinished
    OD_HD void init() {
        const KCtx &K = *c.K;
        for (u32 i = 0; i < kSgprCount; ++i)
            s[i] = 0;
        for (u32 i = 0; i < kVgprCount; ++i)
            v[i] = 0;
        exec = ~0ull;
        vcc = 0;
        scc = 0;
        m0 = 0;
        bad = false;
        s[4] = (u32)kSemSettingsBase;
        s[5] = (u32)(kSemSettingsBase >> 32);
        for (u32 d = 0; d < K.cfg.dims && d < 3; ++d) {
            v[d] = c.env.local_id[d];
            s[6 + d] = c.env.group_id[d];
        }
        for (u32 i = 0; i < 16; ++i)
            tc_key[i] = 0;
        opsp = K.in->ops;
        insp = K.ins;
        pc = 0;
        steps = 0;
        stop = false;
        held = false;
    }
    // (one out-of-line copy: k_semcheck calls it twice, with and without a limit)
    OD_NOINL void run(long limit = kSemFuel + 1) {
        const KCtx &K = *c.K;
        held = false;
        for (;;) {
            stop = stop || pc >= K.nins || bad;
            const bool hold = !stop && steps >= limit;
#ifdef __CUDA_ARCH__
            // The warp's lanes run the same instructions on different data;
            // stepping only the lanes at the lowest pc keeps them at one
            // instruction (one dispatch path) instead of serializing lanes
            // that drifted apart.  Each lane still executes exactly its own
            // instruction sequence.
            const u32 key = stop || hold ? ~0u : pc;
            const u32 lo = __reduce_min_sync(wm, key);
            if (lo == ~0u) {
                held = hold;
                break;
            }
            if (key != lo)
                continue;
#else
            if (stop || hold) {
                held = hold;
                break;
            }
#endif
            if (++steps > kSemFuel) {
                bad = true;
                continue;
            }
            const Ins &I = insp[pc];
            if (I.flags & IF_PARSE_FAILED) {
                bad = true;
                continue;
            }
            u32 next = pc + 1;
            if (I.prefix == PX_S) {
                if (!scalar(I, next)) {
                    stop = true;
                    continue;
                }
            } else if (I.prefix == PX_V) {
                vector(I);
            } else if (I.prefix == PX_FLAT) {
                flat(I);
            } else {
                bad = true;
                continue;
            }
            pc = next;
        }
    }
};

// --------------------------------------------------------------- evaluator
// Variables by (register class, number): open addressing, key 0 = empty.
struct SemVars {
    u64 *key;
    u64 *val;
    bool full;
    OD_INL u32 slot(u64 k) const {
        u64 h = k * 0x9e3779b97f4a7c15ull;
        return (u32)(h >> 40) & (kSemVarCap - 1);
    }
    OD_INL u64 get(u64 k) const {
        for (u32 i = slot(k), q = 0; q < kSemVarCap; ++q, i = (i + 1) & (kSemVarCap - 1)) {
            if (key[i] == k)
                return val[i];
            if (!key[i])
                return 0;
        }
        return 0;
    }
    OD_INL void set(u64 k, u64 x) {
        for (u32 i = slot(k), q = 0; q < kSemVarCap; ++q, i = (i + 1) & (kSemVarCap - 1)) {
            if (key[i] == k || !key[i]) {
                key[i] = k;
                val[i] = x;
                return;
            }
        }
        full = true;
    }
};

OD_INL u64 sem_var_key(u32 cls, u32 num) { return ((u64)(cls + 1) << 32) | num; }
OD_INL u64 sem_mask(u64 x, u32 bits) { return bits >= 64 ? x : x & ((1ull << bits) - 1); }

struct SemEval {
    SemCtx &c;
    SemMem &mem;
    SemVars vars;
    u64 *stk; // (node, state) | value pairs
    bool bad, full;

    OD_HD u64 builtin_value(u32 fn, u32 d) const {
        const SemEnv &v = c.env;
        d = d < 3 ? d : 0;
        switch (fn) {
        case F_GLOBAL_ID: return (u64)v.group_id[d] * v.cws[d] + v.local_id[d] + v.global_offset[d];
        case F_LOCAL_ID: return v.local_id[d];
        case F_GROUP_ID: return v.group_id[d];
        case F_GLOBAL_SIZE: return (u64)(u32)(v.cws[d] * v.num_groups[d]);
        case F_LOCAL_SIZE: return v.cws[d];
        case F_NUM_GROUPS: return v.num_groups[d];
        case F_GLOBAL_OFFSET: return v.global_offset[d];
        case F_WORK_DIM: return v.dims;
        default: return 0;
        }
    }
    OD_HD u64 arg_value(u32 name_id) const {
        const KConfig &cfg = c.K->cfg;
        for (u32 j = 0; j < cfg.nargs && j < 32; ++j)
            if (cfg.args[j].name_id == name_id)
                return c.argv[j];
        return 0;
    }
    // Evaluator::extend  oracle.cpp:665-673
    static OD_HD u64 extend(u64 x, DT from) {
        if (dt_bits(from) >= 64)
            return x;
        x = sem_mask(x, dt_bits(from));
        if (dt_is_signed(from) && dt_bits(from) == 32 && (x >> 31))
            return x | 0xffffffff00000000ull;
        return x;
    }
    OD_HD u64 leaf(const ENode &x) const {
        switch (x.kind) {
        case E_CONST: return (u64)x.a | ((u64)x.b << 32);
        case E_BUILTIN: return sem_mask(builtin_value(x.op, x.x), dt_bits(x.type));
        case E_ARG: return sem_mask(arg_value(x.a), dt_is_pointer(x.type) ? 64 : dt_bits(x.type));
        case E_KBASE: return kSemSettingsBase;
        case E_VAR: return vars.get(sem_var_key(x.x, x.a));
        default: return 0;
        }
    }
    OD_HD u64 load_width(u64 a, u32 bytes) {
        if (bytes == 8)
            return (u64)mem.load(a) | ((u64)mem.load(a + 4) << 32);
        return mem.load(a);
    }
    OD_HD u64 unary(const EArena &E, const ENode &x, u64 a) {
        switch (x.op) {
        case U_LNOT: return a == 0;
        case U_BITNOT: return sem_mask(~a, dt_bits(x.type));
        case U_NEG: return sem_mask(~a + 1, dt_bits(x.type));
        case U_LO32: return a & 0xffffffffull;
        case U_HI32: return a >> 32;
        case U_CAST: {
            const DT from = E.n[x.a].type;
            if (dt_bits(x.type) > dt_bits(from))
                return extend(a, from);
            return sem_mask(a, dt_bits(x.type));
        }
        default: bad = true; return 0;
        }
    }
    OD_HD u64 binary(const EArena &E, const ENode &x, u64 a, u64 b) {
        const u32 op = x.op;
        if (op == O_CONCAT64)
            return (a & 0xffffffffull) | (b << 32);
        const u32 bits = dt_bits(x.type) >= 64 ? 64 : 32;
        const DT ta = E.n[x.a].type, tb = E.n[x.b].type;
        if (dt_is_float(x.type) || (is_cmp(op) && dt_is_float(ta))) {
            const float p = SemMachine::__uint_as_float_h((u32)a), q = SemMachine::__uint_as_float_h((u32)b);
            switch (op) {
            case O_ADD: return SemMachine::__float_as_uint_h(sem_fadd(c, p, q));
            case O_SUB: return SemMachine::__float_as_uint_h(sem_fsub(c, p, q));
            case O_MUL: return SemMachine::__float_as_uint_h(sem_fmul(c, p, q));
            case O_DIV: return SemMachine::__float_as_uint_h(sem_fdiv(c, p, q));
            case O_CMPEQ: return p == q;
            case O_CMPNE: return p != q;
            case O_CMPLT: return p < q;
            case O_CMPLE: return p <= q;
            case O_CMPGT: return p > q;
            case O_CMPGE: return p >= q;
            default: bad = true; return 0;
            }
        }
        const u32 ob = dt_bits(ta) > dt_bits(tb) ? dt_bits(ta) : dt_bits(tb);
        auto s_of = [&](u64 u) { return ob >= 64 ? (i64)u : (i64)(i32)(u32)u; };
        auto u_of = [&](u64 u) { return ob >= 64 ? u : (u & 0xffffffffull); };
        switch (op) {
        case O_ADD: return sem_mask(a + b, bits);
        case O_SUB: return sem_mask(a - b, bits);
        case O_MUL: return sem_mask(a * b, bits);
        case O_DIV:
            if (u_of(b) == 0) {
                bad = true;
                return 0;
            }
            return sem_mask(u_of(a) / u_of(b), bits);
        case O_MULHI: return (u32)(((a & 0xffffffffull) * (b & 0xffffffffull)) >> 32);
        case O_MULHIS: return (u32)((u64)((i64)(i32)(u32)a * (i64)(i32)(u32)b) >> 32);
        case O_AND: return a & b;
        case O_OR: return a | b;
        case O_XOR: return sem_mask(a ^ b, bits);
        case O_SHL: return sem_mask(a << (b & (bits - 1)), bits);
        case O_LSHR: return sem_mask(a, bits) >> (b & (bits - 1));
        case O_ASHR:
            if (bits == 64)
                return (u64)((i64)a >> (b & 63));
            return (u32)((i32)(u32)a >> (b & 31));
        case O_CMPEQ: return u_of(a) == u_of(b);
        case O_CMPNE: return u_of(a) != u_of(b);
        case O_CMPLT: return s_of(a) < s_of(b);
        case O_CMPLE: return s_of(a) <= s_of(b);
        case O_CMPGT: return s_of(a) > s_of(b);
        case O_CMPGE: return s_of(a) >= s_of(b);
        case O_CMPLTU: return u_of(a) < u_of(b);
        case O_CMPLEU: return u_of(a) <= u_of(b);
        case O_CMPGTU: return u_of(a) > u_of(b);
        case O_CMPGEU: return u_of(a) >= u_of(b);
        default: bad = true; return 0;
        }
    }
    // eval  oracle.cpp:675-707, iterative: frames (node << 2 | state) with a
    // value stack above them; a ternary evaluates only its taken side, a
    // deref loads at its evaluation point, as the recursive reference does.
    OD_HD u64 eval(u32 root) {
        const EArena &E = c.K->E;
        if (!root) {
            bad = true; // "missing expression"
            return 0;
        }
        // frames grow up from 0, values down from the top of the stack slice
        u32 fp = 0, vp = kSemStackCap;
        auto push_frame = [&](u32 e, u32 st) {
            if (fp + 1 >= vp) {
                full = true;
                return;
            }
            stk[fp++] = ((u64)e << 8) | st;
        };
        auto push_val = [&](u64 x) {
            if (vp - 1 <= fp) {
                full = true;
                return;
            }
            stk[--vp] = x;
        };
        push_frame(root, 0);
        while (fp && !bad && !full) {
            const u64 fr = stk[fp - 1];
            const u32 e = (u32)(fr >> 8), st = (u32)(fr & 0xff);
            if (!e) {
                bad = true;
                return 0;
            }
            const ENode x = E.n[e];
            switch (x.kind) {
            case E_UNARY:
            case E_DEREF:
                if (st == 0) {
                    stk[fp - 1] = fr | 1;
                    if (!x.a) {
                        bad = true;
                        break;
                    }
                    push_frame(x.a, 0);
                } else {
                    const u64 a = stk[vp++];
                    --fp;
                    push_val(x.kind == E_DEREF ? load_width(a, dt_byte_size(x.type)) : unary(E, x, a));
                }
                break;
            case E_BINARY:
                if (st < 2) {
                    const u32 ch = st == 0 ? x.a : x.b;
                    stk[fp - 1] = (fr & ~0xffull) | (st + 1);
                    if (!ch) {
                        bad = true;
                        break;
                    }
                    push_frame(ch, 0);
                } else {
                    const u64 b = stk[vp++], a = stk[vp++];
                    --fp;
                    push_val(binary(E, x, a, b));
                }
                break;
            case E_TERNARY:
                if (st == 0) {
                    stk[fp - 1] = fr | 1;
                    if (!x.a) {
                        bad = true;
                        break;
                    }
                    push_frame(x.a, 0);
                } else if (st == 1) {
                    const u64 cnd = stk[vp++];
                    const u32 side = cnd ? x.b : x.c;
                    stk[fp - 1] = (fr & ~0xffull) | 2;
                    if (!side) {
                        bad = true;
                        break;
                    }
                    push_frame(side, 0);
                } else {
                    --fp; // the taken side's value stays on the value stack
                }
                break;
            default:
                --fp;
                push_val(leaf(x));
                break;
            }
        }
        if (bad || full)
            return 0;
        return stk[vp];
    }
    // exec_body / exec_stmt  oracle.cpp:786-834, over the statement lists
    // (hoisted decls, then the body), If arms through a small list stack.
    OD_NOINL void run(u32 hoist, u32 body) {
        const KCtx &K = *c.K;
        u32 lst[64];
        u32 sp = 0;
        const u32 lists[2] = {hoist, body};
        for (u32 li = 0; li < 2 && !bad && !full; ++li) {
            lst[sp++] = K.lists[lists[li]].head;
            while (sp && !bad && !full) {
                const u32 si = lst[sp - 1];
                if (!si) {
                    --sp;
                    continue;
                }
                const Stmt &S = K.st[si];
                lst[sp - 1] = S.next;
                switch (S.kind) {
                case SK_ASSIGN: vars.set(sem_var_key(S.cls, S.a), eval(S.b)); break;
                case SK_DECL: vars.set(sem_var_key(S.cls, S.a), S.b ? eval(S.b) : 0); break;
                case SK_STORE: {
                    const u64 a = eval(S.a);
                    const u64 x = eval(S.b);
                    if (bad || full)
                        break;
                    mem.store(a, (u32)x);
                    if (dt_byte_size(S.c) == 8)
                        mem.store(a + 4, (u32)(x >> 32));
                    break;
                }
                case SK_IF: {
                    const u64 cnd = eval(S.a);
                    if (sp >= 64) {
                        full = true;
                        break;
                    }
                    lst[sp++] = cnd ? S.b : S.c;
                    break;
                }
                default: bad = true; break; // inline asm, labels, gotos
                }
                if (vars.full)
                    full = true;
            }
        }
    }
};

} // namespace od
