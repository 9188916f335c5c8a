// ocldec-b200: base definitions shared by every device pass.
//
// Fixed-width, pointer-free replacements for the reference's heap types:
//   DataType            type_recovery.hpp:37-62   -> one packed u32
//   Operand             asm_frontend.hpp:74-90    -> Opnd, 16 B
//   Expr (shared_ptr)   expr.hpp:99-128           -> 24 B arena node, u32 ids
// All device code is plain CUDA C++ for sm_100a; the same headers compile
// for the host only inside tools/devhost.cpp (a developer harness that is not
// part of the shipped library).
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define OD_HD __host__ __device__
#define OD_INL __host__ __device__ inline
#define OD_NOINL __host__ __device__ __noinline__ inline
// Hot lowering helpers: out of line by default (instruction-cache size);
// -DOD_HOT_INLINE=1 inlines them into their callers (locality experiment).
#if defined(OD_HOT_INLINE) && OD_HOT_INLINE
#define OD_HOT __host__ __device__ __forceinline__
#else
#define OD_HOT __host__ __device__ __noinline__ inline
#endif
#else
#define OD_HD
#define OD_INL inline
#ifdef OD_HOST_PROFILE
#define OD_NOINL inline __attribute__((noinline))
#else
#define OD_NOINL inline
#endif
#define OD_HOT OD_NOINL
#define __host__
#define __device__
struct uint4 {
    uint32_t x, y, z, w;
};
inline uint4 make_uint4(uint32_t x, uint32_t y, uint32_t z, uint32_t w) { return uint4{x, y, z, w}; }
#endif

namespace od {

typedef uint8_t u8;
typedef uint16_t u16;
typedef uint32_t u32;
typedef uint64_t u64;
typedef int32_t i32;
typedef int64_t i64;

// ---------------------------------------------------------------- DataType
// type_recovery.hpp:22-62.  Packed as base | bits<<8 | depth<<16 | space<<24.
enum Base : u32 { B_UNKNOWN = 0, B_BINARY, B_SIGNED, B_UNSIGNED, B_FLOAT, B_VOID };
enum Space : u32 { AS_NONE = 0, AS_GLOBAL, AS_LOCAL, AS_CONSTANT, AS_PRIVATE };

typedef u32 DT;
OD_INL DT dt_make(u32 base, u32 bits, u32 depth = 0, u32 space = 0) {
    return base | (bits << 8) | (depth << 16) | (space << 24);
}
OD_INL u32 dt_base(DT t) { return t & 0xff; }
OD_INL u32 dt_bits(DT t) { return (t >> 8) & 0xff; }
OD_INL u32 dt_depth(DT t) { return (t >> 16) & 0xff; }
OD_INL u32 dt_space(DT t) { return (t >> 24) & 0xff; }
OD_INL DT dt_with_bits(DT t, u32 bits) { return (t & ~0xff00u) | (bits << 8); }
OD_INL DT dt_with_base(DT t, u32 b) { return (t & ~0xffu) | b; }
OD_INL DT dt_with_space(DT t, u32 s) { return (t & 0x00ffffffu) | (s << 24); }
OD_INL bool dt_is_pointer(DT t) { return dt_depth(t) > 0; }
OD_INL bool dt_is_float(DT t) { return dt_base(t) == B_FLOAT && !dt_is_pointer(t); }
OD_INL bool dt_is_signed(DT t) { return dt_base(t) == B_SIGNED && !dt_is_pointer(t); }
OD_INL bool dt_is_unknown(DT t) { return dt_base(t) == B_UNKNOWN; }

#define DT_UNKNOWN (::od::dt_make(::od::B_UNKNOWN, 32))
#define DT_B32 (::od::dt_make(::od::B_BINARY, 32))
#define DT_B64 (::od::dt_make(::od::B_BINARY, 64))
#define DT_I32 (::od::dt_make(::od::B_SIGNED, 32))
#define DT_U32 (::od::dt_make(::od::B_UNSIGNED, 32))
#define DT_U64 (::od::dt_make(::od::B_UNSIGNED, 64))
#define DT_F32 (::od::dt_make(::od::B_FLOAT, 32))

// DataType::byte_size  type_recovery.cpp:13-25
OD_INL u32 dt_byte_size(DT t) {
    if (dt_is_pointer(t))
        return 8;
    switch (dt_bits(t)) {
    case 8: return 1;
    case 16: return 2;
    case 24:
    case 32: return 4;
    case 64: return 8;
    default: return 4;
    }
}

// DataType::pointee  type_recovery.cpp:27-34
OD_INL DT dt_pointee(DT t) {
    u32 d = dt_depth(t);
    if (d > 0)
        --d;
    u32 s = d == 0 ? AS_NONE : dt_space(t);
    return dt_make(dt_base(t), dt_bits(t), d, s);
}

OD_INL DT dt_pointer_to(DT t, u32 space) {
    return dt_make(dt_base(t), dt_bits(t), dt_depth(t) + 1, space);
}

// unify  type_recovery.cpp:84-121 (only .type is consumed by the pipeline)
OD_INL DT dt_unify(DT first, DT second) {
    if (first == second)
        return first;
    if (dt_base(first) == B_UNKNOWN)
        return second;
    if (dt_base(second) == B_UNKNOWN)
        return first;
    if (dt_is_pointer(first) || dt_is_pointer(second))
        return first;
    DT r = first;
    u32 bits = dt_bits(first) > dt_bits(second) ? dt_bits(first) : dt_bits(second);
    r = dt_with_bits(r, bits);
    if (dt_base(first) == dt_base(second))
        return r;
    if (dt_base(first) == B_BINARY)
        return dt_with_base(r, dt_base(second));
    return r;
}

// Type suffix (type_recovery.hpp:66-73): base letter code + width, packed
// as base<<8 | bits; 0 = none.
enum SfxBase : u32 { SB_I = 1, SB_U = 2, SB_F = 3, SB_B = 4 };
OD_INL u32 sfx_base(u32 s) { return s >> 8; }
OD_INL u32 sfx_bits(u32 s) { return s & 0xff; }
// type_from_suffix  type_recovery.cpp:75-82
OD_INL DT dt_from_suffix(u32 s) {
    switch (sfx_base(s)) {
    case SB_I: return dt_make(B_SIGNED, sfx_bits(s));
    case SB_U: return dt_make(B_UNSIGNED, sfx_bits(s));
    case SB_F: return dt_make(B_FLOAT, sfx_bits(s));
    default: return dt_make(B_BINARY, sfx_bits(s));
    }
}

OD_INL u32 ctz32(u32 m) {
#ifdef __CUDA_ARCH__
    return (u32)__ffs((int)m) - 1;
#else
    return (u32)__builtin_ctz(m);
#endif
}

OD_INL u32 ctz64(u64 m) {
#ifdef __CUDA_ARCH__
    return (u32)__ffsll((long long)m) - 1;
#else
    return (u32)__builtin_ctzll(m);
#endif
}

OD_INL u32 popc32(u32 m) {
#ifdef __CUDA_ARCH__
    return (u32)__popc(m);
#else
    return (u32)__builtin_popcount(m);
#endif
}

OD_INL u32 cas_u32(u32 *p, u32 cmp, u32 val) {
#ifdef __CUDA_ARCH__
    return atomicCAS(p, cmp, val);
#else
    const u32 o = *p;
    if (o == cmp)
        *p = val;
    return o;
#endif
}
OD_INL void max_u32(u32 *p, u32 v) {
#ifdef __CUDA_ARCH__
    atomicMax(p, v);
#else
    if (*p < v)
        *p = v;
#endif
}

OD_INL u64 fetch_add_u64(unsigned long long *p, u64 v) {
#ifdef __CUDA_ARCH__
    return (u64)atomicAdd(p, (unsigned long long)v);
#else
    const u64 o = *p;
    *p += v;
    return o;
#endif
}

// ------------------------------------------------------- warp cooperation
// k_front runs each kernel's front on all 32 lanes of its warp redundantly
// (every lane holds the same state and takes the same branches).  Loops over
// independent items are split across the lanes executing them (the active
// mask m): lane wrank(m) takes items wrank, wrank + wsize, ...; results are
// combined with warp reductions or written to distinct arena words and
// published with wsync.  The same code is correct on a lone lane (m has one
// bit: the loop covers every item), which is how the other phases and the
// host build run it.
OD_INL u32 wmask() {
#ifdef __CUDA_ARCH__
    return __activemask();
#else
    return 1u;
#endif
}
OD_INL u32 wrank(u32 m) {
#ifdef __CUDA_ARCH__
    return (u32)__popc(m & ((1u << (threadIdx.x & 31)) - 1));
#else
    (void)m;
    return 0;
#endif
}
OD_INL u32 wsize(u32 m) {
#ifdef __CUDA_ARCH__
    return (u32)__popc(m);
#else
    (void)m;
    return 1;
#endif
}
OD_INL bool wleader(u32 m) { return wrank(m) == 0; }
OD_INL void wsync(u32 m) {
#ifdef __CUDA_ARCH__
    __syncwarp(m);
#else
    (void)m;
#endif
}
OD_INL u32 wor(u32 m, u32 v) {
#ifdef __CUDA_ARCH__
    return __reduce_or_sync(m, v);
#else
    (void)m;
    return v;
#endif
}
OD_INL u32 wmax(u32 m, u32 v) {
#ifdef __CUDA_ARCH__
    return __reduce_max_sync(m, v);
#else
    (void)m;
    return v;
#endif
}
OD_INL u32 wadd(u32 m, u32 v) {
#ifdef __CUDA_ARCH__
    return __reduce_add_sync(m, v);
#else
    (void)m;
    return v;
#endif
}
OD_INL u32 wballot(u32 m, bool pred) {
#ifdef __CUDA_ARCH__
    return __ballot_sync(m, pred);
#else
    (void)m;
    return pred ? 1u : 0u;
#endif
}
// lanes of ballot b below this lane (b holds lane positions)
OD_INL u32 wbelow(u32 b) {
#ifdef __CUDA_ARCH__
    return (u32)__popc(b & ((1u << (threadIdx.x & 31)) - 1));
#else
    (void)b;
    return 0;
#endif
}
OD_INL u32 wmin(u32 m, u32 v) {
#ifdef __CUDA_ARCH__
    return __reduce_min_sync(m, v);
#else
    (void)m;
    return v;
#endif
}
// v of the mask's lowest lane
OD_INL u64 wbcast64(u32 m, u64 v) {
#ifdef __CUDA_ARCH__
    return __shfl_sync(m, (unsigned long long)v, __ffs(m) - 1);
#else
    (void)m;
    return v;
#endif
}

constexpr u32 kNoRank = 0xffffffffu;

// ------------------------------------------------------------- characters
// <cctype> in the "C" locale, as the reference uses it.
OD_INL bool c_space(u8 c) { return c == ' ' || (c >= 9 && c <= 13); }
OD_INL bool c_alpha(u8 c) { return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z'); }
OD_INL bool c_digit(u8 c) { return c >= '0' && c <= '9'; }
// asm_frontend.cpp:18-24
OD_INL bool c_ident_start(u8 c) { return c_alpha(c) || c == '_' || c == '.' || c == '$'; }
OD_INL bool c_ident_char(u8 c) { return c_ident_start(c) || c_digit(c) || c == '@'; }

// A byte span inside the listing buffer (offsets are chunk-relative).
struct Span {
    u32 off, len;
};

// trim (asm_frontend.cpp:26-40): isspace on both ends.
OD_INL Span trim_span(const u8 *t, Span s) {
    u32 b = s.off, e = s.off + s.len;
    while (b < e && (t[b] == ' ' || (t[b] >= 9 && t[b] <= 13)))
        ++b;
    while (e > b && (t[e - 1] == ' ' || (t[e - 1] >= 9 && t[e - 1] <= 13)))
        --e;
    return Span{b, e - b};
}

OD_INL u64 fnv1a64(const u8 *p, u32 n) {
    u64 h = 1469598103934665603ull;
    for (u32 i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

OD_INL bool span_eq(const u8 *t, Span a, const char *lit) {
    u32 i = 0;
    for (; i < a.len; ++i) {
        if (lit[i] == 0 || (u8)lit[i] != t[a.off + i])
            return false;
    }
    return lit[i] == 0;
}

OD_INL bool bytes_eq(const u8 *a, const u8 *b, u32 n) {
    for (u32 i = 0; i < n; ++i)
        if (a[i] != b[i])
            return false;
    return true;
}

// parse_int  asm_frontend.cpp:109-128: optional sign, decimal or 0x hex,
// full-match into uint64 (overflow fails), then int64 cast and negation.
OD_INL bool parse_int(const u8 *p, u32 n, i64 *out) {
    bool neg = false;
    if (n > 0 && (p[0] == '-' || p[0] == '+')) {
        neg = p[0] == '-';
        ++p;
        --n;
    }
    if (n == 0)
        return false;
    u32 base = 10;
    if (n > 2 && p[0] == '0' && (p[1] == 'x' || p[1] == 'X')) {
        base = 16;
        p += 2;
        n -= 2;
    }
    u64 v = 0;
    for (u32 i = 0; i < n; ++i) {
        u8 c = p[i];
        u32 d;
        if (c >= '0' && c <= '9')
            d = c - '0';
        else if (base == 16 && c >= 'a' && c <= 'f')
            d = c - 'a' + 10;
        else if (base == 16 && c >= 'A' && c <= 'F')
            d = c - 'A' + 10;
        else
            return false;
        // overflow of v * base + d, i.e. v > (2^64 - 1 - d) / base, without
        // the 64-bit division: base 16 overflows iff v >= 2^60; base 10 iff
        // v > 1844674407370955161, or v equals it and d > 5
        if (base == 16 ? (v >> 60) != 0
                       : (v > 1844674407370955161ull || (v == 1844674407370955161ull && d > 5)))
            return false;
        v = v * base + d;
    }
    i64 s = (i64)v;
    *out = neg ? (i64)(0ull - (u64)s) : s;
    return true;
}

// ---------------------------------------------------------------- operands
// OperandKind / SpecialReg  asm_frontend.hpp:64-72
enum OpKind : u8 { OK_SREG = 0, OK_VREG, OK_SPECIAL, OK_LITERAL, OK_SYMBOL, OK_ANNOT };
enum Special : u8 { SP_EXEC = 0, SP_VCC, SP_SCC, SP_M0, SP_EXEC_LO, SP_EXEC_HI, SP_VCC_LO, SP_VCC_HI };

struct Opnd {
    u8 kind;
    u8 special;
    u16 pad;
    u32 count;     // registers covered (1 for non-register kinds, 2 for exec/vcc)
    union {
        i64 value; // OK_LITERAL
        struct {
            u32 a; // register: first index; symbol/annotation: text offset
            u32 b; // symbol/annotation: text length
        } r;
    };
};

OD_INL bool op_is_sreg(const Opnd &o) { return o.kind == OK_SREG; }
OD_INL bool op_is_vreg(const Opnd &o) { return o.kind == OK_VREG; }
OD_INL bool op_is_special(const Opnd &o, u32 s) { return o.kind == OK_SPECIAL && o.special == s; }
OD_INL bool op_is_sreg_pair(const Opnd &o) { return o.kind == OK_SREG && o.count == 2; }

// ------------------------------------------------------------- mnemonics
// decompose_mnemonic  asm_frontend.cpp:375-423
enum Prefix : u8 { PX_OTHER = 0, PX_S, PX_V, PX_DS, PX_FLAT };

// Root strings the pipeline dispatches on.  Everything else is
// R_UNKNOWN plus the prefix flags below.
enum Root : u16 {
    R_UNKNOWN = 0,
    R_LOAD_DWORD, R_LOAD_DWORDX2, R_LOAD_DWORDX4, R_MOV, R_ADD, R_SUB, R_MUL, R_ADDK, R_MULK,
    R_AND, R_OR, R_XOR, R_ANDN2, R_LSHL, R_LSHR, R_ASHR, R_AND_SAVEEXEC, R_WAITCNT, R_NOP,
    R_ENDPGM, R_BRANCH, R_BARRIER, R_CNDMASK, R_SUBREV, R_ADDC, R_MUL_LO, R_MUL_HI, R_MAC,
    R_MAD, R_LSHLREV, R_LSHRREV, R_ASHRREV, R_STORE_DWORD, R_STORE_DWORDX2,
    R_CBRANCH_SCC0, R_CBRANCH_SCC1, R_CBRANCH_VCCZ, R_CBRANCH_VCCNZ, R_CBRANCH_EXECZ,
    R_CBRANCH_EXECNZ,
    R_CMP_EQ, R_CMP_NE, R_CMP_LG, R_CMP_NEQ, R_CMP_LT, R_CMP_LE, R_CMP_GT, R_CMP_GE,
    R_COUNT
};

// Prefix properties of the root string that the reference tests with rfind.
enum RootFlag : u8 {
    RF_CBRANCH = 1, // root starts with "cbranch_"   (cfg.cpp:44-46, 288)
    RF_CMP = 2,     // root starts with "cmp_"       (cfg.cpp:307, sym_state.cpp:543,765)
    RF_STORE = 4,   // root starts with "store"      (cfg.cpp:302)
    RF_LSHR = 8,    // root starts with "lshr"       (sym_state.cpp:748)
    RF_ASHR = 16,   // root starts with "ashr"       (sym_state.cpp:750)
};

#define OD_ROOT_STRINGS                                                                        \
    "", "load_dword", "load_dwordx2", "load_dwordx4", "mov", "add", "sub", "mul", "addk", "mulk", \
        "and", "or", "xor", "andn2", "lshl", "lshr", "ashr", "and_saveexec", "waitcnt", "nop",    \
        "endpgm", "branch", "barrier", "cndmask", "subrev", "addc", "mul_lo", "mul_hi", "mac",     \
        "mad", "lshlrev", "lshrrev", "ashrrev", "store_dword", "store_dwordx2", "cbranch_scc0",    \
        "cbranch_scc1", "cbranch_vccz", "cbranch_vccnz", "cbranch_execz", "cbranch_execnz",         \
        "cmp_eq", "cmp_ne", "cmp_lg", "cmp_neq", "cmp_lt", "cmp_le", "cmp_gt", "cmp_ge"

// ----------------------------------------------------------- registers
// Dense numbering  registers.hpp:38-48
enum : u32 {
    kSgprCount = 104,
    kVgprCount = 256,
    kRegIdVgpr0 = 104,
    kRegIdExecLo = 360,
    kRegIdExecHi = 361,
    kRegIdVccLo = 362,
    kRegIdVccHi = 363,
    kRegIdScc = 364,
    kRegIdM0 = 365,
    kNumRegIds = 366,
    kPhysSlots = 364, // exec and vcc halves share one slot (sym_state.cpp:37-50)
    kLiveWords = 12,  // ceil(366 / 32)
};

// RegisterFile::slot(id) -> physical slot / name class (sgpr, vgpr, exec,
// vcc, scc, m0), which is also what reg_id_name() prints (sym_state.cpp:16-33).
OD_INL u32 phys_of(u32 id) {
    if (id < kRegIdExecLo)
        return id;
    switch (id) {
    case kRegIdExecLo:
    case kRegIdExecHi: return 360;
    case kRegIdVccLo:
    case kRegIdVccHi: return 361;
    case kRegIdScc: return 362;
    default: return 363;
    }
}

// ------------------------------------------------------------ output text
// Bounds-checked byte writer; overflow sets a flag (the kernel is retried
// with a bigger arena).
struct Writer {
    u8 *p;
    u32 n, cap;
    bool overflow;
    OD_INL void put(u8 c) {
        if (n < cap)
            p[n] = c;
        else
            overflow = true;
        ++n;
    }
    // The bulk writers keep the cursor in registers and check the capacity
    // once per call (the writer itself lives in local memory).
    // string literal: length known at compile time
    template <u32 N> OD_INL void lit(const char (&s)[N]) { putn(reinterpret_cast<const u8 *>(s), N - 1); }
    OD_NOINL void puts(const char *s) {
        u8 *const d = p;
        const u32 c = cap;
        u32 k = n;
        bool ov = false;
        for (u8 ch; (ch = (u8)*s) != 0; ++s, ++k) {
            if (k < c)
                d[k] = ch;
            else
                ov = true;
        }
        n = k;
        if (ov)
            overflow = true;
    }
    OD_NOINL void putn(const u8 *s, u32 len) {
        const u32 k = n;
        if (k + len <= cap) {
            u8 *d = p + k;
            for (u32 i = 0; i < len; ++i)
                d[i] = s[i];
        } else {
            for (u32 i = 0; i < len; ++i)
                if (k + i < cap)
                    p[k + i] = s[i];
            overflow = true;
        }
        n = k + len;
    }
    OD_NOINL void put_u64(u64 v) {
        u8 buf[24];
        u32 k = 0;
        do {
            buf[k++] = u8('0' + v % 10);
            v /= 10;
        } while (v);
        u8 out[24];
        for (u32 i = 0; i < k; ++i)
            out[i] = buf[k - 1 - i];
        putn(out, k);
    }
    OD_NOINL void put_i64(i64 v) {
        if (v < 0) {
            put('-');
            put_u64(0ull - (u64)v);
        } else {
            put_u64((u64)v);
        }
    }
    OD_NOINL void put_hex(u64 v) {
        u8 buf[20];
        u32 k = 0;
        do {
            u32 d = u32(v & 15);
            buf[k++] = u8(d < 10 ? '0' + d : 'a' + d - 10);
            v >>= 4;
        } while (v);
        u8 out[20];
        for (u32 i = 0; i < k; ++i)
            out[i] = buf[k - 1 - i];
        putn(out, k);
    }
    OD_NOINL void spaces(u32 len) {
        const u32 k = n;
        if (k + len <= cap) {
            u8 *d = p + k;
            for (u32 i = 0; i < len; ++i)
                d[i] = ' ';
        } else {
            for (u32 i = 0; i < len; ++i)
                if (k + i < cap)
                    p[k + i] = ' ';
            overflow = true;
        }
        n = k + len;
    }
};

} // namespace od
