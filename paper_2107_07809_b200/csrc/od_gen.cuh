// ocldec-b200: counter-based synthetic GCN corpus generator.
//
// Kernel k of a corpus is a pure function of (shape, seed, k): its RNG state
// is splitmix64(seed ^ k) (the constants of oracle.cpp:22-27), and only
// integer arithmetic is used, so the host (CPU baseline, oracle checks) and
// the device (HBM-resident bench corpora) produce byte-identical listings.
//
// Vocabulary: the dispatch set of SURVEY A.1, in the corpus.cpp layout —
// implicit 6-argument block, s_load of pointer args at 0x30+, the
// s_lshl/v_add global-id idiom and the v_add/v_addc 64-bit address idiom —
// plus the seven make_nest branch layouts (nestgen.cpp:80-160) and back-edge
// loops.  Second ALU sources never alias the accumulator, which keeps the
// rendered expression trees linear (SURVEY §7 hard part 2).
#pragma once

#include "od_base.cuh"

namespace od {

enum GenShape : u32 {
    GS_C1 = 1, // small vector add (~40 instrs)
    GS_C2 = 2, // straight-line ALU kernels, 200 +- 50 instrs
    GS_C3 = 3, // branching kernels (nest layouts + 10% loops)
    GS_C4 = 4, // 70% C2-style / 30% C3-style, heavy-tailed size, mean ~500
    GS_C5 = 5, // long deep-CFG kernels, 10k +- 2k, 64-bit pairs
};

struct GenCfg {
    u32 shape;
    u32 stress; // sprinkle comments, odd syntax, fallbacks, failures (parity tests)
    u64 seed;
};

OD_INL u64 splitmix64(u64 x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

struct Gen {
    Writer *w;
    u64 st;
    u32 nins;
    u32 label;
    u32 stress;
    u32 nptr;     // pointer args (loaded in s[2i:2i+1] for i < 2, else s[10+2(i-2)])
    u32 ptr_kind[4]; // 0 int, 1 uint, 2 float, 3 long
    u32 nscal;    // scalar args loaded in s16..
    u32 scal_kind[3];
    u32 cws_log2;
    u32 budget;   // remaining conditionals (nests)
    u32 depth_max;

    OD_INL u64 rnd() {
        st += 0x9e3779b97f4a7c15ull;
        u64 z = st;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    OD_INL u32 r(u32 n) { return (u32)(rnd() % n); }

    // ---- text helpers
    OD_INL void I(const char *m) {
        w->puts("        ");
        w->puts(m);
        w->put(' ');
    }
    OD_INL void I0(const char *m) {
        w->puts("        ");
        w->puts(m);
    }
    OD_INL void E() {
        if (stress && r(40) == 0)
            w->puts(r(2) ? "   # note" : " ; trailing");
        w->put('\n');
        ++nins;
    }
    OD_INL void C() { w->puts(", "); }
    OD_INL void S(u32 n) {
        w->put('s');
        w->put_u64(n);
    }
    OD_INL void V(u32 n) {
        w->put('v');
        w->put_u64(n);
    }
    OD_INL void SP(u32 lo) {
        w->puts("s[");
        w->put_u64(lo);
        w->put(':');
        w->put_u64(lo + 1);
        w->put(']');
    }
    OD_INL void VP(u32 lo) {
        w->puts("v[");
        w->put_u64(lo);
        w->put(':');
        w->put_u64(lo + 1);
        w->put(']');
    }
    OD_INL void L(u64 v) {
        if (v < 4096)
            w->put_u64(v);
        else {
            w->puts("0x");
            w->put_hex(v);
        }
    }
    OD_INL void lab_def(u32 l) {
        w->puts("L");
        w->put_u64(l);
        w->puts(":\n");
    }
    OD_INL void lab_ref(u32 l) {
        w->puts("L");
        w->put_u64(l);
    }

    OD_INL u32 ptr_sreg(u32 i) const { return i < 2 ? 2 * i : 10 + 2 * (i - 2); }
    OD_INL u32 elem_shift(u32 i) const { return ptr_kind[i] == 3 ? 3 : 2; }

    // Literal palette: 80% [0,4095], 15% [4096, 2^32), 5% [-64,-1].
    OD_INL void lit() {
        u32 k = r(100);
        if (k < 80)
            w->put_u64(r(4096));
        else if (k < 95) {
            w->puts("0x");
            w->put_hex(4096 + (rnd() % 0xffffefffull));
        } else {
            w->put('-');
            w->put_u64(1 + r(64));
        }
    }
    OD_INL void flit() {
        // f32 palette of envgen.cpp:21-22 as bit patterns, plus pi
        static const u32 kF[12] = {0x00000000u, 0x3f800000u, 0xbf800000u, 0x3f000000u,
                                   0xbe800000u, 0x40000000u, 0x40600000u, 0xc1000000u,
                                   0x42c80000u, 0x3f400000u, 0xbe000000u, 0x40490fdbu};
        u32 b = kF[r(12)];
        w->puts("0x");
        w->put_hex(b);
    }

    // A second ALU source that is never the accumulator.
    OD_INL void src(u32 acc, u32 other_v, bool is_float) {
        u32 k = r(10);
        if (k < 3 && nscal) {
            S(16 + r(nscal));
        } else if (k < 6) {
            if (is_float)
                flit();
            else
                lit();
        } else if (k < 8 && other_v != acc) {
            V(other_v);
        } else {
            V(0); // global id (acc is never v0)
        }
    }

    // ---- header
    OD_INL void header(u64 k, u32 dims) {
        w->puts(".kernel k");
        w->put_u64(k);
        w->puts("\n    .config\n        .dims ");
        w->puts(dims == 1 ? "x" : dims == 2 ? "xy" : "xyz");
        w->puts("\n        .cws ");
        w->put_u64(1u << cws_log2);
        w->puts(", 1, 1\n        .sgprsnum 104\n        .vgprsnum 64\n        .useargs\n");
        w->puts("        .arg _.global_offset_0, \"size_t\", long\n"
                "        .arg _.global_offset_1, \"size_t\", long\n"
                "        .arg _.global_offset_2, \"size_t\", long\n"
                "        .arg _.printf_buffer, \"size_t\", void*, global, , rdonly\n"
                "        .arg _.vqueue_pointer, \"size_t\", long\n"
                "        .arg _.aqlwrap_pointer, \"size_t\", long\n");
        static const char *const kPT[4] = {"int*", "uint*", "float*", "long*"};
        static const char *const kPN[4] = {"src", "dst", "aux", "tab"};
        for (u32 i = 0; i < nptr; ++i) {
            w->puts("        .arg ");
            w->puts(kPN[i]);
            w->puts(", \"");
            w->puts(kPT[ptr_kind[i]]);
            w->puts("\", ");
            w->puts(kPT[ptr_kind[i]]);
            w->puts(", global\n");
        }
        static const char *const kST[3] = {"int", "uint", "float"};
        static const char *const kSN[3] = {"n", "m", "alpha"};
        for (u32 i = 0; i < nscal; ++i) {
            w->puts("        .arg ");
            w->puts(kSN[i]);
            w->puts(", \"");
            w->puts(kST[scal_kind[i]]);
            w->puts("\", ");
            w->puts(kST[scal_kind[i]]);
            w->put('\n');
        }
        w->puts("    .text\n");
    }

    // Prologue: pointer/scalar loads, global id in v0 (corpus.cpp:52-57).
    OD_INL void prologue(u32 dims) {
        u32 off = 0x30;
        for (u32 i = 0; i < nptr; ++i) {
            I("s_load_dwordx2");
            SP(ptr_sreg(i));
            C();
            SP(4);
            C();
            w->puts("0x");
            w->put_hex(off);
            E();
            off += 8;
        }
        for (u32 i = 0; i < nscal; ++i) {
            I("s_load_dword");
            S(16 + i);
            C();
            SP(4);
            C();
            w->puts("0x");
            w->put_hex(off);
            E();
            off += 4;
        }
        I("s_lshl_b32");
        S(9);
        C();
        S(6);
        C();
        w->put_u64(cws_log2);
        E();
        I("v_add_u32");
        V(0);
        C();
        w->puts("vcc");
        C();
        S(9);
        C();
        V(0);
        E();
        if (r(4) == 0) {
            // add the global offset back (copy_offset idiom)
            I("s_load_dwordx2");
            SP(20);
            C();
            SP(4);
            C();
            w->puts("0x0");
            E();
            I0("s_waitcnt lgkmcnt(0)");
            E();
            I("v_add_u32");
            V(0);
            C();
            w->puts("vcc");
            C();
            S(20);
            C();
            V(0);
            E();
        } else {
            I0("s_waitcnt lgkmcnt(0)");
            E();
        }
        if (dims > 1 && r(2)) {
            // touch the other dimensions' ids
            I("v_mov_b32");
            V(30);
            C();
            S(7);
            E();
            I("v_add_u32");
            V(30);
            C();
            w->puts("vcc");
            C();
            V(30);
            C();
            V(1);
            E();
        }
    }

    // Address of element v0 (+ optional offset reg) of pointer p into v[lo:lo+1].
    OD_INL void address(u32 p, u32 idx_v, u32 lo) {
        u32 t = lo + 2 < 60 ? lo + 2 : 1;
        I("v_lshlrev_b32");
        V(t);
        C();
        w->put_u64(elem_shift(p));
        C();
        V(idx_v);
        E();
        I("v_mov_b32");
        V(lo + 1);
        C();
        S(ptr_sreg(p) + 1);
        E();
        I("v_add_u32");
        V(lo);
        C();
        w->puts("vcc");
        C();
        S(ptr_sreg(p));
        C();
        V(t);
        E();
        I("v_addc_u32");
        V(lo + 1);
        C();
        w->puts("vcc");
        C();
        V(lo + 1);
        C();
        w->puts("0");
        C();
        w->puts("vcc");
        E();
    }

    // One VALU op updating acc.
    OD_INL void valu(u32 acc, u32 other, bool is_float, bool allow_select) {
        if (is_float) {
            switch (r(5)) {
            case 0:
                I("v_add_f32"); V(acc); C(); V(acc); C(); src(acc, other, true); E(); break;
            case 1:
                I("v_mul_f32"); V(acc); C(); src(acc, other, true); C(); V(acc); E(); break;
            case 2:
                I("v_mac_f32"); V(acc); C(); src(acc, other, true); C(); src(acc, other, true); E(); break;
            case 3:
                I("v_mad_f32"); V(acc); C(); V(acc); C(); src(acc, other, true); C(); src(acc, other, true); E(); break;
            default:
                if (allow_select) {
                    I("v_cmp_gt_f32"); w->puts("vcc"); C(); V(acc); C(); src(acc, other, true); E();
                    I("v_cndmask_b32"); V(acc); C(); V(acc); C(); src(acc, other, true); C(); w->puts("vcc"); E();
                } else {
                    I("v_sub_f32"); V(acc); C(); V(acc); C(); src(acc, other, true); E();
                }
                break;
            }
            return;
        }
        switch (r(15)) {
        case 0: I("v_add_u32"); V(acc); C(); w->puts("vcc"); C(); V(acc); C(); src(acc, other, false); E(); break;
        case 1: I("v_sub_u32"); V(acc); C(); w->puts("vcc"); C(); V(acc); C(); src(acc, other, false); E(); break;
        case 2: I("v_subrev_u32"); V(acc); C(); w->puts("vcc"); C(); src(acc, other, false); C(); V(acc); E(); break;
        case 3: I("v_mul_lo_u32"); V(acc); C(); V(acc); C(); src(acc, other, false); E(); break;
        case 4: I("v_mul_hi_u32"); V(acc); C(); V(acc); C(); src(acc, other, false); E(); break;
        case 5: I("v_and_b32"); V(acc); C(); V(acc); C(); src(acc, other, false); E(); break;
        case 6: I("v_or_b32"); V(acc); C(); src(acc, other, false); C(); V(acc); E(); break;
        case 7: I("v_xor_b32"); V(acc); C(); V(acc); C(); src(acc, other, false); E(); break;
        case 8: I("v_lshlrev_b32"); V(acc); C(); w->put_u64(1 + r(8)); C(); V(acc); E(); break;
        case 9: I("v_lshrrev_b32"); V(acc); C(); w->put_u64(1 + r(8)); C(); V(acc); E(); break;
        case 10: I("v_ashrrev_i32"); V(acc); C(); w->put_u64(1 + r(8)); C(); V(acc); E(); break;
        case 11: I("v_mad_u32_u24"); V(acc); C(); V(acc); C(); src(acc, other, false); C(); src(acc, other, false); E(); break;
        case 12: I("v_mul_u32_u24"); V(acc); C(); src(acc, other, false); C(); V(acc); E(); break;
        case 13: I("v_add_i32"); V(acc); C(); w->puts("vcc"); C(); src(acc, other, false); C(); V(acc); E(); break;
        default:
            if (allow_select) {
                I(r(2) ? "v_cmp_gt_u32" : "v_cmp_lt_i32"); w->puts("vcc"); C(); V(acc); C(); src(acc, other, false); E();
                I("v_cndmask_b32"); V(acc); C(); V(acc); C(); src(acc, other, false); C(); w->puts("vcc"); E();
            } else {
                I("v_lshlrev_b32"); V(acc); C(); w->put_u64(1 + r(4)); C(); V(acc); E();
            }
            break;
        }
    }

    // 1-3 SALU ops on scalar args into s24..s27, folded into acc.
    OD_INL void salu(u32 acc) {
        if (!nscal)
            return;
        u32 n = 1 + r(3);
        u32 d = 24 + r(4);
        static const char *const kOps[12] = {"s_add_u32", "s_sub_u32", "s_mul_i32", "s_and_b32",
                                             "s_or_b32", "s_xor_b32", "s_andn2_b32", "s_lshl_b32",
                                             "s_lshr_b32", "s_ashr_i32", "s_addk_i32", "s_mulk_i32"};
        I("s_mov_b32");
        S(d);
        C();
        S(16 + r(nscal));
        E();
        for (u32 i = 0; i < n; ++i) {
            u32 o = r(12);
            I(kOps[o]);
            S(d);
            C();
            if (o >= 10) {
                w->puts("0x");
                w->put_hex(1 + r(255));
            } else {
                S(d);
                C();
                if (o >= 7)
                    w->put_u64(1 + r(7));
                else if (r(2))
                    S(16 + r(nscal));
                else
                    lit();
            }
            E();
        }
        I("v_add_u32");
        V(acc);
        C();
        w->puts("vcc");
        C();
        S(d);
        C();
        V(acc);
        E();
    }

    // Stress-only oddities (never in bench shapes).
    OD_INL void oddity() {
        switch (r(9)) {
        case 0: I("ds_read_b32"); V(40); C(); V(0); E(); break;
        case 1: I0("s_barrier"); E(); break;
        case 2: I("v_cmpx_lt_u32"); w->puts("vcc"); C(); V(0); C(); w->put_u64(r(50)); E(); break;
        case 3: I0("s_nop 0"); E(); break;
        case 4: I("v_mov_b32"); V(41); C(); S(5); w->puts("    /* mid */ "); E(); break;
        case 5: I("s_mov_b32"); w->puts("m0"); C(); w->puts("-1"); E(); break;
        case 6: I("v_mov_b32"); V(42); C(); w->puts("s[5:3]"); E(); break; // parse_failed
        case 7: w->puts("\n   \n"); break;
        default: I("flat_load_dword"); V(43); C(); VP(2); w->puts(" glc slc"); E(); break;
        }
    }

    // Load-compute-store group (~10-16 instrs).
    OD_INL void group(u32 nvalu) {
        u32 p = r(nptr);
        u32 q = r(nptr);
        u32 lo = 2 + 2 * r(8);     // address pair v[lo:lo+1], lo in 2..16
        u32 acc = 20 + r(10);      // accumulator v20..v29
        u32 other = 31 + r(6);     // an older value v31..v36
        bool fl = ptr_kind[p] == 2;
        bool wide = ptr_kind[p] == 3;
        address(p, 0, lo);
        if (wide) {
            I("flat_load_dwordx2");
            VP(acc & ~1u);
            C();
            VP(lo);
            E();
            I0("s_waitcnt vmcnt(0)");
            E();
            u32 q2 = r(nptr);
            u32 lo2 = 44 + 2 * r(4);
            address(q2, 0, lo2);
            if (ptr_kind[q2] == 3) {
                I("flat_store_dwordx2");
                VP(lo2);
                C();
                VP(acc & ~1u);
                E();
            } else {
                I("flat_store_dword");
                VP(lo2);
                C();
                V(acc & ~1u);
                E();
            }
            return;
        }
        I("flat_load_dword");
        V(acc);
        C();
        VP(lo);
        E();
        I0("s_waitcnt vmcnt(0)");
        E();
        if (r(3) == 0) {
            I("v_mov_b32");
            V(other);
            C();
            V(acc);
            E();
        }
        bool sel = true;
        for (u32 i = 0; i < nvalu; ++i) {
            valu(acc, other, fl, sel);
            sel = false;
        }
        if (!fl && r(2))
            salu(acc);
        if (stress && r(6) == 0)
            oddity();
        if (q != p && ptr_kind[q] != 3) {
            u32 lo2 = 44 + 2 * r(4);
            address(q, 0, lo2);
            lo = lo2;
        }
        I("flat_store_dword");
        VP(lo);
        C();
        V(acc);
        E();
    }

    // Small payload used inside branch arms.
    OD_INL void payload(u32 depth) {
        u32 k = r(4);
        if (k == 0) {
            group(1 + r(2));
        } else {
            u32 v = 20 + r(10);
            I("v_mov_b32");
            V(v);
            C();
            lit();
            E();
            if (k == 1) {
                valu(v, 31 + r(6), false, false);
            }
            if (k == 3 && nscal) {
                I("s_add_u32");
                S(28 + r(3));
                C();
                S(16 + r(nscal));
                C();
                w->put_u64(r(100));
                E();
            }
        }
        (void)depth;
    }

    OD_INL void mask(u32 depth) {
        SP(32 + 2 * depth);
    }
    OD_INL void cmp_vcc() {
        I(r(2) ? "v_cmp_lt_u32" : "v_cmp_gt_u32");
        w->puts("vcc");
        C();
        V(0);
        C();
        if (nscal && r(2))
            S(16 + r(nscal));
        else
            w->put_u64(1 + r(300));
        E();
    }
    OD_INL void cmp_scc() {
        I(r(2) ? "s_cmp_lt_u32" : "s_cmp_eq_u32");
        S(nscal ? 16 + r(nscal) : 9);
        C();
        w->put_u64(r(20));
        E();
    }

    // nestgen.cpp:48-59 body: payload, then up to 2 conditionals.
    OD_INL void body(u32 depth) {
        payload(depth);
        if (depth < depth_max) {
            u32 items = r(3);
            for (u32 i = 0; i < items && budget > 0; ++i) {
                --budget;
                conditional(depth);
                payload(depth);
            }
        }
    }

    // nestgen.cpp:61-160 (the seven layouts)
    OD_INL void conditional(u32 depth) {
        const bool with_else = r(2) == 0;
        if (with_else) {
            switch (r(4)) {
            case 0: { // scc diamond
                u32 els = label++, join = label++;
                cmp_scc();
                I("s_cbranch_scc0");
                lab_ref(els);
                E();
                body(depth + 1);
                I("s_branch");
                lab_ref(join);
                E();
                lab_def(els);
                body(depth + 1);
                lab_def(join);
                break;
            }
            case 1: { // mask form 1
                u32 flow = label++, join = label++;
                cmp_vcc();
                I("s_and_saveexec_b64");
                mask(depth);
                C();
                w->puts("vcc");
                E();
                I("s_cbranch_execz");
                lab_ref(flow);
                E();
                body(depth + 1);
                lab_def(flow);
                I("s_xor_b64");
                w->puts("exec, exec, ");
                mask(depth);
                E();
                I("s_cbranch_execz");
                lab_ref(join);
                E();
                body(depth + 1);
                lab_def(join);
                I("s_or_b64");
                w->puts("exec, exec, ");
                mask(depth);
                E();
                break;
            }
            case 2: { // mask form 2
                cmp_vcc();
                I("s_and_saveexec_b64");
                mask(depth);
                C();
                w->puts("vcc");
                E();
                body(depth + 1);
                I("s_andn2_b64");
                w->puts("exec, ");
                mask(depth);
                w->puts(", exec");
                E();
                body(depth + 1);
                I("s_or_b64");
                w->puts("exec, exec, ");
                mask(depth);
                E();
                break;
            }
            default: { // mask form 3
                u32 join = label++;
                cmp_vcc();
                I("s_and_saveexec_b64");
                mask(depth);
                C();
                w->puts("vcc");
                E();
                body(depth + 1);
                I("s_xor_b64");
                w->puts("exec, exec, ");
                mask(depth);
                E();
                I("s_cbranch_execz");
                lab_ref(join);
                E();
                body(depth + 1);
                lab_def(join);
                I("s_or_b64");
                w->puts("exec, exec, ");
                mask(depth);
                E();
                break;
            }
            }
        } else {
            switch (r(3)) {
            case 0: { // scc if
                u32 end = label++;
                cmp_scc();
                I("s_cbranch_scc0");
                lab_ref(end);
                E();
                body(depth + 1);
                lab_def(end);
                break;
            }
            case 1: { // mask bypass
                u32 end = label++;
                cmp_vcc();
                I("s_and_saveexec_b64");
                mask(depth);
                C();
                w->puts("vcc");
                E();
                I("s_cbranch_execz");
                lab_ref(end);
                E();
                body(depth + 1);
                lab_def(end);
                I("s_or_b64");
                w->puts("exec, exec, ");
                mask(depth);
                E();
                break;
            }
            default: { // mask plain
                cmp_vcc();
                I("s_and_saveexec_b64");
                mask(depth);
                C();
                w->puts("vcc");
                E();
                body(depth + 1);
                I("s_or_b64");
                w->puts("exec, exec, ");
                mask(depth);
                E();
                break;
            }
            }
        }
    }

    // A back-edge loop: labels and gotos in the output (lower.cpp:187-250).
    OD_INL void loop() {
        u32 top = label++;
        I("s_mov_b32");
        S(26);
        C();
        w->puts("0");
        E();
        lab_def(top);
        payload(0);
        I("s_add_u32");
        S(26);
        C();
        S(26);
        C();
        w->puts("1");
        E();
        I("s_cmp_lt_u32");
        S(26);
        C();
        w->put_u64(2 + r(14));
        E();
        I(r(4) ? "s_cbranch_scc1" : "s_cbranch_vccnz");
        lab_ref(top);
        E();
    }
};

// Target instruction count for kernel k of a shape (integer-only draws).
OD_INL u32 gen_target(Gen &g, u32 shape) {
    switch (shape) {
    case GS_C1: return 40;
    case GS_C2: return 150 + g.r(101);
    case GS_C4: {
        // heavy-tailed mix with mean ~500, clamped to [40, 4000]
        u32 k = g.r(100);
        if (k < 85)
            return 40 + g.r(761);
        if (k < 98)
            return 40 + g.r(1961);
        return 40 + g.r(3961);
    }
    case GS_C5: return 8000 + g.r(4001);
    default: return 0;
    }
}

// Writes kernel k of the corpus into *w (w->cap == 0: sizing only).
// Returns the number of instruction lines emitted.
OD_NOINL u32 gen_kernel(const GenCfg &cfg, u64 k, Writer *w) {
    Gen g;
    g.w = w;
    g.st = splitmix64(cfg.seed ^ (k * 0x9e3779b97f4a7c15ull + 0x2107078090ull));
    g.nins = 0;
    g.label = 0;
    g.stress = cfg.stress;
    g.budget = 0;
    g.depth_max = 6;
    u32 shape = cfg.shape;
    bool branching = shape == GS_C3 || shape == GS_C5;
    if (shape == GS_C4)
        branching = g.r(10) < 3;
    g.cws_log2 = 6 + g.r(3);
    u32 dims = 1;
    if (g.r(8) == 0)
        dims = 2 + g.r(2);
    g.nptr = 2 + g.r(2);
    for (u32 i = 0; i < g.nptr; ++i) {
        u32 pk = g.r(3);
        if (shape == GS_C5 && g.r(2))
            pk = 3;
        g.ptr_kind[i] = pk;
    }
    g.nscal = 1 + g.r(3);
    for (u32 i = 0; i < g.nscal; ++i)
        g.scal_kind[i] = g.r(2);
    if (g.r(4) == 0)
        g.scal_kind[g.nscal - 1] = 2;
    g.header(k, dims);
    g.prologue(dims);
    u32 target = gen_target(g, shape);
    if (shape == GS_C1) {
        // vector add: two loads, add, store (plus a few ALU ops)
        g.nptr = g.nptr < 3 ? g.nptr : 3;
        while (g.nins + 12 < target)
            g.group(1 + g.r(3));
    } else if (!branching) {
        while (g.nins + 14 < target)
            g.group(3 + g.r(4));
    } else if (shape == GS_C3) {
        g.budget = 1 + g.r(14);
        if (g.r(10) == 0)
            g.loop();
        g.payload(0);
        u32 top = 1 + g.r(2);
        for (u32 i = 0; i < top && g.budget > 0; ++i) {
            --g.budget;
            g.conditional(0);
            g.payload(0);
        }
    } else {
        // long branching kernels: sequential nests until the target
        if (target == 0)
            target = 300;
        bool looped = false;
        while (g.nins < target) {
            g.budget = 1 + g.r(14);
            if (!looped && shape != GS_C5 && g.r(10) == 0) {
                g.loop();
                looped = true;
            }
            --g.budget;
            g.conditional(0);
            g.payload(0);
            if (g.r(3) == 0)
                g.group(2 + g.r(3));
        }
    }
    if (cfg.stress && g.r(10) == 0) {
        // trailing label after the last instruction: synthetic s_endpgm
        w->puts("L_tail:\n");
        return g.nins;
    }
    g.I0("s_endpgm");
    w->put('\n');
    return g.nins + 1;
}

} // namespace od
