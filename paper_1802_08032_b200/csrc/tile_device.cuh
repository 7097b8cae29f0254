// tile_device.cuh — device code of the tile pass (the hot kernel), shared by
// the ahead-of-time build (tile_pass.cu: the interpreter instantiation) and
// the per-pass JIT (tile_jit.cpp compiles it with NVRTC together with a
// generated straight-line program for one pass shape).
//
// Structure (qgpu_device.h: TileParams / TilePhase / TileOp):
//  * one persistent CTA (16 warps) per SM walks tiles of 2^12 amplitudes
//    (qubits 0-4 plus 7 higher qubits chosen per pass);
//  * HBM <-> shared memory through TMA bulk copies, three 64 KiB stages
//    deep: each warp loads, stores and refills the 8 segments (512 B runs of
//    qubits 0-4) it owns in the last phase, posting its bytes on the stage's
//    tx-count mbarrier (16 arrivals per fill) — no end-of-tile block barrier;
//  * the ops run in phases: every thread holds 8 amplitudes in registers
//    spanning the phase's 3 register qubits; lane bits 0-2 span qubits 0-2,
//    lane bits 3-4 qubits 3-4 or two other tile qubits, the 16 warps the
//    rest. Pair ops on register qubits stay in registers, on lane qubits
//    they use warp shuffles, diagonal gates and channels are elementwise
//    anywhere; between phases the tile is re-laid out through shared memory
//    behind a barrier over the warps that exchange data (named barriers for
//    groups, the CTA otherwise).
//
// Code-generation notes (each measured with ncu on this kernel):
//  * interpreter: the op table is copied to shared memory once per launch,
//    an op's header and coefficients are loaded one op ahead (OpCtx), the
//    host resolves each op to one handler code (TileCode) and the build
//    passes -jump-table-density=1 to NVVM: one brx.idx per op;
//  * JIT: the same handlers, called straight-line (step_c<RB, CODE>) with
//    literal headers and layouts; coefficients as constant-bank operands;
//  * outer-qubit controls are evaluated once per tile (a ballot per 32 ops),
//    not per op and phase;
//  * handlers never branch per element on run-time values (selects only where
//    lane / register controls need them) — per-element branches made ptxas
//    copy the whole 64-register tile around them;
//  * coefficient signs are applied to register operands (exact), so the
//    coefficients themselves can stay constant-bank operands.
#pragma once

#include "pair_math.cuh"

namespace qgpu {

namespace {

template <int RB>
using Regs = double2[1 << RB];

// ------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem_dst)),
        "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_store(void* gmem_dst, const void* smem_src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem_dst),
                 "r"(smem_u32(smem_src)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void tma_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void tma_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// 16-byte shared-memory accesses as single v2.f64 instructions: left to
// itself ptxas split some into two 8-byte accesses when the two doubles sat
// in non-adjacent registers, which made 2-way bank conflicts (ncu: 26 %
// excess wavefronts in JIT kernels)
#ifdef QGPU_PLAIN_SMEM
__device__ __forceinline__ double2 lds16(const double2* p) { return *p; }
__device__ __forceinline__ void sts16(double2* p, double2 v) { *p = v; }
#else
__device__ __forceinline__ double2 lds16(const double2* p) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
    return v;
}
__device__ __forceinline__ void sts16(double2* p, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(smem_u32(p)), "d"(v.x), "d"(v.y) : "memory");
}
#endif

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- handlers
//
// Ping-pong: every handler reads the tile s and writes every element of the
// tile d (a fresh register set), so the results of all switch arms land in
// the same registers with no copies; the op loop alternates s and d. (An
// in-place update leaves each pair's results in rotated registers, and ptxas
// then copies the whole tile back at every loop iteration: measured 30 %
// slower.) SEL variants apply a per-element predicate: register controls
// `rcm` and lane controls (`tok`).

__device__ __forceinline__ double2 diag_a(const double* c, double2 v) {
    return make_double2(fma(c[0], v.x, -(c[1] * v.y)), fma(c[0], v.y, c[1] * v.x));
}
__device__ __forceinline__ double2 diag_d(const double* c, double2 v) {
    // fma(-d_im, y, ...) with the (exact) negation on the register operand
    return make_double2(fma(c[7], -v.y, c[6] * v.x), fma(c[7], v.x, c[6] * v.y));
}

__device__ __forceinline__ bool sel_on(int i, uint32_t rcm, bool tok) {
    return tok && (static_cast<uint32_t>(i) & rcm) == rcm;
}

// 2x2 gate on register bit J (compile time).
template <int RB, int J, int CLS, bool SEL>
__device__ __forceinline__ void h_reg(const Regs<RB>& s, Regs<RB>& d, const double* c, uint32_t rcm,
                                      bool tok) {
    if constexpr (J < RB) {
#pragma unroll
        for (int lo = 0; lo < (1 << RB); ++lo) {
            constexpr int bit = 1 << J;
            if (lo & bit) continue;
            double2 l = s[lo], h = s[lo | bit];
            pair_update<CLS>(l, h, c);
            if constexpr (SEL) {
                const bool on = sel_on(lo, rcm, tok);
                d[lo] = on ? l : s[lo];
                d[lo | bit] = on ? h : s[lo | bit];
            } else {
                d[lo] = l;
                d[lo | bit] = h;
            }
        }
    }
}

// 2x2 gate on lane bit b: the partner amplitude comes from lane ^ 2^b, and
// each lane computes its own half (distributed.cpp:183-184:
// own_lo ? lo_out(mine, theirs) : hi_out(theirs, mine)).
template <int RB, int CLS, bool SEL>
__device__ __forceinline__ void h_lane(const Regs<RB>& s, Regs<RB>& d, const double* c, uint32_t b,
                                       uint32_t rcm, bool tok, uint32_t lane) {
    const uint32_t mask = 1u << b;
    const bool own_lo = (lane & mask) == 0;
    const double q0 = own_lo ? c[0] : c[4], q1 = own_lo ? c[1] : c[5];
    const double q2 = own_lo ? c[2] : c[6], q3 = own_lo ? c[3] : c[7];
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) {
        double2 th;
        th.x = __shfl_xor_sync(0xffffffffu, s[i].x, mask);
        th.y = __shfl_xor_sync(0xffffffffu, s[i].y, mask);
        double2 r;
        if constexpr (CLS == CLS_SWAP) {
            r = th;
        } else {
            const double2 lo = own_lo ? s[i] : th;
            const double2 hi = own_lo ? th : s[i];
            r = row<CLS == CLS_REAL ? 0b1010 : 0>(q0, q1, q2, q3, lo, hi);
        }
        if constexpr (SEL)
            d[i] = sel_on(i, rcm, tok) ? r : s[i];
        else
            d[i] = r;
    }
}

// Diagonal gate, target on register bit J: a * v where the bit is 0, d * v
// where it is 1 (rounding of the reference's low / high row). DO_A = false
// leaves the low side alone (a == 1 exactly).
template <int RB, int J, bool DO_A, bool SEL>
__device__ __forceinline__ void h_diag_reg(const Regs<RB>& s, Regs<RB>& d, const double* c, uint32_t rcm,
                                           bool tok) {
    if constexpr (J < RB) {
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            const bool bit = (i >> J) & 1;
            if (!bit && !DO_A) { // compile time
                d[i] = s[i];
                continue;
            }
            const double2 r = bit ? diag_d(c, s[i]) : diag_a(c, s[i]);
            if constexpr (SEL)
                d[i] = sel_on(i, rcm, tok) ? r : s[i];
            else
                d[i] = r;
        }
    }
}

// Diagonal gate whose target bit differs per lane: coefficients picked once
// per thread; per element the operands swap:
//   re = fma(P, X1, Q * Y1), im = fma(R, Y2, S * X2)
//   bit 0: P = R = a_re, Q = S = a_im, (X1, Y1) = (x, -y), (X2, Y2) = (x, y)  (diag_a)
//   bit 1: P = R = d_im, Q = S = d_re, (X1, Y1) = (-y, x), (X2, Y2) = (y, x)  (diag_d)
// (negations are exact, and sit on register operands: see diag_d)
template <int RB, bool SEL>
__device__ __forceinline__ void h_diag_lane(const Regs<RB>& s, Regs<RB>& d, const double* c, uint32_t bit,
                                            uint32_t rcm, bool tok) {
    // signs moved from the coefficients onto the (exact) operand negations
    const double P = bit ? c[7] : c[0], Q = bit ? c[6] : c[1];
    const double R = bit ? c[7] : c[0], S = bit ? c[6] : c[1];
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) {
        const double x = s[i].x, y = s[i].y;
        const double X1 = bit ? -y : x, Y1 = bit ? x : -y; // re = fma(P, X1, Q * Y1)
        const double X2 = bit ? y : x, Y2 = bit ? x : y;   // im = fma(R, Y2, S * X2)
        const double2 r = make_double2(fma(P, X1, Q * Y1), fma(R, Y2, S * X2));
        if constexpr (SEL)
            d[i] = sel_on(i, rcm, tok) ? r : s[i];
        else
            d[i] = r;
    }
}

// Diagonal gate whose target bit is the same for the whole warp (a warp or
// outer qubit): a warp-uniform branch picks the side.
template <int RB, bool SEL>
__device__ __forceinline__ void h_diag_uniform(const Regs<RB>& s, Regs<RB>& d, const double* c, uint32_t bit,
                                               uint32_t rcm, bool tok) {
    if (bit) {
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            const double2 r = diag_d(c, s[i]);
            d[i] = SEL ? (sel_on(i, rcm, tok) ? r : s[i]) : r;
        }
    } else {
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            const double2 r = diag_a(c, s[i]);
            d[i] = SEL ? (sel_on(i, rcm, tok) ? r : s[i]) : r;
        }
    }
}

template <int RB>
__device__ __forceinline__ void h_copy(const Regs<RB>& s, Regs<RB>& d) {
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) d[i] = s[i];
}

__device__ __forceinline__ uint32_t fixed_bit_of(uint32_t kind, uint32_t pos, uint32_t lane, uint32_t w,
                                                 uint64_t gbase) {
    return kind == TL_LANE   ? (lane >> pos) & 1u
           : kind == TL_WARP ? (w >> pos) & 1u
                             : static_cast<uint32_t>((gbase >> pos) & 1u);
}

// An op's header and coefficients, loaded one op ahead.
struct OpCtx {
    uint64_t h;
    double c[8];
};

// Explicit shared-window addresses: through a generic pointer, ptxas
// re-derived the CTA's shared window (S2R SR_CgaCtaId) at every op.
__device__ __forceinline__ void load_ctx(OpCtx& x, uint32_t sops_addr, int o) {
    const uint32_t a = sops_addr + static_cast<uint32_t>(o) * static_cast<uint32_t>(sizeof(TileOp));
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(x.h) : "r"(a));
#pragma unroll
    for (int k = 0; k < 8; k += 2)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                     : "=d"(x.c[k]), "=d"(x.c[k + 1])
                     : "r"(a + 16u + 8u * static_cast<uint32_t>(k)));
}

// Coefficients only (a JIT program's headers are literals). Volatile, so
// NVVM cannot hoist them out of the tile loop: hoisting all of a pass's
// coefficients into registers spilled (measured: 128 regs + 576 B stack).
__device__ __forceinline__ void load_coef(OpCtx& x, uint32_t sops_addr, int o) {
    const uint32_t a = sops_addr + static_cast<uint32_t>(o) * static_cast<uint32_t>(sizeof(TileOp));
#pragma unroll
    for (int k = 0; k < 8; k += 2)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                     : "=d"(x.c[k]), "=d"(x.c[k + 1])
                     : "r"(a + 16u + 8u * static_cast<uint32_t>(k)));
}

// Controls on outer qubits are uniform per tile: per tile, each warp
// evaluates them once for all ops (one ballot per 32 ops) into a 64-bit mask
// of the ops that run; the op loop walks the set bits. Controls on warp
// qubits are not skipped but folded into the per-element predicate like lane
// / register ones: a warp that skipped would idle at the next phase barrier
// while its sub-partition ran the other warps alone.
__device__ __forceinline__ uint64_t active_ops(const TileOp* ops, int nops, uint64_t gbase, uint32_t lane) {
    bool a0 = false, a1 = false;
    if (static_cast<int>(lane) < nops) {
        const uint64_t m = ops[lane].outer_cmask;
        a0 = (gbase & m) == m;
    }
    if (static_cast<int>(lane) + 32 < nops) {
        const uint64_t m = ops[lane + 32].outer_cmask;
        a1 = (gbase & m) == m;
    }
    return static_cast<uint64_t>(__ballot_sync(0xffffffffu, a0)) |
           static_cast<uint64_t>(__ballot_sync(0xffffffffu, a1)) << 32;
}

__device__ __forceinline__ int lowest(uint64_t m) { return __ffsll(static_cast<long long>(m)) - 1; }

// One op of handler code CODE: s -> d. The header's other fields are decoded
// here (constants when the JIT emits the header as a literal). The
// interpreter reaches this through step() (one jump table per op); a JIT
// program instantiates only the codes it uses.
template <int RB, int CODE>
__device__ __forceinline__ void step_c(const Regs<RB>& s, Regs<RB>& d, const OpCtx& x, uint32_t lane,
                                       uint32_t w, uint64_t gbase) {
    const uint64_t h = x.h;
    const double* c = x.c;
    const uint32_t q0p = (h >> 13) & 63u;
    const uint32_t rcm = static_cast<uint32_t>((h >> 32) & 15u);
    const uint32_t lcm = static_cast<uint32_t>((h >> 27) & 31u), wcm = static_cast<uint32_t>((h >> 36) & 15u);
    const bool tok = (lane & lcm) == lcm && (w & wcm) == wcm;
    if constexpr (CODE >= TC_REG && CODE < TC_REG + 16) {
        constexpr int row = (CODE - TC_REG) / 4, J = (CODE - TC_REG) % 4;
        constexpr int CLS = row == 0 ? CLS_GENERIC : row == 1 ? CLS_REAL : row == 2 ? CLS_RX : CLS_SWAP;
        h_reg<RB, J, CLS, false>(s, d, c, 0, true);
    } else if constexpr (CODE >= TC_REG_SEL && CODE < TC_REG_SEL + 8) {
        constexpr int J = (CODE - TC_REG_SEL) % 4;
        constexpr int CLS = (CODE - TC_REG_SEL) / 4 == 0 ? CLS_GENERIC : CLS_SWAP;
        h_reg<RB, J, CLS, true>(s, d, c, rcm, tok);
    } else if constexpr (CODE == TC_LANE_GENERIC) {
        h_lane<RB, CLS_GENERIC, false>(s, d, c, q0p, 0, true, lane);
    } else if constexpr (CODE == TC_LANE_REAL) {
        h_lane<RB, CLS_REAL, false>(s, d, c, q0p, 0, true, lane);
    } else if constexpr (CODE == TC_LANE_SWAP) {
        h_lane<RB, CLS_SWAP, false>(s, d, c, q0p, 0, true, lane);
    } else if constexpr (CODE == TC_LANE_SEL_GENERIC) {
        h_lane<RB, CLS_GENERIC, true>(s, d, c, q0p, rcm, tok, lane);
    } else if constexpr (CODE == TC_LANE_SEL_SWAP) {
        h_lane<RB, CLS_SWAP, true>(s, d, c, q0p, rcm, tok, lane);
    } else if constexpr (CODE >= TC_DIAG_REG && CODE < TC_DIAG_REG + 4) {
        h_diag_reg<RB, CODE - TC_DIAG_REG, true, false>(s, d, c, 0, true);
    } else if constexpr (CODE >= TC_DIAG_REG_D && CODE < TC_DIAG_REG_D + 4) {
        h_diag_reg<RB, CODE - TC_DIAG_REG_D, false, false>(s, d, c, 0, true);
    } else if constexpr (CODE >= TC_DIAG_REG_SEL && CODE < TC_DIAG_REG_SEL + 4) {
        h_diag_reg<RB, CODE - TC_DIAG_REG_SEL, true, true>(s, d, c, rcm, tok);
    } else if constexpr (CODE >= TC_DIAG_REG_D_SEL && CODE < TC_DIAG_REG_D_SEL + 4) {
        h_diag_reg<RB, CODE - TC_DIAG_REG_D_SEL, false, true>(s, d, c, rcm, tok);
    } else if constexpr (CODE == TC_DIAG_LANE) {
        h_diag_lane<RB, false>(s, d, c, (lane >> q0p) & 1u, 0, true);
    } else if constexpr (CODE == TC_DIAG_LANE_SEL) {
        h_diag_lane<RB, true>(s, d, c, (lane >> q0p) & 1u, rcm, tok);
    } else if constexpr (CODE == TC_DIAG_UNIFORM || CODE == TC_DIAG_UNIFORM_SEL) {
        const uint32_t flags = (h >> 6) & 15u;
        const uint32_t bit = fixed_bit_of((h >> 11) & 3u, q0p, lane, w, gbase);
        if (bit ? (flags & DF_D_ONE) : (flags & DF_A_ONE)) // identity side
            h_copy<RB>(s, d);
        else if constexpr (CODE == TC_DIAG_UNIFORM)
            h_diag_uniform<RB, false>(s, d, c, bit, 0, true);
        else
            h_diag_uniform<RB, true>(s, d, c, bit, rcm, tok);
    } else if constexpr (CODE == TC_DEPHASE) { // density.cpp:56-59: scale where bit(q0) != bit(q1)
        const uint32_t q0k = (h >> 11) & 3u, q1k = (h >> 19) & 3u, q1p = (h >> 21) & 63u;
        const uint32_t rm = (q0k == TL_REG ? 1u << q0p : 0u) ^ (q1k == TL_REG ? 1u << q1p : 0u);
        const uint32_t f = (q0k == TL_REG ? 0u : fixed_bit_of(q0k, q0p, lane, w, gbase)) ^
                           (q1k == TL_REG ? 0u : fixed_bit_of(q1k, q1p, lane, w, gbase));
        const double sc = c[0];
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            const bool on = (__popc(static_cast<uint32_t>(i) & rm) & 1u) ^ f;
            const double k = on ? sc : 1.0; // x * 1.0 is exact
            d[i] = make_double2(s[i].x * k, s[i].y * k);
        }
    } else if constexpr (CODE >= TC_DEPOL && CODE < TC_DEPOL + 6) {
        // depolarising on register bits J0 < J1 (t and t+N of a density
        // matrix), the arithmetic of k_depolarise (density.cpp:62-81): the
        // 00 / 11 corners mix, the off-diagonal corners scale
        constexpr int pi = CODE - TC_DEPOL;
        constexpr int J0 = pi < 3 ? 0 : pi < 5 ? 1 : 2;
        constexpr int J1 = pi == 0 ? 1 : pi == 1 ? 2 : pi == 2 ? 3 : pi == 3 ? 2 : 3;
        if constexpr (J1 < RB) {
            const double keep = c[0], swap = c[1], off = c[2];
#pragma unroll
            for (int i = 0; i < (1 << RB); ++i) {
                if (i & ((1 << J0) | (1 << J1))) continue;
                const int i01 = i | (1 << J0), i10 = i | (1 << J1), i11 = i01 | i10;
                const double2 d0 = s[i], d1 = s[i11];
                d[i] = make_double2(fma(swap, d1.x, keep * d0.x), fma(swap, d1.y, keep * d0.y));
                d[i11] = make_double2(fma(swap, d0.x, keep * d1.x), fma(swap, d0.y, keep * d1.y));
                d[i01] = make_double2(s[i01].x * off, s[i01].y * off);
                d[i10] = make_double2(s[i10].x * off, s[i10].y * off);
            }
        }
    } else if constexpr (CODE == TC_COLLAPSE) { // keep bit(q0) (and bit(q1)) == outcome, scaled
        const uint32_t flags = (h >> 6) & 15u;
        const uint32_t q0k = (h >> 11) & 3u, q1k = (h >> 19) & 3u, q1p = (h >> 21) & 63u;
        const uint32_t o = (h >> 10) & 1u;
        const bool two = flags & 1;
        const bool r0 = q0k == TL_REG, r1 = q1k == TL_REG;
        const uint32_t f0 = r0 ? 0u : fixed_bit_of(q0k, q0p, lane, w, gbase);
        const uint32_t f1 = r1 ? 0u : fixed_bit_of(q1k, q1p, lane, w, gbase);
        const double sc = c[0];
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            const uint32_t b0 = r0 ? (static_cast<uint32_t>(i) >> q0p) & 1u : f0;
            const uint32_t b1 = r1 ? (static_cast<uint32_t>(i) >> q1p) & 1u : f1;
            const bool keep = b0 == o && (!two || b1 == o);
            d[i] = make_double2(keep ? s[i].x * sc : 0.0, keep ? s[i].y * sc : 0.0);
        }
    } else {
        static_assert(CODE < 0, "unknown tile handler code");
    }
}

// The interpreter's dispatch: one jump table over the handler codes.
template <int RB>
__device__ __forceinline__ void step(const Regs<RB>& s, Regs<RB>& d, const OpCtx& x, uint32_t lane,
                                     uint32_t w, uint64_t gbase) {
    switch (static_cast<uint32_t>(x.h & 63u)) {
#define QGPU_CASE(K) \
    case K: step_c<RB, K>(s, d, x, lane, w, gbase); break;
#define QGPU_CASE8(K) QGPU_CASE(K) QGPU_CASE(K + 1) QGPU_CASE(K + 2) QGPU_CASE(K + 3) \
    QGPU_CASE(K + 4) QGPU_CASE(K + 5) QGPU_CASE(K + 6) QGPU_CASE(K + 7)
        QGPU_CASE8(0) QGPU_CASE8(8) QGPU_CASE8(16) QGPU_CASE8(24) QGPU_CASE8(32) QGPU_CASE8(40)
        QGPU_CASE(48) QGPU_CASE(49) QGPU_CASE(50) QGPU_CASE(51) QGPU_CASE(52) QGPU_CASE(53)
        QGPU_CASE(54) QGPU_CASE(55) QGPU_CASE(56)
#undef QGPU_CASE8
#undef QGPU_CASE
    default: __builtin_unreachable(); // the host emits TileCode values only
    }
}

// Global index of tile T's amplitude 0: T's bits deposited into the qubits
// outside the tile. Linear in T, so a table per byte of T (built once per
// launch) replaces the per-bit insertion loop.
template <int RB, int WB>
__device__ __forceinline__ uint64_t tile_gbase_slow(const TileParams& P, uint64_t T) {
    uint64_t gb = T << kLaneQubits;
#pragma unroll
    for (int j = 0; j < RB + WB; ++j) gb = insert_zero_bit(gb, P.high_sorted[j]); // ascending
    return gb;
}

// The interpreter: the phase body dispatches every op through one jump table
// (Prog::kInterp); a JIT program replaces it with straight-line code.
struct Interp {
    static constexpr bool kInterp = true;
};

template <int RB, int WB, int NBUF, class Prog>
__device__ __forceinline__ void tile_pass_body(double2* __restrict__ amps, const TileParams& P) {
    constexpr int R = 1 << RB;
    constexpr int K = kLaneQubits + RB + WB;
    extern __shared__ __align__(128) double2 smem[];
    __shared__ TileOp sops[kMaxTileOps + 1]; // + 1: the prefetch may read one past
    __shared__ uint64_t full[NBUF];
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t w = threadIdx.x >> 5;
    const int nph = P.num_phases;
    const bool any_outer = P.any_outer != 0;
    constexpr int kGbaseChunks = (36 - K + 7) / 8; // tile indices of <= 36 local qubits
    const uint64_t G = gridDim.x;
    const uint64_t ntiles = P.num_tiles > blockIdx.x ? (P.num_tiles - blockIdx.x + G - 1) / G : 0;

    __shared__ uint64_t gtab[kGbaseChunks][256];
    auto tile_gbase = [&](uint64_t T) {
        uint64_t g = 0;
#pragma unroll
        for (int k = 0; k < kGbaseChunks; ++k) g |= gtab[k][(T >> (8 * k)) & 255u];
        return g;
    };

    // Each warp owns 8 whole 512-byte segments of the tile in the last phase
    // (tile bits 0-4 are never warp bits, so a warp's amplitudes there are
    // the segments with its own warp bits: P.fin_seg[w]). It stores them and
    // refills their slots itself — lanes 0-7 one bulk copy each, lane 0
    // posting the warp's 4 KiB on the stage's tx-count mbarrier (16
    // arrivals per fill) — so no block barrier separates tiles.
    constexpr uint32_t SEG_BYTES = 32u * sizeof(double2);
    // runs of 2^fin_run segments are contiguous in HBM (and, by the host's
    // tile-bit order, in shared memory): lanes 0 .. (8 >> fin_run) - 1 move
    // one run each
    const int frun = P.fin_run;
    constexpr uint32_t SEGS = 1u << RB; // segments a warp owns in the last phase
    const uint32_t ncopy = SEGS >> frun;
    const uint32_t run_bytes = SEG_BYTES << frun;
    const uint32_t my_rseg = lane < ncopy ? P.fin_seg[w][lane << frun] : 0;
    const uint64_t my_goff = P.seg_off[my_rseg];
    const uint32_t my_soff = my_rseg << kLaneQubits;
    auto load_mine = [&](uint64_t t) {
        const int b = static_cast<int>(t % NBUF);
        const uint64_t gb = tile_gbase(blockIdx.x + t * G);
        double2* buf = smem + (static_cast<size_t>(b) << K);
        if (lane < ncopy) tma_load(buf + my_soff, amps + gb + my_goff, run_bytes, &full[b]);
        if (lane == 0) mbar_expect_tx(&full[b], SEGS * SEG_BYTES);
    };
    constexpr uint32_t kCopyLanes = SEGS; // one segment (run) per lane (a
    // lane-0 unrolled issue with uniform addresses measured 5 % slower)
    if (threadIdx.x == 0) {
        for (int b = 0; b < NBUF; ++b) mbar_init(&full[b], 1u << WB);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int k = threadIdx.x; k < kGbaseChunks * 256; k += blockDim.x)
        gtab[k >> 8][k & 255] = tile_gbase_slow<RB, WB>(P, static_cast<uint64_t>(k & 255) << (8 * (k >> 8)));
    __syncthreads();
    for (uint64_t t = 0; t < NBUF && t < ntiles; ++t) load_mine(t);
    const int nops = P.phases[nph - 1].op_end;
    const uint32_t sops_addr = smem_u32(sops);
    // this thread's HBM offset in the last phase (lane bits 0-2: qubits 0-2)
    const uint64_t fin_thread = P.fin_gwarp[w] + (lane & 7u) + ((lane >> 3) & 1u ? P.fin_glane[0] : 0) +
                                ((lane >> 4) & 1u ? P.fin_glane[1] : 0);
    {
        const uint64_t* src = reinterpret_cast<const uint64_t*>(P.ops);
        uint64_t* dst = reinterpret_cast<uint64_t*>(sops);
        constexpr int WORDS = sizeof(TileOp) / sizeof(uint64_t);
        for (int k = threadIdx.x; k < (kMaxTileOps + 1) * WORDS; k += blockDim.x)
            dst[k] = k < nops * WORDS ? src[k] : 0; // entry kMaxTileOps: the prefetch sentinel
    }
    __syncthreads();

    for (uint64_t t = 0; t < ntiles; ++t) {
        const int b = static_cast<int>(t % NBUF);
        double2* buf = smem + (static_cast<size_t>(b) << K);
        const uint64_t gb = tile_gbase(blockIdx.x + t * G);
        const uint64_t gbase = gb + P.global_offset;
        const uint64_t act = any_outer ? active_ops(sops, nops, gbase, lane) : ~uint64_t{0};
        mbar_wait(&full[b], static_cast<uint32_t>((t / NBUF) & 1));
        bool wrote = false, last_skipped = false; // (uniform per tile)
        if constexpr (Prog::kInterp) {
        int prev_ph = -1;                         // the last phase executed
        for (int ph = 0; ph < nph; ++ph) {
            const TilePhase& Q = P.phases[ph];
            const int end = Q.op_end;
            uint64_t m = act & ((uint64_t{1} << end) - 1) &
                         ~((uint64_t{1} << Q.op_begin) - 1);
            if (m == 0) { // no op runs: the tile stays as it is in shared memory
                last_skipped = ph == nph - 1;
                continue;
            }
            // end < 64 always: kMaxTileOps entries plus the sentinel
            if (wrote) { // the previous phase's writes are in (within the group)
                // group barriers hold for the transition ph - 1 -> ph only; if
                // outer controls skipped phase ph - 1 on this tile, the data
                // comes from an earlier layout: sync the whole CTA
                const int c = prev_ph == ph - 1 ? Q.sync_bits : 0;
                if (c == 0)
                    __syncthreads();
                else if (c >= WB)
                    __syncwarp();
                else
                    asm volatile("bar.sync %0, %1;" ::"r"(Q.bar_base + (w >> (WB - c))), "r"(32 << (WB - c))
                                 : "memory");
            }
            wrote = true;
            prev_ph = ph;
            if constexpr (Prog::kInterp) {
                const uint32_t wofs = Q.warp_off[w] + (lane & 7u) + ((lane >> 3) & 1u ? Q.lane_off[0] : 0u) +
                                      ((lane >> 4) & 1u ? Q.lane_off[1] : 0u);
                double2 a[R], b[R];
#pragma unroll
                for (int i = 0; i < R; ++i) a[i] = lds16(buf + wofs + Q.reg_off[i]);
                bool in_a = true; // the phase's result is in a (else b)
                // ops alternate a -> b, b -> a; the contexts alternate too,
                // each loaded one op ahead. `runm` has a bit per op that runs
                // on this tile, plus a stop bit at the phase end (sops[end] is
                // a valid entry: the next phase's first op or the sentinel).
                const uint64_t runm = m | (uint64_t{1} << end);
                // next op at or after `from`: one bit scan
                auto next = [&](int from) { return lowest(runm & (~uint64_t{0} << from)); };
                int o = next(Q.op_begin);
                OpCtx ca, cb;
                load_ctx(ca, sops_addr, o);
                for (;;) {
                    const int on = next(o + 1);
                    load_ctx(cb, sops_addr, on);
                    step<RB>(a, b, ca, lane, w, gbase);
                    if (on >= end) {
                        in_a = false;
                        break;
                    }
                    o = next(on + 1);
                    load_ctx(ca, sops_addr, o);
                    step<RB>(b, a, cb, lane, w, gbase);
                    if (o >= end) break;
                }
                if (ph == nph - 1) { // the last phase stores straight to HBM
                    double2* out = amps + gb + fin_thread;
                    if (in_a) {
#pragma unroll
                        for (int i = 0; i < R; ++i) __stcs(out + P.fin_greg[i], a[i]);
                    } else {
#pragma unroll
                        for (int i = 0; i < R; ++i) __stcs(out + P.fin_greg[i], b[i]);
                    }
                } else if (in_a) {
#pragma unroll
                    for (int i = 0; i < R; ++i) sts16(buf + wofs + Q.reg_off[i], a[i]);
                } else {
#pragma unroll
                    for (int i = 0; i < R; ++i) sts16(buf + wofs + Q.reg_off[i], b[i]);
                }
            }
        }
        } else {
            // a generated program (tile_jit.cpp): the whole phase sequence
            // straight-line, with literal op masks, layouts, barriers and ops
            Prog::template tile<RB, WB>(act, buf, amps + gb + fin_thread, P, lane, w, gbase, sops_addr, wrote,
                                        last_skipped);
        }
        // The last phase stored its results to HBM. If outer controls skipped
        // it after an earlier phase wrote (rare), the tile's final values are
        // in shared memory, written by any warp: sync, then each warp moves
        // its own last-phase positions. If no phase ran, HBM already holds
        // the tile.
        if (last_skipped && wrote) {
            __syncthreads();
            const TilePhase& Q = P.phases[nph - 1];
            const uint32_t wofs = Q.warp_off[w] + (lane & 7u) + ((lane >> 3) & 1u ? Q.lane_off[0] : 0u) +
                                  ((lane >> 4) & 1u ? Q.lane_off[1] : 0u);
            double2* out = amps + gb + fin_thread;
#pragma unroll
            for (int i = 0; i < R; ++i) __stcs(out + P.fin_greg[i], buf[wofs + Q.reg_off[i]]);
        }
        // Every access to this warp's last-phase positions happened before
        // its last phase (the data-flow barriers order them), and the stores
        // read registers: the warp refills its slots of this stage with tile
        // t + NBUF at once.
        if (t + NBUF < ntiles) {
            // every lane's reads of the slots were consumed (the values went
            // into the ops and stores): a warp sync suffices before the async
            // refill, as in a TMA consumer release. (A proxy fence here
            // compiled to MEMBAR.ALL.CTA, waiting for the HBM stores: 11 % of
            // the stall samples.)
#ifdef QGPU_REFILL_FENCE
            fence_proxy_async();
#endif
            __syncwarp();
            load_mine(t + NBUF);
        }
    }
}

} // namespace

} // namespace qgpu
