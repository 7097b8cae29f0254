// tile_pass.cu — the hot kernel: one HBM read + write of the state applies a
// whole run of queued ops (gates, dephasing, collapse), in order.
//
// Structure (qgpu_device.h: TileParams / TilePhase / TileOp):
//  * one persistent CTA per SM walks tiles of 2^12 amplitudes (qubits 0-4 plus
//    7 higher qubits chosen per pass);
//  * HBM <-> shared memory through TMA: warp 0 issues cp.async.bulk loads of
//    tile t+1 (completion on an mbarrier) and bulk stores of tile t, three
//    64 KiB stages deep, so the streaming overlaps the ops on the current tile
//    and no register holds data in flight;
//  * the ops run in phases: every thread holds 16 amplitudes in registers
//    spanning the phase's 4 register qubits (lanes span qubits 0-4, the 8
//    warps the remaining 3 tile qubits). Pair ops on register qubits stay in
//    registers, on lane qubits they use warp shuffles, diagonal gates and
//    channels are elementwise anywhere; between phases the tile is re-laid out
//    through shared memory.
//
// Register discipline: each op reads one register array and writes every
// element of the other (the op loop alternates A -> B, B -> A). Updating one
// array in place made ptxas copy the whole 64-register tile on every op
// (ncu: IMAD.MOV = 45% of issued instructions); with disjoint source and
// destination each result is computed straight into its final register.
#include "pair_math.cuh"
#include "qgpu_kernels.h"
#include "runtime.h"

#include <cstdio>
#include <cuda_runtime.h>

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

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- handlers
//
// Every handler reads `s` and writes all of `d`. SEL variants apply a
// per-element predicate (controls on register bits `rcm`, or on lane bits via
// `tok`); the common, uncontrolled variants have none.

__device__ __forceinline__ double2 diag_a(const double* c, double2 v) {
    return make_double2(fma(c[0], v.x, -(c[1] * v.y)), fma(c[0], v.y, c[1] * v.x));
}
__device__ __forceinline__ double2 diag_d(const double* c, double2 v) {
    return make_double2(fma(-c[7], v.y, c[6] * v.x), fma(c[7], v.x, c[6] * v.y));
}

template <int RB>
__device__ __forceinline__ void h_copy(const Regs<RB>& s, Regs<RB>& d) {
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) d[i] = s[i];
}

// 2x2 gate on register bit J (compile time): lo = i with bit J clear.
template <int RB, int J, int CLS, bool SEL>
__device__ __forceinline__ void h_reg_pair(const Regs<RB>& s, Regs<RB>& d, const double* c,
                                           uint32_t rcm, bool tok) {
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) {
        constexpr int bit = 1 << J;
        const int lo = i & ~bit, hi = i | bit;
        double2 r;
        if constexpr (CLS == CLS_SWAP)
            r = s[i ^ bit];
        else if (i & bit)
            r = row<ClassZ<CLS>::z1>(c[4], c[5], c[6], c[7], s[lo], s[hi]);
        else
            r = row<ClassZ<CLS>::z0>(c[0], c[1], c[2], c[3], s[lo], s[hi]);
        if constexpr (SEL) {
            const bool on = tok && (static_cast<uint32_t>(lo) & rcm) == rcm;
            d[i] = on ? r : s[i];
        } else {
            d[i] = r;
        }
    }
}

// In-place form of h_reg_pair (one array): pair by pair, both outputs are
// computed before either input is overwritten.
template <int RB, int J, int CLS, bool SEL>
__device__ __forceinline__ void h_reg_pair_ip(Regs<RB>& v, const double* c, uint32_t rcm, bool tok) {
    if constexpr (J < RB) {
#pragma unroll
        for (int lo = 0; lo < (1 << RB); ++lo) {
            constexpr int bit = 1 << J;
            if (lo & bit) continue;
            double2 l = v[lo], h = v[lo | bit];
            pair_update<CLS>(l, h, c);
            if constexpr (SEL) {
                const bool on = tok && (static_cast<uint32_t>(lo) & rcm) == rcm;
                v[lo] = on ? l : v[lo];
                v[lo | bit] = on ? h : v[lo | bit];
            } else {
                v[lo] = l;
                v[lo | bit] = h;
            }
        }
    }
}

// 2x2 gate on lane bit b: the partner amplitude comes from lane ^ 2^b, and
// each lane computes its own half (distributed.cpp:183-184:
// own_lo ? lo_out(mine, theirs) : hi_out(theirs, mine)).
template <int RB, int CLS, bool SEL>
__device__ __forceinline__ void h_lane_pair(const Regs<RB>& s, Regs<RB>& d, const double* c, uint32_t b,
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
        if constexpr (SEL) {
            const bool on = tok && (static_cast<uint32_t>(i) & rcm) == rcm;
            d[i] = on ? r : s[i];
        } else {
            d[i] = r;
        }
    }
}

// Diagonal gate with its target on register bit J: a * v where the bit is 0,
// d * v where it is 1 (rounding of the reference's low / high row). A side
// whose coefficient is exactly 1 keeps its input (flags).
template <int RB, int J>
__device__ __forceinline__ void h_diag_reg(const Regs<RB>& s, Regs<RB>& d, const double* c, uint32_t rcm,
                                           bool tok, bool a_one, bool d_one) {
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) {
        const bool bit = (i >> J) & 1;
        const double2 r = bit ? diag_d(c, s[i]) : diag_a(c, s[i]);
        const bool on = tok && !(bit ? d_one : a_one) && (static_cast<uint32_t>(i) & rcm) == rcm;
        d[i] = on ? r : s[i];
    }
}

// Diagonal gate whose target bit is fixed for this thread (lane, warp or
// outer qubit): coefficients picked once; per element the operands swap:
//   re = fma(P, X, Q * Y), im = fma(R, Y, S * X)
//   bit 0: P = a_re, Q = -a_im, R = a_re, S = a_im, (X, Y) = (x, y)
//   bit 1: P = -d_im, Q = d_re, R = d_im, S = d_re, (X, Y) = (y, x)
template <int RB>
__device__ __forceinline__ void h_diag_fixed(const Regs<RB>& s, Regs<RB>& d, const double* c,
                                             uint32_t bit, uint32_t rcm, bool tok, bool a_one,
                                             bool d_one) {
    const double P = bit ? -c[7] : c[0], Q = bit ? c[6] : -c[1];
    const double R = bit ? c[7] : c[0], S = bit ? c[6] : c[1];
    const bool doit = tok && !(bit ? d_one : a_one);
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) {
        const double X = bit ? s[i].y : s[i].x, Y = bit ? s[i].x : s[i].y;
        const double2 r = make_double2(fma(P, X, Q * Y), fma(R, Y, S * X));
        const bool on = doit && (static_cast<uint32_t>(i) & rcm) == rcm;
        d[i] = on ? r : s[i];
    }
}

__device__ __forceinline__ uint32_t fixed_bit_of(uint32_t kind, uint32_t pos, uint32_t lane, uint32_t w,
                                                 uint64_t gbase) {
    return kind == TL_LANE   ? (lane >> pos) & 1u
           : kind == TL_WARP ? (w >> pos) & 1u
                             : static_cast<uint32_t>((gbase >> pos) & 1u);
}

// One op: s -> d. `h` is the op's header, loaded by the caller one op ahead
// so its constant-bank latency hides behind the previous op; its low 6 bits
// are the handler code the host resolved (qgpu_device.h: TileCode), so
// dispatch is a single jump table.
template <int RB, bool IP, int J, int CLS, bool SEL>
__device__ __forceinline__ void reg_op(const Regs<RB>& s, Regs<RB>& d, const double* c, uint32_t rcm,
                                       bool tok) {
    if constexpr (J < RB) {
        if constexpr (IP)
            h_reg_pair_ip<RB, J, CLS, SEL>(d, c, rcm, tok);
        else
            h_reg_pair<RB, J, CLS, SEL>(s, d, c, rcm, tok);
    }
}

// IP (in place): s and d are the same array; every handler but the register
// pairs is elementwise (reads element i before writing it), so only those
// switch to their pairwise in-place form.
template <int RB, bool IP>
__device__ __forceinline__ void step(const Regs<RB>& s, Regs<RB>& d, uint64_t h, const TileOp& op,
                                     uint32_t lane, uint32_t w, uint64_t gbase) {
    static_assert(RB <= 4, "register-bit dispatch is written for up to 4 register qubits");
    const uint32_t code = h & 63u, flags = (h >> 6) & 15u;
    const uint32_t q0k = (h >> 11) & 3u, q0p = (h >> 13) & 63u;
    const uint32_t lane_cm = (h >> 27) & 31u, rcm = (h >> 32) & 15u, warp_cm = (h >> 36) & 15u;
    const uint64_t ocm = op.outer_cmask;
    // Controls fold into one per-thread predicate. (A separate early-out that
    // copied s to d for a failing warp made ptxas hoist that whole-tile copy
    // above the branch, i.e. onto every op.)
    const bool tok = (lane & lane_cm) == lane_cm && (w & warp_cm) == warp_cm && (gbase & ocm) == ocm;
    const bool a_one = flags & DF_A_ONE, d_one = flags & DF_D_ONE;
    const double* c = op.m; // coefficients are read from the constant bank where used
    switch (code) {
    case TC_REG + 0: reg_op<RB, IP,0, CLS_GENERIC, false>(s, d, c, 0, true); break;
    case TC_REG + 1: reg_op<RB, IP,1, CLS_GENERIC, false>(s, d, c, 0, true); break;
    case TC_REG + 2: reg_op<RB, IP,2, CLS_GENERIC, false>(s, d, c, 0, true); break;
    case TC_REG + 3: reg_op<RB, IP,3, CLS_GENERIC, false>(s, d, c, 0, true); break;
    case TC_REG + 4: reg_op<RB, IP,0, CLS_REAL, false>(s, d, c, 0, true); break;
    case TC_REG + 5: reg_op<RB, IP,1, CLS_REAL, false>(s, d, c, 0, true); break;
    case TC_REG + 6: reg_op<RB, IP,2, CLS_REAL, false>(s, d, c, 0, true); break;
    case TC_REG + 7: reg_op<RB, IP,3, CLS_REAL, false>(s, d, c, 0, true); break;
    case TC_REG + 8: reg_op<RB, IP,0, CLS_RX, false>(s, d, c, 0, true); break;
    case TC_REG + 9: reg_op<RB, IP,1, CLS_RX, false>(s, d, c, 0, true); break;
    case TC_REG + 10: reg_op<RB, IP,2, CLS_RX, false>(s, d, c, 0, true); break;
    case TC_REG + 11: reg_op<RB, IP,3, CLS_RX, false>(s, d, c, 0, true); break;
    case TC_REG + 12: reg_op<RB, IP,0, CLS_SWAP, false>(s, d, c, 0, true); break;
    case TC_REG + 13: reg_op<RB, IP,1, CLS_SWAP, false>(s, d, c, 0, true); break;
    case TC_REG + 14: reg_op<RB, IP,2, CLS_SWAP, false>(s, d, c, 0, true); break;
    case TC_REG + 15: reg_op<RB, IP,3, CLS_SWAP, false>(s, d, c, 0, true); break;
    case TC_REG_SEL + 0: reg_op<RB, IP,0, CLS_GENERIC, true>(s, d, c, rcm, tok); break;
    case TC_REG_SEL + 1: reg_op<RB, IP,1, CLS_GENERIC, true>(s, d, c, rcm, tok); break;
    case TC_REG_SEL + 2: reg_op<RB, IP,2, CLS_GENERIC, true>(s, d, c, rcm, tok); break;
    case TC_REG_SEL + 3: reg_op<RB, IP,3, CLS_GENERIC, true>(s, d, c, rcm, tok); break;
    case TC_REG_SEL + 4: reg_op<RB, IP,0, CLS_SWAP, true>(s, d, c, rcm, tok); break;
    case TC_REG_SEL + 5: reg_op<RB, IP,1, CLS_SWAP, true>(s, d, c, rcm, tok); break;
    case TC_REG_SEL + 6: reg_op<RB, IP,2, CLS_SWAP, true>(s, d, c, rcm, tok); break;
    case TC_REG_SEL + 7: reg_op<RB, IP,3, CLS_SWAP, true>(s, d, c, rcm, tok); break;
    case TC_LANE_GENERIC: h_lane_pair<RB, CLS_GENERIC, false>(s, d, c, q0p, 0, true, lane); break;
    case TC_LANE_REAL: h_lane_pair<RB, CLS_REAL, false>(s, d, c, q0p, 0, true, lane); break;
    case TC_LANE_SWAP: h_lane_pair<RB, CLS_SWAP, false>(s, d, c, q0p, 0, true, lane); break;
    case TC_LANE_SEL_GENERIC: h_lane_pair<RB, CLS_GENERIC, true>(s, d, c, q0p, rcm, tok, lane); break;
    case TC_LANE_SEL_SWAP: h_lane_pair<RB, CLS_SWAP, true>(s, d, c, q0p, rcm, tok, lane); break;
    case TC_DIAG_REG + 0: h_diag_reg<RB, 0>(s, d, c, rcm, tok, a_one, d_one); break;
    case TC_DIAG_REG + 1: h_diag_reg<RB, 1>(s, d, c, rcm, tok, a_one, d_one); break;
    case TC_DIAG_REG + 2: h_diag_reg<RB, 2>(s, d, c, rcm, tok, a_one, d_one); break;
    case TC_DIAG_REG + 3: h_diag_reg<RB, 3>(s, d, c, rcm, tok, a_one, d_one); break;
    case TC_DIAG_FIXED:
        h_diag_fixed<RB>(s, d, c, fixed_bit_of(q0k, q0p, lane, w, gbase), rcm, tok, a_one, d_one);
        break;
    case TC_DEPHASE: { // density.cpp:56-59: scale where bit(q0) != bit(q1)
        const uint32_t q1k = (h >> 19) & 3u, q1p = (h >> 21) & 63u;
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
        break;
    }
    default: { // PO_COLLAPSE: keep bit(q0) (and bit(q1)) == outcome, scaled
        const uint32_t q1k = (h >> 19) & 3u, q1p = (h >> 21) & 63u;
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
        break;
    }
    }
}

template <int RB, int WB>
__device__ __forceinline__ uint64_t tile_gbase(const TileParams& P, uint64_t T) {
    uint64_t gb = T << kLaneQubits;
#pragma unroll
    for (int j = 0; j < RB + WB; ++j) gb = insert_zero_bit(gb, P.high_pos[j]);
    return gb;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Named barrier among the consumer warps only (the producer never joins).
template <int NTHREADS>
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(NTHREADS) : "memory");
}

// Warp-specialised: warps 0 .. 2^WB - 1 apply the ops, the last warp is the
// TMA producer. full[b]: stage b holds a loaded tile (tx-count barrier).
// done[b]: the consumers have written stage b's last phase (one arrival per
// consumer warp); the producer then bulk-stores it and, once the store has
// read the stage, refills it with the tile NBUF ahead.
template <int RB, int WB, int NBUF, bool INPLACE>
__global__ void __launch_bounds__((32 << WB) + 32, 1) // 9 warps: <= 168 registers
k_tile_pass(double2* __restrict__ amps, const __grid_constant__ TileParams P) {
    constexpr int R = 1 << RB;
    constexpr int K = kLaneQubits + RB + WB;
    constexpr int NSEG = 1 << (RB + WB);
    constexpr int NCW = 1 << WB; // consumer warps
    constexpr uint32_t TILE_BYTES = sizeof(double2) << K;
    extern __shared__ __align__(128) double2 smem[];
    __shared__ uint64_t full[NBUF], done[NBUF];
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t w = threadIdx.x >> 5;
    const int nph = P.num_phases;
    const uint64_t G = gridDim.x;
    const uint64_t ntiles = P.num_tiles > blockIdx.x ? (P.num_tiles - blockIdx.x + G - 1) / G : 0;

    if (threadIdx.x == 0) {
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&done[b], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (w == NCW) { // ---------------------------------------------- producer
        // runs of 2^seg_run segments are contiguous in HBM: one bulk copy each
        const int run = P.seg_run;
        auto copies = [&](uint64_t t, bool load) {
            const int b = static_cast<int>(t % NBUF);
            const uint64_t gb = tile_gbase<RB, WB>(P, blockIdx.x + t * G);
            double2* buf = smem + (static_cast<size_t>(b) << K);
            for (int sg = lane << run; sg < NSEG; sg += 32 << run) {
                if (load)
                    tma_load(buf + (sg << kLaneQubits), amps + gb + P.seg_off[sg],
                             (32u * sizeof(double2)) << run, &full[b]);
                else
                    tma_store(amps + gb + P.seg_off[sg], buf + (sg << kLaneQubits),
                              (32u * sizeof(double2)) << run);
            }
        };
        auto store = [&](uint64_t t) {
            mbar_wait(&done[t % NBUF], static_cast<uint32_t>((t / NBUF) & 1));
            copies(t, false);
            tma_commit();
        };
        for (uint64_t t = 0; t < ntiles; ++t) {
            if (t >= NBUF) { // stage t % NBUF still holds tile t - NBUF
                store(t - NBUF);
                tma_wait_read<0>();
                __syncwarp();
            }
            if (lane == 0) mbar_expect_tx(&full[t % NBUF], TILE_BYTES);
            __syncwarp();
            copies(t, true);
        }
        for (uint64_t t = ntiles > NBUF ? ntiles - NBUF : 0; t < ntiles; ++t) store(t);
        tma_wait_all();
        return;
    }

    // ------------------------------------------------------------ consumers
    for (uint64_t t = 0; t < ntiles; ++t) {
        const int b = static_cast<int>(t % NBUF);
        double2* buf = smem + (static_cast<size_t>(b) << K);
        const uint64_t gbase = tile_gbase<RB, WB>(P, blockIdx.x + t * G) + P.global_offset;
        mbar_wait(&full[b], static_cast<uint32_t>((t / NBUF) & 1));
        for (int ph = 0; ph < nph; ++ph) {
            if (ph > 0) consumer_sync<32 * NCW>(); // previous phase's writes are in
            const TilePhase& Q = P.phases[ph];
            const uint32_t wofs = Q.warp_off[w] + lane;
            const int end = Q.op_end;
            int o = Q.op_begin;
            uint64_t h = o < end ? P.ops[o].hdr : 0; // headers are read one op ahead
            if constexpr (INPLACE) {
                double2 A[R];
#pragma unroll
                for (int i = 0; i < R; ++i) A[i] = buf[wofs + Q.reg_off[i]];
                for (; o < end; ++o) {
                    const uint64_t hn = o + 1 < end ? P.ops[o + 1].hdr : 0;
                    step<RB, true>(A, A, h, P.ops[o], lane, w, gbase);
                    h = hn;
                }
#pragma unroll
                for (int i = 0; i < R; ++i) buf[wofs + Q.reg_off[i]] = A[i];
            } else {
                double2 A[R], B[R];
#pragma unroll
                for (int i = 0; i < R; ++i) A[i] = buf[wofs + Q.reg_off[i]];
                for (; o + 1 < end; o += 2) {
                    const uint64_t h1 = P.ops[o + 1].hdr;
                    step<RB, false>(A, B, h, P.ops[o], lane, w, gbase);
                    h = o + 2 < end ? P.ops[o + 2].hdr : 0;
                    step<RB, false>(B, A, h1, P.ops[o + 1], lane, w, gbase);
                }
                if (o < end) {
                    step<RB, false>(A, B, h, P.ops[o], lane, w, gbase);
#pragma unroll
                    for (int i = 0; i < R; ++i) buf[wofs + Q.reg_off[i]] = B[i];
                } else {
#pragma unroll
                    for (int i = 0; i < R; ++i) buf[wofs + Q.reg_off[i]] = A[i];
                }
            }
        }
        fence_proxy_async(); // generic-proxy writes -> visible to the bulk store
        __syncwarp();
        if (lane == 0) mbar_arrive(&done[b]);
    }
}

} // namespace

void launch_tile_pass(double2* amps, const TileParams& p, cudaStream_t s) {
    constexpr int NBUF = 3;
#ifndef QGPU_TILE_INPLACE
#define QGPU_TILE_INPLACE 0
#endif
    auto kern = k_tile_pass<kPhaseRegBits, kTileWarpBits, NBUF, QGPU_TILE_INPLACE != 0>;
    constexpr size_t smem = NBUF * (sizeof(double2) << kTileQubits);
    static bool set = false;
    if (!set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        set = true;
    }
    uint64_t blocks = p.num_tiles;
    if (blocks > 148) blocks = 148; // persistent: one CTA per SM
    kern<<<static_cast<unsigned>(blocks), kTileThreads + 32, smem, s>>>(amps, p);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kern);
        char msg[256];
        snprintf(msg, sizeof msg,
                 "tile pass launch: %s (regs %d, max threads %d, static smem %zu, dyn smem %zu)",
                 cudaGetErrorString(e), fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes,
                 smem);
        throw DeviceError(msg);
    }
    count_launch();
}

} // namespace qgpu
