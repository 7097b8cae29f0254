// kernels.cu — hand-written sm_100a kernels for the state-vector /
// density-matrix gate path. FP64, HBM-bandwidth bound: no tensor cores.
//
// Arithmetic parity: every pair update evaluates exactly the fma chain the
// reference's pair_lo_out / pair_hi_out compile to
// (/root/reference/proj/include/qsim/detail/pair_math.hpp:30-45, contracted by
// GCC as read from the reference objects; restated in oracle/qsim_oracle.c):
//   re = fma(-q3, y1, fma(q2, x1, fma(q0, x0, -(q1 * y0))))
//   im = fma( q3, x1, fma(q2, y1, fma(q0, y0,   q1 * x0)))
// with (q0..q3) = (a_re, a_im, b_re, b_im) for the low output and
// (c_re, c_im, d_re, d_im) for the high one, (x0,y0) = lo, (x1,y1) = hi.
// Terms with an exactly-zero coefficient are dropped at compile time per gate
// class (value-identical: such an fma only adds a signed zero). The result is
// bit-identical to the reference on every amplitude (tests/test_gpu_parity.py).
#include "qgpu_kernels.h"

#include <atomic>
#include <cuda_runtime.h>

namespace qgpu {

namespace {

std::atomic<uint64_t> g_launches{0};

inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

__device__ __forceinline__ uint64_t insert_zero_bit(uint64_t x, int pos) {
    const uint64_t low = x & ((uint64_t{1} << pos) - 1);
    return ((x >> pos) << (pos + 1)) | low;
}

// pair_math.hpp:56-61
__device__ __forceinline__ uint64_t pair_base_index(uint64_t i, int t) {
    const uint64_t low_mask = (uint64_t{1} << t) - 1;
    return ((i & ~low_mask) << 1) | (i & low_mask);
}

// One output row of the pair update; Z = coefficients known to be zero
// (bit0 q0, bit1 q1, bit2 q2, bit3 q3).
template <int Z>
__device__ __forceinline__ double2 row(double q0, double q1, double q2, double q3,
                                       double2 lo, double2 hi) {
    constexpr bool n0 = !(Z & 1), n1 = !(Z & 2), n2 = !(Z & 4), n3 = !(Z & 8);
    double re, im;
    if constexpr (n0 && n1) {
        re = fma(q0, lo.x, -(q1 * lo.y));
        im = fma(q0, lo.y, q1 * lo.x);
    } else if constexpr (n0) {
        re = q0 * lo.x;
        im = q0 * lo.y;
    } else if constexpr (n1) {
        re = -(q1 * lo.y);
        im = q1 * lo.x;
    } else {
        re = 0.0;
        im = 0.0;
    }
    if constexpr (n2) {
        re = fma(q2, hi.x, re);
        im = fma(q2, hi.y, im);
    }
    if constexpr (n3) {
        re = fma(-q3, hi.y, re);
        im = fma(q3, hi.x, im);
    }
    return make_double2(re, im);
}

// Zero patterns of the two rows per class (see GateClass in qgpu_device.h).
template <int CLS> struct ClassZ;
template <> struct ClassZ<CLS_GENERIC> { static constexpr int z0 = 0, z1 = 0; };
template <> struct ClassZ<CLS_REAL> { static constexpr int z0 = 0b1010, z1 = 0b1010; };
template <> struct ClassZ<CLS_RX> { static constexpr int z0 = 0b0110, z1 = 0b1001; };

template <int CLS>
__device__ __forceinline__ void pair_update(double2& lo, double2& hi, const double* m) {
    if constexpr (CLS == CLS_SWAP) {
        const double2 t = lo;
        lo = hi;
        hi = t;
    } else {
        const double2 l = lo, h = hi;
        lo = row<ClassZ<CLS>::z0>(m[0], m[1], m[2], m[3], l, h);
        hi = row<ClassZ<CLS>::z1>(m[4], m[5], m[6], m[7], l, h);
    }
}

// Diagonal gate on one amplitude whose target bit is b: a * v (b = 0) or
// d * v (b = 1), each with the rounding of its reference row (the a term is
// the fused first product of the low row; the d term is the second product of
// the high row, so it rounds the other way round).
__device__ __forceinline__ double2 diag_mul(const double* m, uint32_t b, double2 v) {
    const double ar = m[0], ai = m[1], dr = m[6], di = m[7];
    const double s1 = b ? -di : ar, t1 = b ? v.y : v.x;
    const double s2 = b ? dr : -ai, t2 = b ? v.x : v.y;
    const double u1 = b ? di : ar, w1 = b ? v.x : v.y;
    const double u2 = b ? dr : ai, w2 = b ? v.y : v.x;
    return make_double2(fma(s1, t1, s2 * t2), fma(u1, w1, u2 * w2));
}

// ------------------------------------------------------------ fused pass

template <int H>
using RegTile = double2[1 << H];

template <int H, int J, int CLS>
__device__ __forceinline__ void reg_pair(RegTile<H>& v, const PassOp& op, bool tok) {
    const uint32_t rcm = op.reg_cmask;
#pragma unroll
    for (int i = 0; i < (1 << H); ++i) {
        if (i & (1 << J)) continue;
        if (tok && (static_cast<uint32_t>(i) & rcm) == rcm)
            pair_update<CLS>(v[i], v[i | (1 << J)], op.m);
    }
}

template <int H, int CLS>
__device__ __forceinline__ void reg_pair_dispatch(RegTile<H>& v, const PassOp& op, bool tok) {
    switch (op.q0.pos) {
    case 0: if constexpr (H > 0) reg_pair<H, 0, CLS>(v, op, tok); break;
    case 1: if constexpr (H > 1) reg_pair<H, 1, CLS>(v, op, tok); break;
    case 2: if constexpr (H > 2) reg_pair<H, 2, CLS>(v, op, tok); break;
    case 3: if constexpr (H > 3) reg_pair<H, 3, CLS>(v, op, tok); break;
    case 4: if constexpr (H > 4) reg_pair<H, 4, CLS>(v, op, tok); break;
    default: break;
    }
}

template <int H>
__device__ __forceinline__ void lane_pair(RegTile<H>& v, const PassOp& op, bool tok,
                                          uint32_t lane) {
    const uint32_t bitmask = 1u << op.q0.pos;
    const bool own_lo = (lane & bitmask) == 0;
    const uint32_t rcm = op.reg_cmask;
    const double* m = op.m;
    // Row coefficients of the half this lane owns (distributed.cpp:183-184:
    // own_lo ? lo_out(mine, theirs) : hi_out(theirs, mine)).
    const double q0 = own_lo ? m[0] : m[4], q1 = own_lo ? m[1] : m[5];
    const double q2 = own_lo ? m[2] : m[6], q3 = own_lo ? m[3] : m[7];
#pragma unroll
    for (int i = 0; i < (1 << H); ++i) {
        double2 theirs;
        theirs.x = __shfl_xor_sync(0xffffffffu, v[i].x, bitmask);
        theirs.y = __shfl_xor_sync(0xffffffffu, v[i].y, bitmask);
        if (!(tok && (static_cast<uint32_t>(i) & rcm) == rcm)) continue;
        const double2 lo = own_lo ? v[i] : theirs;
        const double2 hi = own_lo ? theirs : v[i];
        switch (op.cls) {
        case CLS_SWAP: v[i] = theirs; break;
        case CLS_REAL: v[i] = row<0b1010>(q0, q1, q2, q3, lo, hi); break;
        default: v[i] = row<0>(q0, q1, q2, q3, lo, hi); break; // GENERIC, RX
        }
    }
}

__device__ __forceinline__ uint32_t fixed_bit(QubitLoc q, uint32_t lane, uint64_t gbase) {
    return q.kind == LOC_LANE ? (lane >> q.pos) & 1u
                              : static_cast<uint32_t>((gbase >> q.pos) & 1u);
}

template <int H>
__device__ __forceinline__ void elementwise(RegTile<H>& v, const PassOp& op, bool tok,
                                            uint32_t lane, uint64_t gbase) {
    const uint32_t rcm = op.reg_cmask;
    const bool reg0 = op.q0.kind == LOC_REG, reg1 = op.q1.kind == LOC_REG;
    const uint32_t f0 = fixed_bit(op.q0, lane, gbase);
    const uint32_t f1 = fixed_bit(op.q1, lane, gbase);
#pragma unroll
    for (int i = 0; i < (1 << H); ++i) {
        if (!(tok && (static_cast<uint32_t>(i) & rcm) == rcm)) continue;
        const uint32_t b0 = reg0 ? (static_cast<uint32_t>(i) >> op.q0.pos) & 1u : f0;
        const uint32_t b1 = reg1 ? (static_cast<uint32_t>(i) >> op.q1.pos) & 1u : f1;
        switch (op.kind) {
        case PO_DIAG:
            if (!((b0 == 0 && (op.flags & DF_A_ONE)) || (b0 == 1 && (op.flags & DF_D_ONE))))
                v[i] = diag_mul(op.m, b0, v[i]);
            break;
        case PO_DEPHASE: // density.cpp:56-59
            if (b0 != b1) {
                v[i].x *= op.m[0];
                v[i].y *= op.m[0];
            }
            break;
        case PO_COLLAPSE: {
            const bool keep = b0 == op.outcome && (!(op.flags & 1) || b1 == op.outcome);
            if (keep) {
                v[i].x *= op.m[0];
                v[i].y *= op.m[0];
            } else {
                v[i] = make_double2(0.0, 0.0);
            }
            break;
        }
        default: break;
        }
    }
}

template <int H>
__global__ void __launch_bounds__(256)
k_fused_pass(double2* __restrict__ amps, const __grid_constant__ PassParams P) {
    constexpr int R = 1 << H;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp0 = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t T = warp0; T < P.num_tiles; T += nwarps) {
        uint64_t b = T << kLaneQubits;
#pragma unroll
        for (int j = 0; j < H; ++j) b = insert_zero_bit(b, P.reg_pos[j]);
        double2 v[R];
#pragma unroll
        for (int i = 0; i < R; ++i) v[i] = __ldcs(amps + b + P.reg_off[i] + lane);
        const uint64_t gbase = b + P.global_offset;
        for (int o = 0; o < P.num_ops; ++o) {
            const PassOp& op = P.ops[o];
            const bool tok = (lane & op.lane_cmask) == op.lane_cmask &&
                             (gbase & op.outer_cmask) == op.outer_cmask;
            switch (op.kind) {
            case PO_PAIR_REG:
                switch (op.cls) {
                case CLS_REAL: reg_pair_dispatch<H, CLS_REAL>(v, op, tok); break;
                case CLS_RX: reg_pair_dispatch<H, CLS_RX>(v, op, tok); break;
                case CLS_SWAP: reg_pair_dispatch<H, CLS_SWAP>(v, op, tok); break;
                default: reg_pair_dispatch<H, CLS_GENERIC>(v, op, tok); break;
                }
                break;
            case PO_PAIR_LANE:
                lane_pair<H>(v, op, tok, lane);
                break;
            default:
                elementwise<H>(v, op, tok, lane, gbase);
                break;
            }
        }
#pragma unroll
        for (int i = 0; i < R; ++i) __stcs(amps + b + P.reg_off[i] + lane, v[i]);
    }
}

// ---------------------------------------------------------------- tile pass
//
// One CTA per 2^12-amplitude tile (qgpu_device.h: TileParams). The op loop
// is warp-uniform: every branch below depends only on the op (or on a
// compile-time register index), never on the lane, except the final selects
// that apply lane/warp/outer controls.

template <int RB>
using Regs = double2[1 << RB];

template <int RB, int J, int CLS>
__device__ __forceinline__ void tile_reg_pair(Regs<RB>& v, const double* c, uint32_t rcm, bool tok) {
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) {
        if (i & (1 << J)) continue;
        if ((static_cast<uint32_t>(i) & rcm) != rcm) continue; // uniform
        double2 lo = v[i], hi = v[i | (1 << J)];
        pair_update<CLS>(lo, hi, c);
        if (tok) {
            v[i] = lo;
            v[i | (1 << J)] = hi;
        }
    }
}

template <int RB, int CLS>
__device__ __forceinline__ void tile_reg_dispatch(Regs<RB>& v, const double* c, int J, uint32_t rcm,
                                                  bool tok) {
    switch (J) {
    case 0: tile_reg_pair<RB, 0, CLS>(v, c, rcm, tok); break;
    case 1: if constexpr (RB > 1) tile_reg_pair<RB, 1, CLS>(v, c, rcm, tok); break;
    case 2: if constexpr (RB > 2) tile_reg_pair<RB, 2, CLS>(v, c, rcm, tok); break;
    default: if constexpr (RB > 3) tile_reg_pair<RB, 3, CLS>(v, c, rcm, tok); break;
    }
}

template <int RB, int CLS>
__device__ __forceinline__ void tile_lane_pair(Regs<RB>& v, const double* c, uint32_t b, uint32_t rcm,
                                               bool tok, uint32_t lane) {
    const uint32_t mask = 1u << b;
    const bool own_lo = (lane & mask) == 0;
    // distributed.cpp:183-184: own_lo ? lo_out(mine, theirs) : hi_out(theirs, mine)
    const double q0 = own_lo ? c[0] : c[4], q1 = own_lo ? c[1] : c[5];
    const double q2 = own_lo ? c[2] : c[6], q3 = own_lo ? c[3] : c[7];
#pragma unroll
    for (int i = 0; i < (1 << RB); ++i) {
        if ((static_cast<uint32_t>(i) & rcm) != rcm) continue; // uniform: shuffles stay converged
        double2 th;
        th.x = __shfl_xor_sync(0xffffffffu, v[i].x, mask);
        th.y = __shfl_xor_sync(0xffffffffu, v[i].y, mask);
        double2 r;
        if constexpr (CLS == CLS_SWAP) {
            r = th;
        } else {
            const double2 lo = own_lo ? v[i] : th;
            const double2 hi = own_lo ? th : v[i];
            r = row<CLS == CLS_REAL ? 0b1010 : 0>(q0, q1, q2, q3, lo, hi);
        }
        if (tok) v[i] = r;
    }
}

struct BitSrc {
    bool reg;
    uint32_t pos, fixed;
};

__device__ __forceinline__ BitSrc bit_src(uint8_t kind, uint8_t pos, uint32_t lane, uint32_t w,
                                          uint64_t gbase) {
    BitSrc s;
    s.reg = kind == TL_REG;
    s.pos = pos;
    s.fixed = kind == TL_LANE   ? (lane >> pos) & 1u
              : kind == TL_WARP ? (w >> pos) & 1u
                                : static_cast<uint32_t>((gbase >> pos) & 1u);
    return s;
}

__device__ __forceinline__ uint32_t bit_at(const BitSrc& s, int i) {
    return s.reg ? (static_cast<uint32_t>(i) >> s.pos) & 1u : s.fixed;
}

template <int RB>
__device__ __forceinline__ void tile_apply(Regs<RB>& v, const TileOp& op, uint32_t lane, uint32_t w,
                                           uint64_t gbase) {
    const bool tok = (lane & op.lane_cmask) == op.lane_cmask &&
                     (w & op.warp_cmask) == op.warp_cmask &&
                     (gbase & op.outer_cmask) == op.outer_cmask;
    const uint32_t rcm = op.reg_cmask;
    double c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = op.m[k];
    switch (op.kind) {
    case PO_PAIR_REG:
        switch (op.cls) {
        case CLS_SWAP: tile_reg_dispatch<RB, CLS_SWAP>(v, c, op.q0p, rcm, tok); break;
        case CLS_REAL: tile_reg_dispatch<RB, CLS_REAL>(v, c, op.q0p, rcm, tok); break;
        case CLS_RX: tile_reg_dispatch<RB, CLS_RX>(v, c, op.q0p, rcm, tok); break;
        default: tile_reg_dispatch<RB, CLS_GENERIC>(v, c, op.q0p, rcm, tok); break;
        }
        break;
    case PO_PAIR_LANE:
        switch (op.cls) {
        case CLS_SWAP: tile_lane_pair<RB, CLS_SWAP>(v, c, op.q0p, rcm, tok, lane); break;
        case CLS_REAL: tile_lane_pair<RB, CLS_REAL>(v, c, op.q0p, rcm, tok, lane); break;
        default: tile_lane_pair<RB, CLS_GENERIC>(v, c, op.q0p, rcm, tok, lane); break;
        }
        break;
    case PO_DIAG: {
        const BitSrc s0 = bit_src(op.q0k, op.q0p, lane, w, gbase);
        const bool a_one = op.flags & DF_A_ONE, d_one = op.flags & DF_D_ONE;
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            if ((static_cast<uint32_t>(i) & rcm) != rcm) continue;
            const uint32_t b = bit_at(s0, i);
            const double2 r = diag_mul(c, b, v[i]);
            if (tok && !(b ? d_one : a_one)) v[i] = r;
        }
        break;
    }
    case PO_DEPHASE: { // density.cpp:56-59
        const BitSrc s0 = bit_src(op.q0k, op.q0p, lane, w, gbase);
        const BitSrc s1 = bit_src(op.q1k, op.q1p, lane, w, gbase);
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            if (bit_at(s0, i) != bit_at(s1, i)) {
                v[i].x *= c[0];
                v[i].y *= c[0];
            }
        }
        break;
    }
    default: { // PO_COLLAPSE
        const BitSrc s0 = bit_src(op.q0k, op.q0p, lane, w, gbase);
        const BitSrc s1 = bit_src(op.q1k, op.q1p, lane, w, gbase);
        const uint32_t o = op.outcome;
        const bool two = op.flags & 1;
#pragma unroll
        for (int i = 0; i < (1 << RB); ++i) {
            const bool keep = bit_at(s0, i) == o && (!two || bit_at(s1, i) == o);
            v[i].x = keep ? v[i].x * c[0] : 0.0;
            v[i].y = keep ? v[i].y * c[0] : 0.0;
        }
        break;
    }
    }
}

template <int RB, int WB>
__global__ void __launch_bounds__(32 << WB, 2)
k_tile_pass(double2* __restrict__ amps, const __grid_constant__ TileParams P) {
    constexpr int R = 1 << RB;
    extern __shared__ double2 tile[];
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t w = threadIdx.x >> 5;
    const int nph = P.num_phases;
    for (uint64_t T = blockIdx.x; T < P.num_tiles; T += gridDim.x) {
        uint64_t gb = T << kLaneQubits;
#pragma unroll
        for (int j = 0; j < RB + WB; ++j) gb = insert_zero_bit(gb, P.high_pos[j]);
        const uint64_t gbase = gb + P.global_offset;
        double2* base = amps + gb + lane;
        double2 v[R];
        for (int ph = 0; ph < nph; ++ph) {
            const TilePhase& Q = P.phases[ph];
            const uint32_t wofs = Q.warp_off[w];
            if (ph == 0) {
#pragma unroll
                for (int i = 0; i < R; ++i) v[i] = __ldcs(base + P.seg_off[(wofs + Q.reg_off[i]) >> 5]);
            } else {
                __syncthreads();
#pragma unroll
                for (int i = 0; i < R; ++i) v[i] = tile[wofs + Q.reg_off[i] + lane];
            }
            for (int o = Q.op_begin; o < Q.op_end; ++o) tile_apply<RB>(v, P.ops[o], lane, w, gbase);
            if (ph == nph - 1) {
#pragma unroll
                for (int i = 0; i < R; ++i) __stcs(base + P.seg_off[(wofs + Q.reg_off[i]) >> 5], v[i]);
            } else {
#pragma unroll
                for (int i = 0; i < R; ++i) tile[wofs + Q.reg_off[i] + lane] = v[i];
            }
        }
        if (nph > 1) __syncthreads();
    }
}

// --------------------------------------------------------- simple kernels

inline unsigned grid_for(uint64_t work, int threads, unsigned cap = 148u * 16u) {
    uint64_t blocks = (work + threads - 1) / threads;
    if (blocks < 1) blocks = 1;
    if (blocks > cap) blocks = cap;
    return static_cast<unsigned>(blocks);
}

template <int CLS>
__global__ void k_gate_simple(double2* __restrict__ amps, uint64_t num_pairs, int t,
                              uint64_t cmask, Mat2 m) {
    const uint64_t off = uint64_t{1} << t;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
         i < num_pairs; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t base = pair_base_index(i, t);
        if ((base & cmask) != cmask) continue;
        double2 lo = amps[base], hi = amps[base + off];
        pair_update<CLS>(lo, hi, m.m);
        amps[base] = lo;
        amps[base + off] = hi;
    }
}

__global__ void k_diag_simple(double2* __restrict__ amps, uint64_t len, uint64_t goff,
                              int t, uint64_t cmask, Mat2 m, uint8_t flags) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t g = goff + i;
        if ((g & cmask) != cmask) continue;
        const uint32_t b = static_cast<uint32_t>((g >> t) & 1u);
        if ((b == 0 && (flags & DF_A_ONE)) || (b == 1 && (flags & DF_D_ONE))) continue;
        amps[i] = diag_mul(m.m, b, amps[i]);
    }
}

__global__ void k_dephase(double2* __restrict__ amps, uint64_t len, uint64_t goff, int q0,
                          int q1, double scale) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t g = goff + i;
        if (((g >> q0) & 1u) != ((g >> q1) & 1u)) {
            double2 a = amps[i];
            a.x *= scale;
            a.y *= scale;
            amps[i] = a;
        }
    }
}

__global__ void k_collapse(double2* __restrict__ amps, uint64_t len, uint64_t goff, int q0,
                           int q1, int outcome, double scale) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t g = goff + i;
        const bool keep = static_cast<int>((g >> q0) & 1u) == outcome &&
                          (q1 < 0 || static_cast<int>((g >> q1) & 1u) == outcome);
        if (keep) {
            double2 a = amps[i];
            a.x *= scale;
            a.y *= scale;
            amps[i] = a;
        } else {
            amps[i] = make_double2(0.0, 0.0);
        }
    }
}

// density.cpp:62-81 (keep/swap diagonal mix uses the reference's contraction:
// fma(swap, other, keep * own)).
__global__ void k_depolarise(double2* __restrict__ amps, uint64_t count, int t, int tN,
                             double keep, double swap, double off) {
    const uint64_t row = uint64_t{1} << t, col = uint64_t{1} << tN;
    for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; u < count;
         u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t n00 = insert_zero_bit(insert_zero_bit(u, t), tN);
        const uint64_t n11 = n00 | row | col;
        const double2 d0 = amps[n00], d1 = amps[n11];
        amps[n00] = make_double2(fma(swap, d1.x, keep * d0.x), fma(swap, d1.y, keep * d0.y));
        amps[n11] = make_double2(fma(swap, d0.x, keep * d1.x), fma(swap, d0.y, keep * d1.y));
        double2 a = amps[n00 | row], c = amps[n00 | col];
        a.x *= off; a.y *= off;
        c.x *= off; c.y *= off;
        amps[n00 | row] = a;
        amps[n00 | col] = c;
    }
}

template <int CLS>
__global__ void k_combine(double2* __restrict__ mine, const double2* __restrict__ theirs,
                          uint64_t len, uint64_t idx0, uint64_t low_mask, int own_lo, Mat2 m) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (((idx0 + i) & low_mask) != low_mask) continue;
        double2 lo, hi;
        if (own_lo) {
            lo = mine[i];
            hi = theirs[i];
        } else {
            lo = theirs[i];
            hi = mine[i];
        }
        pair_update<CLS>(lo, hi, m.m);
        mine[i] = own_lo ? lo : hi;
    }
}

__global__ void k_combine_depol(double2* __restrict__ mine, const double2* __restrict__ theirs,
                                uint64_t len, uint64_t idx0, int t, int own_col, double keep,
                                double swap, double off) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(((idx0 + i) >> t) & 1u);
        double2 a = mine[i];
        if (r != own_col) {
            a.x *= off;
            a.y *= off;
        } else {
            const double2 o = theirs[i ^ (uint64_t{1} << t)];
            a = make_double2(fma(swap, o.x, keep * a.x), fma(swap, o.y, keep * a.y));
        }
        mine[i] = a;
    }
}

// ----------------------------------------------------------- reductions

// Double-double accumulator (hi + lo); Kahan per element, TwoSum merges.
struct DD {
    double hi, lo;
};

__device__ __forceinline__ DD dd_add(DD a, DD b) {
    const double s = a.hi + b.hi;
    const double bb = s - a.hi;
    const double e = (a.hi - (s - bb)) + (b.hi - bb);
    const double t = e + a.lo + b.lo;
    const double hi = s + t;
    return DD{hi, t - (hi - s)};
}

__device__ __forceinline__ void dd_acc(DD& a, double x) {
    const double s = a.hi + x;
    const double bb = s - a.hi;
    a.lo += (a.hi - (s - bb)) + (x - bb);
    a.hi = s;
}

__device__ __forceinline__ DD block_reduce(DD v) {
    __shared__ DD sm[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        DD w;
        w.hi = __shfl_down_sync(0xffffffffu, v.hi, o);
        w.lo = __shfl_down_sync(0xffffffffu, v.lo, o);
        v = dd_add(v, w);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sm[wid] = v;
    __syncthreads();
    if (wid == 0) {
        v = lane < static_cast<int>(blockDim.x >> 5) ? sm[lane] : DD{0.0, 0.0};
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            DD w;
            w.hi = __shfl_down_sync(0xffffffffu, v.hi, o);
            w.lo = __shfl_down_sync(0xffffffffu, v.lo, o);
            v = dd_add(v, w);
        }
    }
    return v;
}

__global__ void __launch_bounds__(kReduceThreads)
k_reduce_norm(const double2* __restrict__ amps, uint64_t len, uint64_t goff, int t,
              int outcome, double2* __restrict__ partials) {
    DD acc{0.0, 0.0};
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (t >= 0 && static_cast<int>(((goff + i) >> t) & 1u) != outcome) continue;
        const double2 a = __ldcs(amps + i);
        dd_acc(acc, __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y)));
    }
    acc = block_reduce(acc);
    if (threadIdx.x == 0) partials[blockIdx.x] = make_double2(acc.hi, acc.lo);
}

__global__ void k_reduce_diag(const double2* __restrict__ amps, uint64_t len, uint64_t goff,
                              int N, int t, int outcome, int comp, double2* __restrict__ partials) {
    DD acc{0.0, 0.0};
    const uint64_t dim = uint64_t{1} << N;
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < dim;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t g = j * (dim + 1);
        if (g < goff || g >= goff + len) continue;
        if (t >= 0 && static_cast<int>((j >> t) & 1u) != outcome) continue;
        dd_acc(acc, comp ? amps[g - goff].y : amps[g - goff].x);
    }
    acc = block_reduce(acc);
    if (threadIdx.x == 0) partials[blockIdx.x] = make_double2(acc.hi, acc.lo);
}

__global__ void k_reduce_final(const double2* __restrict__ partials, int n,
                               double2* __restrict__ result) {
    DD acc{0.0, 0.0};
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        acc = dd_add(acc, DD{partials[i].x, partials[i].y});
    acc = block_reduce(acc);
    if (threadIdx.x == 0) *result = make_double2(acc.hi, acc.lo);
}

__global__ void k_fill(double2* __restrict__ amps, uint64_t len, double2 value) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        amps[i] = value;
}

} // namespace

uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

void launch_pass(double2* amps, const PassParams& p, cudaStream_t s) {
    constexpr int threads = 256;
    const uint64_t warps = p.num_tiles;
    uint64_t blocks = (warps * 32 + threads - 1) / threads;
    const uint64_t cap = 148ull * 8ull;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    switch (p.H) {
    case 1: k_fused_pass<1><<<static_cast<unsigned>(blocks), threads, 0, s>>>(amps, p); break;
    case 2: k_fused_pass<2><<<static_cast<unsigned>(blocks), threads, 0, s>>>(amps, p); break;
    default: k_fused_pass<3><<<static_cast<unsigned>(blocks), threads, 0, s>>>(amps, p); break;
    }
    count_launch();
}

void launch_tile_pass(double2* amps, const TileParams& p, cudaStream_t s) {
    auto kern = k_tile_pass<kPhaseRegBits, kTileWarpBits>;
    constexpr size_t smem_tile = sizeof(double2) << kTileQubits;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_tile));
        attr_set = true;
    }
    uint64_t blocks = p.num_tiles;
    const uint64_t cap = 148ull * 2ull; // persistent: 2 CTAs per SM
    if (blocks > cap) blocks = cap;
    const size_t smem = p.num_phases > 1 ? smem_tile : 0;
    kern<<<static_cast<unsigned>(blocks), kTileThreads, smem, s>>>(amps, p);
    count_launch();
}

void launch_gate_simple(double2* amps, int local_qubits, int target, uint64_t cmask,
                        const Mat2& m, int cls, cudaStream_t s) {
    const uint64_t pairs = uint64_t{1} << (local_qubits - 1);
    const unsigned g = grid_for(pairs, 256);
    switch (cls) {
    case CLS_REAL: k_gate_simple<CLS_REAL><<<g, 256, 0, s>>>(amps, pairs, target, cmask, m); break;
    case CLS_RX: k_gate_simple<CLS_RX><<<g, 256, 0, s>>>(amps, pairs, target, cmask, m); break;
    case CLS_SWAP: k_gate_simple<CLS_SWAP><<<g, 256, 0, s>>>(amps, pairs, target, cmask, m); break;
    default: k_gate_simple<CLS_GENERIC><<<g, 256, 0, s>>>(amps, pairs, target, cmask, m); break;
    }
    count_launch();
}

void launch_diag_simple(double2* amps, uint64_t len, uint64_t goff, int target, uint64_t cmask,
                        const Mat2& m, uint8_t flags, cudaStream_t s) {
    k_diag_simple<<<grid_for(len, 256), 256, 0, s>>>(amps, len, goff, target, cmask, m, flags);
    count_launch();
}

void launch_dephase(double2* amps, uint64_t len, uint64_t goff, int q0, int q1, double scale,
                    cudaStream_t s) {
    k_dephase<<<grid_for(len, 256), 256, 0, s>>>(amps, len, goff, q0, q1, scale);
    count_launch();
}

void launch_collapse(double2* amps, uint64_t len, uint64_t goff, int q0, int q1, int outcome,
                     double scale, cudaStream_t s) {
    k_collapse<<<grid_for(len, 256), 256, 0, s>>>(amps, len, goff, q0, q1, outcome, scale);
    count_launch();
}

void launch_depolarise(double2* amps, int local_qubits, int t, int tN, double keep, double swap,
                       double off, cudaStream_t s) {
    const uint64_t count = uint64_t{1} << (local_qubits - 2);
    k_depolarise<<<grid_for(count, 256), 256, 0, s>>>(amps, count, t, tN, keep, swap, off);
    count_launch();
}

void launch_combine(double2* mine, const double2* theirs, uint64_t len, uint64_t idx0,
                    uint64_t low_mask, int own_lo, const Mat2& m, int cls, cudaStream_t s) {
    const unsigned g = grid_for(len, 256);
    switch (cls) {
    case CLS_REAL: k_combine<CLS_REAL><<<g, 256, 0, s>>>(mine, theirs, len, idx0, low_mask, own_lo, m); break;
    case CLS_RX: k_combine<CLS_RX><<<g, 256, 0, s>>>(mine, theirs, len, idx0, low_mask, own_lo, m); break;
    case CLS_SWAP: k_combine<CLS_SWAP><<<g, 256, 0, s>>>(mine, theirs, len, idx0, low_mask, own_lo, m); break;
    default: k_combine<CLS_GENERIC><<<g, 256, 0, s>>>(mine, theirs, len, idx0, low_mask, own_lo, m); break;
    }
    count_launch();
}

void launch_combine_depol(double2* mine, const double2* theirs, uint64_t len, uint64_t idx0,
                          int t, int own_col, double keep, double swap, double off,
                          cudaStream_t s) {
    k_combine_depol<<<grid_for(len, 256), 256, 0, s>>>(mine, theirs, len, idx0, t, own_col, keep,
                                                      swap, off);
    count_launch();
}

void launch_reduce_norm(const double2* amps, uint64_t len, uint64_t goff, int t, int outcome,
                        double2* partials, double2* result, cudaStream_t s) {
    k_reduce_norm<<<kReduceBlocks, kReduceThreads, 0, s>>>(amps, len, goff, t, outcome, partials);
    k_reduce_final<<<1, kReduceThreads, 0, s>>>(partials, kReduceBlocks, result);
    count_launch();
    count_launch();
}

void launch_reduce_diag(const double2* amps, uint64_t len, uint64_t goff, int N, int t,
                        int outcome, int comp, double2* partials, double2* result,
                        cudaStream_t s) {
    k_reduce_diag<<<kReduceBlocks, kReduceThreads, 0, s>>>(amps, len, goff, N, t, outcome, comp,
                                                          partials);
    k_reduce_final<<<1, kReduceThreads, 0, s>>>(partials, kReduceBlocks, result);
    count_launch();
    count_launch();
}

void launch_fill(double2* amps, uint64_t len, double2 value, cudaStream_t s) {
    k_fill<<<grid_for(len, 256), 256, 0, s>>>(amps, len, value);
    count_launch();
}

} // namespace qgpu
