// kernels.cu — the sm_100a kernels around the hot tile pass (tile_pass.cu):
// register-only passes for small states, one-gate-per-launch kernels (the
// unfused mode), channels, exchange combines, compensated reductions.
// FP64, HBM-bandwidth bound: no tensor cores. The pair arithmetic is the
// reference's own fma chain (pair_math.cuh), so results are bit-identical to
// the reference on every amplitude (tests/test_gpu_parity.py).
#include "pair_math.cuh"
#include "qgpu_kernels.h"

#include <atomic>
#include <cuda_runtime.h>

namespace qgpu {

namespace {

std::atomic<uint64_t> g_launches{0};

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

// --------------------------------------------------------- simple kernels

inline unsigned grid_for(uint64_t work, int threads, unsigned cap = 148u * 16u) {
    uint64_t blocks = (work + threads - 1) / threads;
    if (blocks < 1) blocks = 1;
    if (blocks > cap) blocks = cap;
    return static_cast<unsigned>(blocks);
}

// The simple kernels are instantiated for both precisions: V = double2 / R =
// double, or V = float2 / R = float (the reference's Precision::Single:
// Mat2<float> narrows the gate matrix, channel factors are narrowed once,
// kernels.cpp:61-62, density.cpp:105-140).
template <class R> struct MatT { R m[8]; };

template <class R> MatT<R> narrow(const Mat2& m) {
    MatT<R> r;
    for (int k = 0; k < 8; ++k) r.m[k] = static_cast<R>(m.m[k]);
    return r;
}

template <class V> struct RealOf;
template <> struct RealOf<double2> { using type = double; };
template <> struct RealOf<float2> { using type = float; };

template <int CLS, class V, class R>
__global__ void k_gate_simple(V* __restrict__ amps, uint64_t num_pairs, int t, uint64_t cmask,
                              MatT<R> m) {
    const uint64_t off = uint64_t{1} << t;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
         i < num_pairs; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t base = pair_base_index(i, t);
        if ((base & cmask) != cmask) continue;
        V lo = amps[base], hi = amps[base + off];
        pair_update<CLS>(lo, hi, m.m);
        amps[base] = lo;
        amps[base + off] = hi;
    }
}

template <class V, class R>
__global__ void k_diag_simple(V* __restrict__ amps, uint64_t len, uint64_t goff, int t,
                              uint64_t cmask, MatT<R> m, uint8_t flags) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t g = goff + i;
        if ((g & cmask) != cmask) continue;
        const uint32_t b = static_cast<uint32_t>((g >> t) & 1u);
        if ((b == 0 && (flags & DF_A_ONE)) || (b == 1 && (flags & DF_D_ONE))) continue;
        amps[i] = diag_mul(m.m, b, amps[i]);
    }
}

template <class V, class R>
__global__ void k_dephase(V* __restrict__ amps, uint64_t len, uint64_t goff, int q0, int q1,
                          R scale) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t g = goff + i;
        if (((g >> q0) & 1u) != ((g >> q1) & 1u)) {
            V a = amps[i];
            a.x *= scale;
            a.y *= scale;
            amps[i] = a;
        }
    }
}

template <class V, class R>
__global__ void k_collapse(V* __restrict__ amps, uint64_t len, uint64_t goff, int q0, int q1,
                           int outcome, R scale) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t g = goff + i;
        const bool keep = static_cast<int>((g >> q0) & 1u) == outcome &&
                          (q1 < 0 || static_cast<int>((g >> q1) & 1u) == outcome);
        V a = amps[i];
        if (keep) {
            a.x *= scale;
            a.y *= scale;
        } else {
            a.x = R(0);
            a.y = R(0);
        }
        amps[i] = a;
    }
}

// density.cpp:62-81 (keep/swap diagonal mix uses the reference's contraction:
// fma(swap, other, keep * own)).
template <class V, class R>
__global__ void k_depolarise(V* __restrict__ amps, uint64_t count, int t, int tN, R keep,
                             R swap, R off) {
    const uint64_t row = uint64_t{1} << t, col = uint64_t{1} << tN;
    for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; u < count;
         u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        // the two bits in either order (the swap layer may permute them)
        const uint64_t n00 = insert_zero_bit(insert_zero_bit(u, t < tN ? t : tN), t < tN ? tN : t);
        const uint64_t n11 = n00 | row | col;
        const V d0 = amps[n00], d1 = amps[n11];
        amps[n00] = V{fma(swap, d1.x, keep * d0.x), fma(swap, d1.y, keep * d0.y)};
        amps[n11] = V{fma(swap, d0.x, keep * d1.x), fma(swap, d0.y, keep * d1.y)};
        V a = amps[n00 | row], c = amps[n00 | col];
        a.x *= off; a.y *= off;
        c.x *= off; c.y *= off;
        amps[n00 | row] = a;
        amps[n00 | col] = c;
    }
}

template <int CLS, class V, class R>
__global__ void k_combine(V* __restrict__ mine, const V* __restrict__ theirs, uint64_t len,
                          uint64_t idx0, uint64_t low_mask, int own_lo, MatT<R> m) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (((idx0 + i) & low_mask) != low_mask) continue;
        V lo, hi;
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

// ---- peer-memory exchange (single-node transport, peer.h) -----------------
// One GPU updates BOTH members of each amplitude pair -- its own element in
// local HBM and the partner's over NVLink (a mapped peer pointer) -- so no
// element is ever read after its owner overwrote it and no staging copy
// exists. The two ranks of a pair split the index range in halves. Four
// independent elements per thread keep enough remote loads in flight.
constexpr int kPeerIlp = 4;

// distributed.cpp:174-187 with both halves written: lo_side[i] / hi_side[i]
// are the pair (own_lo rank's element, partner's element) of local index i.
template <int CLS, class V, class R>
__global__ void __launch_bounds__(256) k_peer_combine(V* __restrict__ lo_side, V* __restrict__ hi_side,
                                                      uint64_t begin, uint64_t n, uint64_t low_mask, MatT<R> m) {
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < n; b += kPeerIlp * T) {
        V lo[kPeerIlp], hi[kPeerIlp];
        bool ok[kPeerIlp];
#pragma unroll
        for (int k = 0; k < kPeerIlp; ++k) {
            const uint64_t i = begin + b + k * T;
            ok[k] = b + k * T < n && (i & low_mask) == low_mask;
            if (ok[k]) {
                lo[k] = lo_side[i];
                hi[k] = hi_side[i];
            }
        }
#pragma unroll
        for (int k = 0; k < kPeerIlp; ++k) {
            if (!ok[k]) continue;
            const uint64_t i = begin + b + k * T;
            pair_update<CLS>(lo[k], hi[k], m.m);
            lo_side[i] = lo[k];
            hi_side[i] = hi[k];
        }
    }
}

// Global<->local qubit swap: element e of the traded half space sits at
// own[pos(e, side_own)] and remote[pos(e, !side_own)], pos(e, s) = e with bit
// v set to s; the two are exchanged (pure moves, exact).
template <class V>
__global__ void __launch_bounds__(256) k_peer_swap(V* __restrict__ own, V* __restrict__ remote, uint64_t e0,
                                                   uint64_t n, int v, int side_own) {
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t low = (uint64_t{1} << v) - 1;
    const uint64_t so = static_cast<uint64_t>(side_own) << v, sr = static_cast<uint64_t>(side_own ^ 1) << v;
    for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < n; b += kPeerIlp * T) {
        V x[kPeerIlp], y[kPeerIlp];
        uint64_t base[kPeerIlp];
#pragma unroll
        for (int k = 0; k < kPeerIlp; ++k) {
            const uint64_t e = e0 + b + k * T;
            base[k] = ((e & ~low) << 1) | (e & low);
            if (b + k * T < n) {
                x[k] = own[base[k] | so];
                y[k] = remote[base[k] | sr];
            }
        }
#pragma unroll
        for (int k = 0; k < kPeerIlp; ++k) {
            if (b + k * T >= n) continue;
            own[base[k] | so] = y[k];
            remote[base[k] | sr] = x[k];
        }
    }
}

// Depolarising with the bra qubit on the rank bits (k_combine_depol's
// arithmetic): corner pair k = (col0[i], col1[i | 2^t]), i = k with a zero
// inserted at bit t; both corners mix as fma(swap, other, keep * self).
template <class V, class R>
__global__ void __launch_bounds__(256) k_peer_combine_depol(V* __restrict__ col0, V* __restrict__ col1,
                                                            uint64_t k0, uint64_t n, int t, R keep, R swap) {
    const uint64_t T = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; b < n; b += kPeerIlp * T) {
        V x[kPeerIlp], y[kPeerIlp];
        uint64_t idx[kPeerIlp];
#pragma unroll
        for (int k = 0; k < kPeerIlp; ++k) {
            idx[k] = insert_zero_bit(k0 + b + k * T, t);
            if (b + k * T < n) {
                x[k] = col0[idx[k]];
                y[k] = col1[idx[k] | (uint64_t{1} << t)];
            }
        }
#pragma unroll
        for (int k = 0; k < kPeerIlp; ++k) {
            if (b + k * T >= n) continue;
            col0[idx[k]] = V{fma(swap, y[k].x, keep * x[k].x), fma(swap, y[k].y, keep * x[k].y)};
            col1[idx[k] | (uint64_t{1} << t)] = V{fma(swap, x[k].x, keep * y[k].x), fma(swap, x[k].y, keep * y[k].y)};
        }
    }
}

// amps[i] *= f for the local indices i whose bit t equals `bit`
template <class V, class R>
__global__ void k_scale_bit(V* __restrict__ amps, uint64_t half, int t, int bit, R f) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < half;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t i = insert_zero_bit(k, t) | (static_cast<uint64_t>(bit) << t);
        V a = amps[i];
        a.x *= f;
        a.y *= f;
        amps[i] = a;
    }
}

template <class V, class R>
__global__ void k_combine_depol(V* __restrict__ mine, const V* __restrict__ theirs, uint64_t len,
                                uint64_t idx0, int t, int own_col, R keep, R swap, R off) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(((idx0 + i) >> t) & 1u);
        V a = mine[i];
        if (r != own_col) {
            a.x *= off;
            a.y *= off;
        } else {
            const V o = theirs[i ^ (uint64_t{1} << t)];
            a = V{fma(swap, o.x, keep * a.x), fma(swap, o.y, keep * a.y)};
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

// Sum of |a|^2 over the amplitudes whose global bit t equals `outcome` (all
// for t < 0). Only qualifying amplitudes are read (half the state for a
// probability), four independent 16 B loads per thread per iteration (one
// in flight per thread left HBM at 4.4 TB/s), compensated per thread, then
// merged in a fixed order (deterministic).
// Single-precision registers widen each amplitude to double before squaring
// (AmpVector::norm_squared, register.cpp:62-73).
template <class V>
__global__ void __launch_bounds__(kReduceThreads)
k_reduce_norm(const V* __restrict__ amps, uint64_t len, uint64_t goff, int t,
              int outcome, double2* __restrict__ partials) {
    DD acc{0.0, 0.0};
    int lb = 0;
    while ((uint64_t{1} << lb) < len) ++lb;
    const bool split = t >= 0 && t < lb;    // bit t varies inside this chunk
    const bool none = t >= lb && static_cast<int>((goff >> t) & 1u) != outcome;
    const uint64_t n = none ? 0 : split ? len >> 1 : len;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    auto at = [&](uint64_t k) {
        if (!split) return k;
        const uint64_t low = k & ((uint64_t{1} << t) - 1);
        return ((k >> t) << (t + 1)) | (static_cast<uint64_t>(outcome) << t) | low;
    };
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n; k += 4 * stride) {
        V v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t kk = k + u * stride;
            v[u] = kk < n ? __ldcs(amps + at(kk)) : V{0, 0};
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double x = v[u].x, y = v[u].y;
            dd_acc(acc, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
        }
    }
    acc = block_reduce(acc);
    if (threadIdx.x == 0) partials[blockIdx.x] = make_double2(acc.hi, acc.lo);
}

template <class V>
__global__ void k_reduce_diag(const V* __restrict__ amps, uint64_t len, uint64_t goff,
                              int N, int t, int outcome, int comp, double2* __restrict__ partials) {
    DD acc{0.0, 0.0};
    const uint64_t dim = uint64_t{1} << N;
    for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < dim;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t g = j * (dim + 1);
        if (g < goff || g >= goff + len) continue;
        if (t >= 0 && static_cast<int>((j >> t) & 1u) != outcome) continue;
        dd_acc(acc, static_cast<double>(comp ? amps[g - goff].y : amps[g - goff].x));
    }
    acc = block_reduce(acc);
    if (threadIdx.x == 0) partials[blockIdx.x] = make_double2(acc.hi, acc.lo);
}

// ---- all single-qubit marginals in one read (calcProbOfOutcome cache) ----
// Block iteration = one chunk of 2^13 amplitudes: thread t reads elements
// t + 256 j (j < 32), so index bits 0-4 are its lane, 5-7 its warp (both
// fixed per thread), 8-12 the loop counter j, and bits >= 13 the chunk.
// Per thread: the chunk's sum and five j-bit sums (32 terms, plain) feed
// double-double accumulators; each warp's chunk sum goes to wsum for the
// chunk bits (k_marginals_hi). A final kernel merges the per-block partials
// in a fixed order (deterministic).
constexpr int kMargChunkBits = 13;
constexpr int kMargLo = 1 + 5 + 3 + 5; // total, lane bits, warp bits, j bits
constexpr int kMargHiMax = 36 - kMargChunkBits;
constexpr int kMargBlocks = 4 * 148;
constexpr int kMargHiBlocks = 2 * 148;

__device__ __forceinline__ void block_reduce_store(DD v, double2* out) {
    v = block_reduce(v);
    if (threadIdx.x == 0) *out = make_double2(v.hi, v.lo);
    __syncthreads(); // block_reduce's shared scratch is reused by the next call
}

template <class V>
__global__ void __launch_bounds__(256) k_marginals(const V* __restrict__ amps, uint64_t nchunks,
                                                   double* __restrict__ wsum, double2* __restrict__ part) {
    DD T{0.0, 0.0}, B[5];
#pragma unroll
    for (int b = 0; b < 5; ++b) B[b] = DD{0.0, 0.0};
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        const V* base = amps + (c << kMargChunkBits) + threadIdx.x;
        V v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __ldcs(base + 256 * j);
        double cs = 0.0, jb[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const double x = v[j].x, y = v[j].y;
            const double p = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
            cs += p;
#pragma unroll
            for (int b = 0; b < 5; ++b)
                if ((j >> b) & 1) jb[b] += p;
        }
        dd_acc(T, cs);
#pragma unroll
        for (int b = 0; b < 5; ++b) dd_acc(B[b], jb[b]);
        double ws = cs;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ws += __shfl_xor_sync(0xffffffffu, ws, o);
        if (lane == 0) wsum[(c << 3) | warp] = ws;
    }
    double2* out = part + static_cast<size_t>(blockIdx.x) * kMargLo;
    block_reduce_store(T, out);
#pragma unroll
    for (int b = 0; b < 5; ++b) block_reduce_store((lane >> b) & 1u ? T : DD{0.0, 0.0}, out + 1 + b);
#pragma unroll
    for (int b = 0; b < 3; ++b) block_reduce_store((warp >> b) & 1u ? T : DD{0.0, 0.0}, out + 6 + b);
#pragma unroll
    for (int b = 0; b < 5; ++b) block_reduce_store(B[b], out + 9 + b);
}

// chunk-bit marginals from the per-(chunk, warp) sums: element i of wsum
// belongs to chunk i >> 3
__global__ void __launch_bounds__(256) k_marginals_hi(const double* __restrict__ wsum, uint64_t nw, int hib,
                                                      double2* __restrict__ part) {
    double acc[kMargHiMax];
#pragma unroll
    for (int b = 0; b < kMargHiMax; ++b) acc[b] = 0.0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < nw;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double w = wsum[i];
        const uint64_t c = i >> 3;
#pragma unroll
        for (int b = 0; b < kMargHiMax; ++b)
            if (b < hib && ((c >> b) & 1u)) acc[b] += w;
    }
    double2* out = part + static_cast<size_t>(blockIdx.x) * kMargHiMax;
    for (int b = 0; b < hib; ++b) block_reduce_store(DD{acc[b], 0.0}, out + b);
}

// out[0] = total, out[1 + q] = sum over bit q == 1, q < m (double-double)
__global__ void __launch_bounds__(256) k_marginals_final(const double2* __restrict__ part, int g1,
                                                         const double2* __restrict__ part2, int g2, int hib,
                                                         double2* __restrict__ out) {
    for (int k = 0; k < kMargLo; ++k) {
        DD a{0.0, 0.0};
        for (int i = threadIdx.x; i < g1; i += blockDim.x) {
            const double2 v = part[static_cast<size_t>(i) * kMargLo + k];
            a = dd_add(a, DD{v.x, v.y});
        }
        block_reduce_store(a, out + k); // k: total, bits 0-4, 5-7, 8-12 in order
    }
    for (int b = 0; b < hib; ++b) {
        DD a{0.0, 0.0};
        for (int i = threadIdx.x; i < g2; i += blockDim.x) {
            const double2 v = part2[static_cast<size_t>(i) * kMargHiMax + b];
            a = dd_add(a, DD{v.x, v.y});
        }
        block_reduce_store(a, out + kMargLo + b); // bit 13 + b
    }
}

// Sum of |a|^2 over the amplitudes whose local index holds `val` on the bits
// of `mask` (up to 8 bits; the selection reductions of deferred collapses):
// only the selected 2^-popcount(mask) of the state is read.
template <class V>
__global__ void __launch_bounds__(kReduceThreads)
k_reduce_norm_sel(const V* __restrict__ amps, uint64_t n, uint64_t mask, uint64_t val,
                  double2* __restrict__ partials) {
    DD acc{0.0, 0.0};
    int pos[8];
    int np = 0;
    for (uint64_t m = mask; m && np < 8; m &= m - 1) pos[np++] = __ffsll(static_cast<long long>(m)) - 1;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    auto at = [&](uint64_t k) {
        for (int j = 0; j < np; ++j) k = insert_zero_bit(k, pos[j]); // ascending positions
        return k | val;
    };
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n; k += 4 * stride) {
        V v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t kk = k + u * stride;
            v[u] = kk < n ? __ldcs(amps + at(kk)) : V{0, 0};
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double x = v[u].x, y = v[u].y;
            dd_acc(acc, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)));
        }
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

template <class V>
__global__ void k_fill(V* __restrict__ amps, uint64_t len, V value) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < len;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        amps[i] = value;
}

} // namespace

uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
std::atomic<uint64_t> g_h2d{0}, g_d2h{0};
}
void count_transfer(uint64_t h2d, uint64_t d2h) {
    if (h2d) g_h2d.fetch_add(h2d, std::memory_order_relaxed);
    if (d2h) g_d2h.fetch_add(d2h, std::memory_order_relaxed);
}
void transfer_bytes(uint64_t* h2d, uint64_t* d2h) {
    *h2d = g_h2d.load(std::memory_order_relaxed);
    *d2h = g_d2h.load(std::memory_order_relaxed);
}

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
    count_transfer(sizeof(PassParams) + sizeof(amps), 0);
    count_launch();
}

namespace {

template <class V, class R>
void gate_simple(V* amps, int local_qubits, int target, uint64_t cmask, const Mat2& mat, int cls,
                 cudaStream_t s) {
    const uint64_t pairs = uint64_t{1} << (local_qubits - 1);
    const unsigned g = grid_for(pairs, 256);
    const MatT<R> m = narrow<R>(mat);
    switch (cls) {
    case CLS_REAL: k_gate_simple<CLS_REAL><<<g, 256, 0, s>>>(amps, pairs, target, cmask, m); break;
    case CLS_RX: k_gate_simple<CLS_RX><<<g, 256, 0, s>>>(amps, pairs, target, cmask, m); break;
    case CLS_SWAP: k_gate_simple<CLS_SWAP><<<g, 256, 0, s>>>(amps, pairs, target, cmask, m); break;
    default: k_gate_simple<CLS_GENERIC><<<g, 256, 0, s>>>(amps, pairs, target, cmask, m); break;
    }
}

template <class V, class R>
void combine(V* mine, const V* theirs, uint64_t len, uint64_t idx0, uint64_t low_mask, int own_lo,
             const Mat2& mat, int cls, cudaStream_t s) {
    const unsigned g = grid_for(len, 256);
    const MatT<R> m = narrow<R>(mat);
    switch (cls) {
    case CLS_REAL: k_combine<CLS_REAL><<<g, 256, 0, s>>>(mine, theirs, len, idx0, low_mask, own_lo, m); break;
    case CLS_RX: k_combine<CLS_RX><<<g, 256, 0, s>>>(mine, theirs, len, idx0, low_mask, own_lo, m); break;
    case CLS_SWAP: k_combine<CLS_SWAP><<<g, 256, 0, s>>>(mine, theirs, len, idx0, low_mask, own_lo, m); break;
    default: k_combine<CLS_GENERIC><<<g, 256, 0, s>>>(mine, theirs, len, idx0, low_mask, own_lo, m); break;
    }
}

template <class V> V* as(void* p) { return static_cast<V*>(p); }
template <class V> const V* as(const void* p) { return static_cast<const V*>(p); }

} // namespace

void launch_gate_simple(void* amps, bool single, int local_qubits, int target, uint64_t cmask,
                        const Mat2& m, int cls, cudaStream_t s) {
    if (single)
        gate_simple<float2, float>(as<float2>(amps), local_qubits, target, cmask, m, cls, s);
    else
        gate_simple<double2, double>(as<double2>(amps), local_qubits, target, cmask, m, cls, s);
    count_launch();
}

void launch_diag_simple(void* amps, bool single, uint64_t len, uint64_t goff, int target,
                        uint64_t cmask, const Mat2& m, uint8_t flags, cudaStream_t s) {
    const unsigned g = grid_for(len, 256);
    if (single)
        k_diag_simple<<<g, 256, 0, s>>>(as<float2>(amps), len, goff, target, cmask, narrow<float>(m), flags);
    else
        k_diag_simple<<<g, 256, 0, s>>>(as<double2>(amps), len, goff, target, cmask, narrow<double>(m), flags);
    count_launch();
}

void launch_dephase(void* amps, bool single, uint64_t len, uint64_t goff, int q0, int q1,
                    double scale, cudaStream_t s) {
    const unsigned g = grid_for(len, 256);
    if (single)
        k_dephase<<<g, 256, 0, s>>>(as<float2>(amps), len, goff, q0, q1, static_cast<float>(scale));
    else
        k_dephase<<<g, 256, 0, s>>>(as<double2>(amps), len, goff, q0, q1, scale);
    count_launch();
}

void launch_collapse(void* amps, bool single, uint64_t len, uint64_t goff, int q0, int q1,
                     int outcome, double scale, cudaStream_t s) {
    const unsigned g = grid_for(len, 256);
    if (single)
        k_collapse<<<g, 256, 0, s>>>(as<float2>(amps), len, goff, q0, q1, outcome, static_cast<float>(scale));
    else
        k_collapse<<<g, 256, 0, s>>>(as<double2>(amps), len, goff, q0, q1, outcome, scale);
    count_launch();
}

void launch_depolarise(void* amps, bool single, int local_qubits, int t, int tN, double keep,
                       double swap, double off, cudaStream_t s) {
    const uint64_t count = uint64_t{1} << (local_qubits - 2);
    const unsigned g = grid_for(count, 256);
    if (single)
        k_depolarise<<<g, 256, 0, s>>>(as<float2>(amps), count, t, tN, static_cast<float>(keep),
                                       static_cast<float>(swap), static_cast<float>(off));
    else
        k_depolarise<<<g, 256, 0, s>>>(as<double2>(amps), count, t, tN, keep, swap, off);
    count_launch();
}

void launch_combine(void* mine, const void* theirs, bool single, uint64_t len, uint64_t idx0,
                    uint64_t low_mask, int own_lo, const Mat2& m, int cls, cudaStream_t s) {
    if (single)
        combine<float2, float>(as<float2>(mine), as<float2>(theirs), len, idx0, low_mask, own_lo, m, cls, s);
    else
        combine<double2, double>(as<double2>(mine), as<double2>(theirs), len, idx0, low_mask, own_lo, m, cls, s);
    count_launch();
}

void launch_combine_depol(void* mine, const void* theirs, bool single, uint64_t len, uint64_t idx0,
                          int t, int own_col, double keep, double swap, double off,
                          cudaStream_t s) {
    const unsigned g = grid_for(len, 256);
    if (single)
        k_combine_depol<<<g, 256, 0, s>>>(as<float2>(mine), as<float2>(theirs), len, idx0, t, own_col,
                                          static_cast<float>(keep), static_cast<float>(swap),
                                          static_cast<float>(off));
    else
        k_combine_depol<<<g, 256, 0, s>>>(as<double2>(mine), as<double2>(theirs), len, idx0, t, own_col,
                                          keep, swap, off);
    count_launch();
}

namespace {
template <class V, class R>
void peer_combine(V* lo_side, V* hi_side, uint64_t begin, uint64_t n, uint64_t low_mask, const Mat2& mat,
                  int cls, cudaStream_t s) {
    const unsigned g = grid_for((n + kPeerIlp - 1) / kPeerIlp, 256);
    const MatT<R> m = narrow<R>(mat);
    switch (cls) {
    case CLS_REAL: k_peer_combine<CLS_REAL><<<g, 256, 0, s>>>(lo_side, hi_side, begin, n, low_mask, m); break;
    case CLS_RX: k_peer_combine<CLS_RX><<<g, 256, 0, s>>>(lo_side, hi_side, begin, n, low_mask, m); break;
    case CLS_SWAP: k_peer_combine<CLS_SWAP><<<g, 256, 0, s>>>(lo_side, hi_side, begin, n, low_mask, m); break;
    default: k_peer_combine<CLS_GENERIC><<<g, 256, 0, s>>>(lo_side, hi_side, begin, n, low_mask, m); break;
    }
}
} // namespace

void launch_peer_combine(void* lo_side, void* hi_side, bool single, uint64_t begin, uint64_t n,
                         uint64_t low_mask, const Mat2& m, int cls, cudaStream_t s) {
    if (n == 0) return;
    if (single)
        peer_combine<float2, float>(as<float2>(lo_side), as<float2>(hi_side), begin, n, low_mask, m, cls, s);
    else
        peer_combine<double2, double>(as<double2>(lo_side), as<double2>(hi_side), begin, n, low_mask, m, cls, s);
    count_launch();
}

void launch_peer_swap(void* own, void* remote, bool single, uint64_t e0, uint64_t n, int v, int side_own,
                      cudaStream_t s) {
    if (n == 0) return;
    const unsigned g = grid_for((n + kPeerIlp - 1) / kPeerIlp, 256);
    if (single)
        k_peer_swap<<<g, 256, 0, s>>>(as<float2>(own), as<float2>(remote), e0, n, v, side_own);
    else
        k_peer_swap<<<g, 256, 0, s>>>(as<double2>(own), as<double2>(remote), e0, n, v, side_own);
    count_launch();
}

void launch_peer_combine_depol(void* col0, void* col1, bool single, uint64_t k0, uint64_t n, int t,
                               double keep, double swap, cudaStream_t s) {
    if (n == 0) return;
    const unsigned g = grid_for((n + kPeerIlp - 1) / kPeerIlp, 256);
    if (single)
        k_peer_combine_depol<<<g, 256, 0, s>>>(as<float2>(col0), as<float2>(col1), k0, n, t,
                                               static_cast<float>(keep), static_cast<float>(swap));
    else
        k_peer_combine_depol<<<g, 256, 0, s>>>(as<double2>(col0), as<double2>(col1), k0, n, t, keep, swap);
    count_launch();
}

void launch_scale_bit(void* amps, bool single, uint64_t len, int t, int bit, double f, cudaStream_t s) {
    const uint64_t half = len / 2;
    const unsigned g = grid_for(half, 256);
    if (single)
        k_scale_bit<<<g, 256, 0, s>>>(as<float2>(amps), half, t, bit, static_cast<float>(f));
    else
        k_scale_bit<<<g, 256, 0, s>>>(as<double2>(amps), half, t, bit, f);
    count_launch();
}

size_t marginals_scratch_bytes(int m) {
    const uint64_t nw = m >= kMargChunkBits ? (uint64_t{1} << (m - kMargChunkBits)) * 8 : 0;
    return nw * sizeof(double) + (static_cast<size_t>(kMargBlocks) * kMargLo +
                                  static_cast<size_t>(kMargHiBlocks) * kMargHiMax) * sizeof(double2);
}

void launch_marginals(const void* amps, bool single, int m, void* scratch, double2* out, cudaStream_t s) {
    const uint64_t nchunks = uint64_t{1} << (m - kMargChunkBits);
    const uint64_t nw = nchunks * 8;
    double* wsum = static_cast<double*>(scratch);
    double2* part = reinterpret_cast<double2*>(wsum + nw);
    double2* part2 = part + static_cast<size_t>(kMargBlocks) * kMargLo;
    const int g1 = static_cast<int>(std::min<uint64_t>(nchunks, kMargBlocks));
    const int hib = m - kMargChunkBits;
    if (single)
        k_marginals<<<g1, 256, 0, s>>>(as<float2>(amps), nchunks, wsum, part);
    else
        k_marginals<<<g1, 256, 0, s>>>(as<double2>(amps), nchunks, wsum, part);
    const int g2 = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((nw + 255) / 256, kMargHiBlocks)));
    if (hib > 0) k_marginals_hi<<<g2, 256, 0, s>>>(wsum, nw, hib, part2);
    k_marginals_final<<<1, 256, 0, s>>>(part, g1, part2, g2, hib, out);
    count_launch();
    count_launch();
    if (hib > 0) count_launch();
}

void launch_reduce_norm_sel(const void* amps, bool single, uint64_t len, uint64_t mask, uint64_t val,
                            double2* partials, double2* result, cudaStream_t s) {
    const uint64_t n = len >> __builtin_popcountll(mask);
    if (single)
        k_reduce_norm_sel<<<kReduceBlocks, kReduceThreads, 0, s>>>(as<float2>(amps), n, mask, val, partials);
    else
        k_reduce_norm_sel<<<kReduceBlocks, kReduceThreads, 0, s>>>(as<double2>(amps), n, mask, val, partials);
    k_reduce_final<<<1, kReduceThreads, 0, s>>>(partials, kReduceBlocks, result);
    count_launch();
    count_launch();
}

void launch_reduce_norm(const void* amps, bool single, uint64_t len, uint64_t goff, int t,
                        int outcome, double2* partials, double2* result, cudaStream_t s) {
    if (single)
        k_reduce_norm<<<kReduceBlocks, kReduceThreads, 0, s>>>(as<float2>(amps), len, goff, t, outcome, partials);
    else
        k_reduce_norm<<<kReduceBlocks, kReduceThreads, 0, s>>>(as<double2>(amps), len, goff, t, outcome, partials);
    k_reduce_final<<<1, kReduceThreads, 0, s>>>(partials, kReduceBlocks, result);
    count_launch();
    count_launch();
}

void launch_reduce_diag(const void* amps, bool single, uint64_t len, uint64_t goff, int N, int t,
                        int outcome, int comp, double2* partials, double2* result,
                        cudaStream_t s) {
    if (single)
        k_reduce_diag<<<kReduceBlocks, kReduceThreads, 0, s>>>(as<float2>(amps), len, goff, N, t, outcome,
                                                              comp, partials);
    else
        k_reduce_diag<<<kReduceBlocks, kReduceThreads, 0, s>>>(as<double2>(amps), len, goff, N, t, outcome,
                                                              comp, partials);
    k_reduce_final<<<1, kReduceThreads, 0, s>>>(partials, kReduceBlocks, result);
    count_launch();
    count_launch();
}

void launch_fill(void* amps, bool single, uint64_t len, double re, double im, cudaStream_t s) {
    const unsigned g = grid_for(len, 256);
    if (single)
        k_fill<<<g, 256, 0, s>>>(as<float2>(amps), len,
                                 make_float2(static_cast<float>(re), static_cast<float>(im)));
    else
        k_fill<<<g, 256, 0, s>>>(as<double2>(amps), len, make_double2(re, im));
    count_launch();
}

} // namespace qgpu
