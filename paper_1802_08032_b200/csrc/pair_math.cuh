// pair_math.cuh — device-side pair arithmetic shared by the kernels.
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
// class (value-identical: such an fma only adds a signed zero).
#pragma once

#include "qgpu_device.h"

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#include <cstdint>
#endif

namespace qgpu {

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
template <int Z, class R, class V>
__device__ __forceinline__ V row(R q0, R q1, R q2, R q3, V lo, V hi) {
    constexpr bool n0 = !(Z & 1), n1 = !(Z & 2), n2 = !(Z & 4), n3 = !(Z & 8);
    R re, im;
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
        re = R(0);
        im = R(0);
    }
    if constexpr (n2) {
        re = fma(q2, hi.x, re);
        im = fma(q2, hi.y, im);
    }
    if constexpr (n3) {
        re = fma(q3, -hi.y, re); // = fma(-q3, y1, re) exactly; the negation stays on
                                 // the register operand so q3 can be a constant-bank one
        im = fma(q3, hi.x, im);
    }
    return V{re, im};
}

// Zero patterns of the two rows per class (see GateClass in qgpu_device.h).
template <int CLS> struct ClassZ;
template <> struct ClassZ<CLS_GENERIC> { static constexpr int z0 = 0, z1 = 0; };
template <> struct ClassZ<CLS_REAL> { static constexpr int z0 = 0b1010, z1 = 0b1010; };
template <> struct ClassZ<CLS_RX> { static constexpr int z0 = 0b0110, z1 = 0b1001; };

template <int CLS, class V, class R>
__device__ __forceinline__ void pair_update(V& lo, V& hi, const R* m) {
    if constexpr (CLS == CLS_SWAP) {
        const V t = lo;
        lo = hi;
        hi = t;
    } else {
        const V l = lo, h = hi;
        lo = row<ClassZ<CLS>::z0>(m[0], m[1], m[2], m[3], l, h);
        hi = row<ClassZ<CLS>::z1>(m[4], m[5], m[6], m[7], l, h);
    }
}

// Diagonal gate on one amplitude whose target bit is b: a * v (b = 0) or
// d * v (b = 1), each with the rounding of its reference row (the a term is
// the fused first product of the low row; the d term is the second product of
// the high row, so it rounds the other way round).
template <class R, class V>
__device__ __forceinline__ V diag_mul(const R* m, uint32_t b, V v) {
    const R ar = m[0], ai = m[1], dr = m[6], di = m[7];
    const R s1 = b ? -di : ar, t1 = b ? v.y : v.x;
    const R s2 = b ? dr : -ai, t2 = b ? v.x : v.y;
    const R u1 = b ? di : ar, w1 = b ? v.x : v.y;
    const R u2 = b ? dr : ai, w2 = b ? v.y : v.x;
    return V{fma(s1, t1, s2 * t2), fma(u1, w1, u2 * w2)};
}

} // namespace qgpu
