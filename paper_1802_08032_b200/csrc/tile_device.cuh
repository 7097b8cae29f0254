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

// double precision (the reference's Precision::Double path)
namespace tile_f64 {
using Real = double;
using Cx = double2;
__device__ __forceinline__ Cx mk(Real x, Real y) { return make_double2(x, y); }
// an amplitude's shared-memory access as one v2.f64 instruction: left to
// itself ptxas split some into two 8-byte accesses when the two doubles sat
// in non-adjacent registers (2-way bank conflicts, ncu: 26 % excess
// wavefronts in JIT kernels)
__device__ __forceinline__ Cx lds16(const Cx* p) {
    Cx v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
                 : "=d"(v.x), "=d"(v.y)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
    return v;
}
__device__ __forceinline__ void sts16(Cx* p, Cx v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))),
                 "d"(v.x), "d"(v.y)
                 : "memory");
}
#include "tile_body.inc"
} // namespace tile_f64

// single precision (Precision::Single: Mat2<float>, float arithmetic)
namespace tile_f32 {
using Real = float;
using Cx = float2;
__device__ __forceinline__ Cx mk(Real x, Real y) { return make_float2(x, y); }
__device__ __forceinline__ Cx lds16(const Cx* p) {
    Cx v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];"
                 : "=f"(v.x), "=f"(v.y)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
    return v;
}
__device__ __forceinline__ void sts16(Cx* p, Cx v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))),
                 "f"(v.x), "f"(v.y)
                 : "memory");
}
#include "tile_body.inc"
} // namespace tile_f32

} // namespace qgpu
