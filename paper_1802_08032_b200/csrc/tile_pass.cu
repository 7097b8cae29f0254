// tile_pass.cu — the ahead-of-time instantiation of the tile pass (the
// interpreter over the op table; device code in tile_device.cuh) and its
// launcher, which prefers a per-pass JIT kernel (tile_jit.cpp) once compiled.
#include "tile_device.cuh"

#include "qgpu_kernels.h"
#include "runtime.h"

#include <cstdio>
#include <string>
#include <cuda_runtime.h>

namespace qgpu {

namespace {

template <int RB, int WB, int NBUF, bool FAST>
__global__ void __launch_bounds__(kTileThreads, 1)
k_tile_pass(double2* __restrict__ amps, const __grid_constant__ TileParams P) {
    tile_f64::tile_pass_body<RB, WB, NBUF, tile_f64::Interp<FAST>>(amps, P);
}

template <int RB, int WB, int NBUF, bool FAST>
__global__ void __launch_bounds__(kTileThreads, kTileCtasF32)
k_tile_pass_f32(float2* __restrict__ amps, const __grid_constant__ TileParams P) {
    tile_f32::tile_pass_body<RB, WB, NBUF, tile_f32::Interp<FAST>>(amps, P);
}

} // namespace

namespace {

template <class T>
void launch_interp(void (*kern)(T*, TileParams), void* amps, const TileParams& p, cudaStream_t s, size_t smem,
                   bool& set, int ctas_per_sm) {
    if (!set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        set = true;
    }
    uint64_t blocks = p.num_tiles;
    if (blocks > 148u * ctas_per_sm) blocks = 148u * ctas_per_sm; // persistent
    kern<<<static_cast<unsigned>(blocks), kTileThreads, smem, s>>>(static_cast<T*>(amps), p);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, kern);
        char msg[256];
        snprintf(msg, sizeof msg, "tile pass launch: %s (regs %d, max threads %d, static smem %zu, dyn smem %zu)",
                 cudaGetErrorString(e), fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes, smem);
        throw DeviceError(msg);
    }
}

} // namespace

void launch_tile_pass(void* amps, const TileParams& p, cudaStream_t s) {
    count_transfer(sizeof(TileParams) + sizeof(amps), 0); // the pass's op table rides in the launch
    if (launch_tile_pass_jit(amps, p, s)) { // straight-line kernel for this pass shape
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw DeviceError(std::string("jit tile pass launch: ") + cudaGetErrorString(e));
        count_launch();
        return;
    }
    constexpr int NBUF = kTileStages;
    if (p.single) {
        static bool set[2] = {false, false};
        launch_interp(p.fast ? k_tile_pass_f32<kPhaseRegBits, kTileWarpBits, NBUF, true>
                             : k_tile_pass_f32<kPhaseRegBits, kTileWarpBits, NBUF, false>,
                      amps, p, s, NBUF * (sizeof(float2) << kTileQubits), set[p.fast ? 1 : 0], kTileCtasF32);
    } else {
        static bool set[2] = {false, false};
        launch_interp(p.fast ? k_tile_pass<kPhaseRegBits, kTileWarpBits, NBUF, true>
                             : k_tile_pass<kPhaseRegBits, kTileWarpBits, NBUF, false>,
                      amps, p, s, NBUF * (sizeof(double2) << kTileQubits), set[p.fast ? 1 : 0], kTileCtasF64);
    }
    count_launch();
}

} // namespace qgpu
