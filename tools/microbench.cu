// Pipe-throughput microbenchmarks on sm_100a (shuffle, FP64 FMA, LDS.128,
// FSEL). Prints warp-instructions per clock per SM. Used to size the tile
// pass phases.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_shfl(float* out, int iters) {
    float a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
    for (int i = 0; i < iters; ++i) {
        a = __shfl_xor_sync(0xffffffffu, a, 1);
        b = __shfl_xor_sync(0xffffffffu, b, 2);
        c = __shfl_xor_sync(0xffffffffu, c, 4);
        d = __shfl_xor_sync(0xffffffffu, d, 8);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

__global__ void k_dfma(double* out, int iters) {
    double a = threadIdx.x, b = 1.0000001, c0 = 0.1, c1 = 0.2, c2 = 0.3, c3 = 0.4, c4 = 0.5, c5 = 0.6, c6 = 0.7, c7 = 0.8;
    for (int i = 0; i < iters; ++i) {
        c0 = fma(a, b, c0); c1 = fma(a, b, c1); c2 = fma(a, b, c2); c3 = fma(a, b, c3);
        c4 = fma(a, b, c4); c5 = fma(a, b, c5); c6 = fma(a, b, c6); c7 = fma(a, b, c7);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
}

__global__ void k_lds(double2* out, int iters) {
    __shared__ double2 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_double2(i, i);
    __syncthreads();
    double2 acc = make_double2(0, 0);
    unsigned idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        double2 x0 = s[(idx) & 2047], x1 = s[(idx + 256) & 2047], x2 = s[(idx + 512) & 2047], x3 = s[(idx + 768) & 2047];
        acc.x += x0.x + x1.x + x2.x + x3.x;
        idx += 32;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

// SHFL and DFMA interleaved, independent: does the shuffle unit overlap the
// FP64 pipe? (time ~ max of the two alone if so, ~ their sum if not)
__global__ void k_mix(double* out, int iters) {
    float a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
    double x = threadIdx.x, y = 1.0000001, c0 = 0.1, c1 = 0.2, c2 = 0.3, c3 = 0.4, c4 = 0.5, c5 = 0.6, c6 = 0.7, c7 = 0.8;
    for (int i = 0; i < iters; ++i) {
        a = __shfl_xor_sync(0xffffffffu, a, 1);
        c0 = fma(x, y, c0); c1 = fma(x, y, c1);
        b = __shfl_xor_sync(0xffffffffu, b, 2);
        c2 = fma(x, y, c2); c3 = fma(x, y, c3);
        c = __shfl_xor_sync(0xffffffffu, c, 4);
        c4 = fma(x, y, c4); c5 = fma(x, y, c5);
        d = __shfl_xor_sync(0xffffffffu, d, 8);
        c6 = fma(x, y, c6); c7 = fma(x, y, c7);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d + c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
}

// indexed shuffles (SHFL.IDX with a per-lane source)
__global__ void k_shfl_idx(float* out, int iters) {
    float a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
    const int src = (threadIdx.x & 31) ^ ((threadIdx.x >> 2) & 1 ? 4 : 0);
    for (int i = 0; i < iters; ++i) {
        a = __shfl_sync(0xffffffffu, a, src);
        b = __shfl_sync(0xffffffffu, b, src ^ 1);
        c = __shfl_sync(0xffffffffu, c, src ^ 2);
        d = __shfl_sync(0xffffffffu, d, src ^ 8);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}

// SHFL and LDS.128 interleaved, independent: do shuffles and shared-memory
// loads share one pipe (time ~ their sum) or overlap (~ the max)?
__global__ void k_shfl_lds(double2* out, int iters) {
    __shared__ double2 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_double2(i, i);
    __syncthreads();
    float a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
    double2 acc = make_double2(0, 0);
    unsigned idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        double2 x0 = s[(idx) & 2047], x1 = s[(idx + 256) & 2047], x2 = s[(idx + 512) & 2047], x3 = s[(idx + 768) & 2047];
        a = __shfl_xor_sync(0xffffffffu, a, 1);
        b = __shfl_xor_sync(0xffffffffu, b, 2);
        c = __shfl_xor_sync(0xffffffffu, c, 4);
        d = __shfl_xor_sync(0xffffffffu, d, 8);
        a = __shfl_xor_sync(0xffffffffu, a, 16);
        b = __shfl_xor_sync(0xffffffffu, b, 1);
        c = __shfl_xor_sync(0xffffffffu, c, 2);
        d = __shfl_xor_sync(0xffffffffu, d, 4);
        a = __shfl_xor_sync(0xffffffffu, a, 8);
        b = __shfl_xor_sync(0xffffffffu, b, 16);
        c = __shfl_xor_sync(0xffffffffu, c, 1);
        d = __shfl_xor_sync(0xffffffffu, d, 2);
        a = __shfl_xor_sync(0xffffffffu, a, 4);
        b = __shfl_xor_sync(0xffffffffu, b, 8);
        c = __shfl_xor_sync(0xffffffffu, c, 16);
        d = __shfl_xor_sync(0xffffffffu, d, 1);
        acc.x += x0.x + x1.x + x2.x + x3.x;
        idx += 32;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = make_double2(acc.x + a + b + c + d, 0);
}

template <class K, class T>
void run(const char* name, K kern, T* buf, int iters, double instr_per_iter_per_warp, int threads) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int blocks = 148 * 4;
    kern<<<blocks, threads>>>(buf, 10);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(buf, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double cycles = ms * 1e-3 * clk * 1e3;
    double warp_instr = double(blocks) * threads / 32 * iters * instr_per_iter_per_warp;
    printf("%-8s %.3f warp-instr/clk/SM (%.2f ms)\n", name, warp_instr / cycles / 148, ms);
}

int main() {
    void* buf;
    cudaMalloc(&buf, 148 * 4 * 1024 * 16);
    run("SHFL", k_shfl, (float*)buf, 20000, 4, 512);
    run("DFMA", k_dfma, (double*)buf, 20000, 8, 512);
    run("LDS.128", k_lds, (double2*)buf, 20000, 4, 256);
    run("SHFL.IDX", k_shfl_idx, (float*)buf, 20000, 4, 512);
    run("MIX", k_mix, (double*)buf, 20000, 12, 512); // 4 SHFL + 8 DFMA per iteration
    // 4 LDS.128 (16 shared cycles) + 16 SHFL per iteration: ~16 cycles if
    // they overlap, ~32 if they share the pipe (warp-instructions counted: 20)
    run("SHFL+LDS", k_shfl_lds, (double2*)buf, 20000, 20, 256);
    return 0;
}
