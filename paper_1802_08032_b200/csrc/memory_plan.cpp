// memory_plan.cpp — the memory model of the partitioned register, re-targeted
// at HBM.
//
// Two models:
//  * the reference's node model, restated exactly so parity is checkable:
//    modeled_bytes_per_rank / max_qubits (distributed.cpp:423-468,
//    distributed.hpp:145-162): per-rank partition bytes times the exchange
//    strategy's factor (FullClone 2x, HalfExchange 1.5x, PerAmplitude
//    1x + block), and the largest n that fits node_bytes - overhead;
//  * the device model of this runtime: what create_register and the
//    exchange engine actually cudaMalloc per rank — the partition
//    (16 B x 2^(n-k)), two exchange sub-chunk buffers once k > 0 (the
//    double-buffered PerAmplitude strategy with block = chunk,
//    runtime.cpp: exchange_rounds) and the reduction scratch. It sizes
//    registers for the 180 GB of a B200: 33 state-vector qubits on one GPU,
//    36 on eight.
#include "qgpu_kernels.h"
#include "runtime.h"

#include <algorithm>
#include <string>

namespace qgpu {

namespace {

using u128 = unsigned __int128;

u128 modeled_bytes_128(int n, int k, int strategy, bool single, uint64_t block) {
    const u128 local = u128{1} << (n - k);
    const u128 ab = single ? 8 : 16; // std::complex<float> / <double> (types.hpp:12)
    switch (strategy) {
    case 0: return ab * local * 2;               // FullClone
    case 1: return ab * local + ab * (local / 2); // HalfExchange
    case 2: return ab * (local + block);          // PerAmplitude
    }
    return 0;
}

} // namespace

uint64_t modeled_bytes_per_rank(int n, int k, int strategy, bool single, uint64_t block) {
    if (n < 1 || k < 0 || k > n) throw DomainError("invalid qubit/rank combination");
    if (strategy < 0 || strategy > 2)
        throw DomainError("unknown strategy " + std::to_string(strategy));
    const u128 b = modeled_bytes_128(n, k, strategy, single, block);
    if (b > ~uint64_t{0}) throw DomainError("modeled byte count overflows 64 bits");
    return static_cast<uint64_t>(b);
}

int max_qubits(uint64_t node_bytes, uint64_t overhead, int strategy, bool single, int k) {
    if (k < 0) throw DomainError("rank count exponent must be non-negative");
    if (strategy < 0 || strategy > 2)
        throw DomainError("unknown strategy " + std::to_string(strategy));
    if (node_bytes <= overhead) return 0;
    const u128 budget = node_bytes - overhead;
    const int min_local = strategy == 1 ? 1 : 0;
    int best = 0;
    for (int n = std::max(1, k + min_local); n <= k + 80; ++n) {
        if (modeled_bytes_128(n, k, strategy, single, 1) <= budget)
            best = n;
        else
            break;
    }
    return best;
}

uint64_t device_bytes_per_rank(int flat, int k, uint64_t chunk_amps, bool single) {
    if (flat < 1 || k < 0 || k > flat || flat - k > 58)
        throw DomainError("invalid qubit/rank combination");
    const uint64_t local = uint64_t{1} << (flat - k);
    const uint64_t amp = single ? sizeof(float2) : sizeof(double2);
    uint64_t bytes = local * amp;
    if (k > 0) bytes += 2 * std::min(local, std::max<uint64_t>(chunk_amps, 1)) * amp;
    bytes += (kReduceBlocks + (uint64_t{1} << k) + 1) * sizeof(double2);
    return bytes;
}

int device_max_qubits(uint64_t device_bytes, int k, uint64_t chunk_amps, bool density, bool single) {
    if (k < 0 || k > 30) throw DomainError("rank count exponent must be in [0, 30]");
    int best = 0;
    for (int N = 1; N <= 58; ++N) {
        const int flat = density ? 2 * N : N;
        if (flat < k || flat - k > 58) {
            if (flat - k > 58) break;
            continue;
        }
        if (density && k > N) continue;
        if (device_bytes_per_rank(flat, k, chunk_amps, single) <= device_bytes)
            best = N;
        else
            break;
    }
    return best;
}

} // namespace qgpu
