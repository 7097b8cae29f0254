// swap_plan.h — global<->local qubit swaps.
//
// The reference exchanges a whole partition for EVERY gate whose target is a
// global (rank-bit) qubit (distributed.cpp:167-231: 16 B x 2^(n-k) each way
// per gate). Here a gate on a global qubit instead swaps that qubit with a
// local one: each rank trades the half of its partition whose local bit v
// differs from its rank bit with its partner (half the bytes of one
// exchange gate, pure copies), after which the qubit is local and every
// following gate on it runs in the fused HBM passes. The runtime keeps the
// logical -> physical qubit map; swaps only move amplitudes, so every gate
// still evaluates the reference's fma chain on the same amplitude pairs and
// results stay bit-identical.
//
// Victim choice (Belady): the runtime buffers up to kSwapWindow logical ops
// (the C-ABI is asynchronous until a value is read) and evicts the local
// position whose logical qubit is next needed locally furthest ahead in that
// window; ties go to the least recently used, then the highest position.
// Candidates are positions v with 2^v >= the exchange sub-chunk, so each
// transferred sub-chunk is contiguous (at least the top five local positions
// on small registers). LRU alone thrashes on layered circuits, which touch
// every qubit once per layer.
#pragma once

#include <cstdint>
#include <vector>

namespace qgpu {

constexpr size_t kSwapWindow = 256; // logical ops buffered for lookahead

struct SwapPlanner {
    int flat = 0;       // qubits of the flat vector
    int local = 0;      // local (per-rank) qubits
    int min_victim = 0; // lowest eligible local position
    std::vector<int> l2p, p2l;
    std::vector<uint64_t> last_use; // per logical qubit
    uint64_t clock = 0;

    void reset(int flat_qubits, int local_qubits, uint64_t chunk_amps);
    bool identity() const;
    void touch(int logical) { last_use[logical] = ++clock; }
    // local physical position to trade for a global one; `busy` = physical
    // positions the current op needs local (never evicted); need0/need1[j] =
    // logical qubits future op j needs local (-1: none), j < nfuture
    // `pending` = physical positions with ops still waiting in the pass
    // window (a victim among those forces them to run first): preferred
    // against on equal lookahead distance
    int victim(uint64_t busy, const int* need0 = nullptr, const int* need1 = nullptr,
               size_t nfuture = 0, uint64_t pending = 0) const;
    // swap the logical qubits at physical positions a and b
    void apply(int a, int b);
    int phys(int logical) const { return logical < 0 ? logical : l2p[logical]; }
    uint64_t phys_mask(uint64_t logical_mask) const;
};

} // namespace qgpu
