// swap_plan.cpp — the logical -> physical qubit map of a partitioned register
// and the eviction rule of the global<->local swaps (swap_plan.h). Pure host
// code: the runtime (runtime.cpp: QuregImpl::enqueue / run_swap) and the
// host-only C-ABI planner (qgpuPlanSwaps, tested without a GPU) share it.
#include "swap_plan.h"

#include "runtime.h"

#include <algorithm>
#include <utility>

namespace qgpu {

void SwapPlanner::reset(int flat_qubits, int local_qubits, uint64_t chunk_amps) {
    flat = flat_qubits;
    local = local_qubits;
    int lc = 0;
    while ((uint64_t{1} << lc) < chunk_amps && lc < 63) ++lc;
    // at least 5 candidates (small registers trade smaller sub-chunks)
    min_victim = std::max(0, std::min(local - 5, lc));
    l2p.resize(flat);
    p2l.resize(flat);
    for (int q = 0; q < flat; ++q) l2p[q] = p2l[q] = q;
    last_use.assign(flat, 0);
    clock = 0;
}

bool SwapPlanner::identity() const {
    for (int q = 0; q < flat; ++q)
        if (l2p[q] != q) return false;
    return true;
}

int SwapPlanner::victim(uint64_t busy, const int* need0, const int* need1, size_t nfuture, uint64_t pending) const {
    // distance to each logical qubit's next local use in the window
    std::vector<size_t> next(flat, ~size_t{0});
    for (size_t j = nfuture; j-- > 0;) {
        if (need0 && need0[j] >= 0) next[need0[j]] = j;
        if (need1 && need1[j] >= 0) next[need1[j]] = j;
    }
    int best = -1;
    size_t best_next = 0;
    bool best_pend = false;
    uint64_t best_use = 0;
    for (int v = local - 1; v >= min_victim; --v) {
        if ((busy >> v) & 1) continue;
        const int L = p2l[v];
        const size_t nx = next[L];
        const bool pend = (pending >> v) & 1;
        const uint64_t u = last_use[L];
        if (best < 0 || nx > best_next || (nx == best_next && best_pend && !pend) ||
            (nx == best_next && pend == best_pend && u < best_use)) {
            best = v;
            best_next = nx;
            best_pend = pend;
            best_use = u;
        }
    }
    if (best < 0) throw DomainError("no local qubit is free for a global<->local swap");
    return best;
}

void SwapPlanner::apply(int a, int b) {
    const int la = p2l[a], lb = p2l[b];
    p2l[a] = lb;
    p2l[b] = la;
    l2p[la] = b;
    l2p[lb] = a;
}

uint64_t SwapPlanner::phys_mask(uint64_t logical_mask) const {
    uint64_t m = 0;
    for (int q = 0; q < flat; ++q)
        if ((logical_mask >> q) & 1) m |= uint64_t{1} << l2p[q];
    return m;
}

} // namespace qgpu
