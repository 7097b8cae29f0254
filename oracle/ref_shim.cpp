// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. A C shim over the UNMODIFIED
// reference library (/root/reference/proj, compiled in place by
// oracle/Makefile into oracle/_ref/). It lets the pytest harness, smoke() and
// bench.py's cpu_baseline leg drive the reference's own code path with the
// same op records the product is checked with. Nothing in the product links
// or loads this file's output.
//
// Every entry point maps one-to-one onto a reference API:
//   ref_run_ops          -> qsim::Register + apply_controlled_gate
//                           (kernels.cpp:105-112) / apply_gate_to_density
//                           (density.cpp:85-116) / apply_dephasing
//                           (density.cpp:118-130) / apply_depolarising
//                           (density.cpp:132-145)
//   ref_run_distributed  -> partition + make_ranks + run_gate_ops +
//                           gather (distributed.cpp:31-42, 257-294, 296-388)
//   ref_random_circuit   -> generate_random_circuit (circuit.cpp:50-100)
//   ref_reductions       -> norm_squared (register.cpp:62-75), trace / purity
//                           (density.cpp:147-159)
//   ref_memory_bytes / ref_max_qubits / ref_modeled_bytes
//                        -> register.cpp:140-151, distributed.cpp:423-468
//   ref_enumerate_pairs  -> kernels.cpp:68-82
//   ref_time_ops         -> the timed gate loop (PAPER.md:339 protocol)
#include "oracle_ops.h"

#include "qsim/circuit.hpp"
#include "qsim/density.hpp"
#include "qsim/distributed.hpp"
#include "qsim/kernels.hpp"
#include "qsim/register.hpp"
#include "qsim/transport.hpp"

#include <chrono>
#include <cstring>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

enum { REF_OK = 0, REF_DOMAIN = 1, REF_RESOURCE = 2, REF_COMM = 3, REF_PARSE = 4,
       REF_OTHER = 5 };

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return REF_OK;
    } catch (const qsim::DomainError& e) {
        g_err = e.what();
        return REF_DOMAIN;
    } catch (const qsim::ResourceError& e) {
        g_err = e.what();
        return REF_RESOURCE;
    } catch (const qsim::CommError& e) {
        g_err = e.what();
        return REF_COMM;
    } catch (const qsim::ParseError& e) {
        g_err = e.what();
        return REF_PARSE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return REF_OTHER;
    }
}

qsim::GateMatrix to_matrix(const orc_op& op) {
    return qsim::GateMatrix{{op.m[0], op.m[1]},
                            {op.m[2], op.m[3]},
                            {op.m[4], op.m[5]},
                            {op.m[6], op.m[7]}};
}

std::vector<int> mask_to_controls(std::uint64_t mask) {
    std::vector<int> c;
    for (int b = 0; b < 64; ++b)
        if (mask >> b & 1) c.push_back(b);
    return c;
}

void apply_one(qsim::Register& reg, const orc_op& op, int workers) {
    const bool density = reg.kind() == qsim::RegisterKind::DensityMatrix;
    switch (op.kind) {
    case ORC_GATE:
        if (density)
            qsim::apply_gate_to_density(reg, mask_to_controls(op.ctrl_mask),
                                        op.target, to_matrix(op), workers);
        else
            qsim::apply_controlled_gate(reg, mask_to_controls(op.ctrl_mask),
                                        op.target, to_matrix(op), workers);
        break;
    case ORC_DEPHASE:
        qsim::apply_dephasing(reg, op.target, op.param, workers);
        break;
    case ORC_DEPOLARISE:
        qsim::apply_depolarising(reg, op.target, op.param, workers);
        break;
    default:
        throw qsim::DomainError("unknown op kind " + std::to_string(op.kind));
    }
}

qsim::RegisterKind kind_of(int density) {
    return density ? qsim::RegisterKind::DensityMatrix
                   : qsim::RegisterKind::StateVector;
}

} // namespace

extern "C" {

int ref_last_error(char* buf, int len) {
    if (buf && len > 0) {
        std::strncpy(buf, g_err.c_str(), static_cast<std::size_t>(len - 1));
        buf[len - 1] = 0;
    }
    return static_cast<int>(g_err.size());
}

unsigned long long ref_kernel_invocations(void) {
    return qsim::detail::kernel_invocations();
}

// Build a register (zero state, or `init` = interleaved re/im when non-null),
// apply `ops` in order, write the final amplitudes to `out` (may be null).
int ref_run_ops(int num_qubits, int density, const double* init, int nops,
                const orc_op* ops, int workers, double* out) {
    return guarded([&] {
        qsim::Register reg(num_qubits, kind_of(density));
        if (init)
            std::memcpy(reg.amps().data64(), init, reg.amps().byte_size());
        for (int i = 0; i < nops; ++i)
            apply_one(reg, ops[i], workers);
        if (out)
            std::memcpy(out, reg.amps().data64(), reg.amps().byte_size());
    });
}

// The same in the reference's single precision (Precision::Single: complex
// float amplitudes, Mat2<float>); `out` receives interleaved floats.
int ref_run_ops_single(int num_qubits, int density, int nops, const orc_op* ops, int workers,
                       float* out) {
    return guarded([&] {
        qsim::Register reg(num_qubits, kind_of(density), qsim::Precision::Single);
        for (int i = 0; i < nops; ++i)
            apply_one(reg, ops[i], workers);
        if (out)
            std::memcpy(out, reg.amps().data32(), reg.amps().byte_size());
    });
}

// Per-op counter of core-kernel entries (kernels.cpp:15-20, 47).
int ref_count_kernel_calls(int num_qubits, int density, const orc_op* op,
                           unsigned long long* calls) {
    return guarded([&] {
        qsim::Register reg(num_qubits, kind_of(density));
        const auto before = qsim::detail::kernel_invocations();
        apply_one(reg, *op, 1);
        *calls = qsim::detail::kernel_invocations() - before;
    });
}

// get_amplitude / set_amplitude boundary semantics (register.cpp:31-53).
int ref_set_get(int num_qubits, int density, unsigned long long index, double re,
                double im, double* out_re, double* out_im) {
    return guarded([&] {
        qsim::Register reg(num_qubits, kind_of(density));
        reg.set_amplitude(index, {re, im});
        const auto a = reg.get_amplitude(index);
        *out_re = a.real();
        *out_im = a.imag();
    });
}

int ref_reductions(int num_qubits, int density, const double* amps,
                   double* norm, double* trace_re, double* trace_im,
                   double* purity) {
    return guarded([&] {
        qsim::Register reg(num_qubits, kind_of(density));
        std::memcpy(reg.amps().data64(), amps, reg.amps().byte_size());
        *norm = reg.norm_squared();
        if (density) {
            const auto t = qsim::trace(reg);
            *trace_re = t.real();
            *trace_im = t.imag();
            *purity = qsim::purity(reg);
        }
    });
}

// Distributed engine: plan (n_flat, k, strategy, block), run `ops` lowered
// exactly as flatten_circuit does (distributed.cpp:93-109), gather.
int ref_run_distributed(int num_qubits, int density, int k, int strategy,
                        unsigned long long block_amps, int nops,
                        const orc_op* ops, int workers, double* out,
                        unsigned long long* msgs_per_rank,
                        unsigned long long* bytes_per_rank,
                        unsigned int* rounds_per_flat_op, int* n_flat_ops) {
    return guarded([&] {
        const int flat = density ? 2 * num_qubits : num_qubits;
        auto plan = qsim::partition(flat, k, static_cast<qsim::Strategy>(strategy));
        plan.block_amps = block_amps;
        std::vector<qsim::FlatGateOp> flat_ops;
        for (int i = 0; i < nops; ++i) {
            if (ops[i].kind != ORC_GATE)
                throw qsim::DomainError("distributed engine runs gates only");
            const auto controls = mask_to_controls(ops[i].ctrl_mask);
            const std::uint64_t mask =
                qsim::detail::make_control_mask(flat, controls, ops[i].target);
            const auto g = to_matrix(ops[i]);
            flat_ops.push_back({mask, ops[i].target, g});
            if (density)
                flat_ops.push_back({mask << num_qubits,
                                    ops[i].target + num_qubits, g.conjugate()});
        }
        auto ranks = qsim::make_ranks(plan, qsim::Precision::Double);
        qsim::InProcessTransport transport(plan.rank_count());
        const auto stats = qsim::run_gate_ops(ranks, plan, flat_ops, transport,
                                              workers);
        const auto reg = qsim::gather(ranks, plan, kind_of(density));
        if (out)
            std::memcpy(out, reg.amps().data64(), reg.amps().byte_size());
        for (int r = 0; r < plan.rank_count(); ++r) {
            if (msgs_per_rank) msgs_per_rank[r] = stats.messages_sent[r];
            if (bytes_per_rank) bytes_per_rank[r] = stats.bytes_sent[r];
        }
        if (rounds_per_flat_op)
            for (std::size_t i = 0; i < stats.exchange_rounds.size(); ++i)
                rounds_per_flat_op[i] = stats.exchange_rounds[i];
        if (n_flat_ops) *n_flat_ops = static_cast<int>(flat_ops.size());
    });
}

// Reference random-circuit generator; writes up to max_ops op records and
// the gate kind (qsim::Gate enum value) of each into names.
int ref_random_circuit(int num_qubits, int depth, unsigned long long seed,
                       int max_ops, orc_op* out, int* names, int* n_out) {
    return guarded([&] {
        const auto c = qsim::generate_random_circuit(
            {num_qubits, depth, seed, qsim::Topology::Linear});
        if (static_cast<int>(c.ops.size()) > max_ops)
            throw qsim::DomainError("output buffer too small");
        for (std::size_t i = 0; i < c.ops.size(); ++i) {
            const auto& op = c.ops[i];
            const auto g = qsim::gate_matrix(op.gate);
            orc_op r{};
            r.kind = ORC_GATE;
            r.target = op.target;
            for (int cq : op.controls) r.ctrl_mask |= std::uint64_t{1} << cq;
            const qsim::Amp e[4] = {g.m00, g.m01, g.m10, g.m11};
            for (int j = 0; j < 4; ++j) {
                r.m[2 * j] = e[j].real();
                r.m[2 * j + 1] = e[j].imag();
            }
            out[i] = r;
            if (names) names[i] = static_cast<int>(op.gate.gate);
        }
        *n_out = static_cast<int>(c.ops.size());
    });
}

// Named-gate matrices (gates.cpp:51-98), for the harness's gate table.
int ref_gate_matrix(int gate, double angle, double* m8) {
    return guarded([&] {
        const auto g = qsim::gate_matrix({static_cast<qsim::Gate>(gate), angle});
        const qsim::Amp e[4] = {g.m00, g.m01, g.m10, g.m11};
        for (int j = 0; j < 4; ++j) {
            m8[2 * j] = e[j].real();
            m8[2 * j + 1] = e[j].imag();
        }
    });
}

int ref_rotation_matrix(double nx, double ny, double nz, double angle, double* m8) {
    return guarded([&] {
        const auto g = qsim::rotation_matrix({nx, ny, nz}, angle);
        const qsim::Amp e[4] = {g.m00, g.m01, g.m10, g.m11};
        for (int j = 0; j < 4; ++j) {
            m8[2 * j] = e[j].real();
            m8[2 * j + 1] = e[j].imag();
        }
    });
}

int ref_is_unitary(const double* m8, double tol, int* out) {
    return guarded([&] {
        const qsim::GateMatrix g{{m8[0], m8[1]}, {m8[2], m8[3]},
                                 {m8[4], m8[5]}, {m8[6], m8[7]}};
        *out = qsim::is_unitary(g, tol) ? 1 : 0;
    });
}

int ref_memory_bytes(int num_qubits, int density, int single,
                     unsigned long long* out) {
    return guarded([&] {
        *out = qsim::memory_bytes(num_qubits, kind_of(density),
                                  single ? qsim::Precision::Single
                                         : qsim::Precision::Double);
    });
}

int ref_modeled_bytes(int num_qubits, int k, int strategy, int single,
                      unsigned long long block, unsigned long long* out) {
    return guarded([&] {
        *out = qsim::modeled_bytes_per_rank(
            num_qubits, k, static_cast<qsim::Strategy>(strategy),
            single ? qsim::Precision::Single : qsim::Precision::Double, block);
    });
}

int ref_max_qubits(unsigned long long node_bytes, unsigned long long overhead,
                   int strategy, int single, int k, int* out) {
    return guarded([&] {
        qsim::MemoryModel m;
        m.node_bytes = node_bytes;
        m.overhead_bytes = overhead;
        m.strategy = static_cast<qsim::Strategy>(strategy);
        m.precision = single ? qsim::Precision::Single : qsim::Precision::Double;
        *out = qsim::max_qubits(m, k);
    });
}

int ref_partition_info(int n, int k, int target, int rank, int* needs_comm,
                       int* peer) {
    return guarded([&] {
        const auto plan = qsim::partition(n, k, qsim::Strategy::FullClone);
        *needs_comm = qsim::needs_communication(plan, target) ? 1 : 0;
        *peer = *needs_comm ? qsim::pair_rank(plan, rank, target) : -1;
    });
}

int ref_enumerate_pairs(int n, int target, unsigned long long* out_lo_hi) {
    return guarded([&] {
        const auto p = qsim::enumerate_pairs(n, target);
        for (std::size_t i = 0; i < p.size(); ++i) {
            out_lo_hi[2 * i] = p[i].lo;
            out_lo_hi[2 * i + 1] = p[i].hi;
        }
    });
}

// CPU baseline timer: allocation + init are outside the clock (PAPER.md:339,
// SPEC.md:499-507); returns seconds of the op loop for each of `reps` reps.
int ref_time_ops_prec(int num_qubits, int density, int single, int nops, const orc_op* ops,
                      int workers, int reps, double* seconds) {
    return guarded([&] {
        qsim::Register reg(num_qubits, kind_of(density),
                           single ? qsim::Precision::Single : qsim::Precision::Double);
        for (int r = 0; r < reps; ++r) {
            reg.init_zero_state();
            const auto t0 = std::chrono::steady_clock::now();
            for (int i = 0; i < nops; ++i)
                apply_one(reg, ops[i], workers);
            const auto t1 = std::chrono::steady_clock::now();
            seconds[r] = std::chrono::duration<double>(t1 - t0).count();
        }
    });
}

int ref_time_ops(int num_qubits, int density, int nops, const orc_op* ops,
                 int workers, int reps, double* seconds) {
    return ref_time_ops_prec(num_qubits, density, 0, nops, ops, workers, reps, seconds);
}

// Text format (circuit.cpp:123-237): parse `text` with the reference parser
// and write serialize() of the result to `out` (NUL-terminated; *len = its
// length). A parse error returns REF_PARSE with the reference's message
// ("line N: ...") in ref_last_error.
int ref_parse_serialize(const char* text, char* out, int cap, int* len) {
    return guarded([&] {
        const std::string s = qsim::serialize(qsim::parse(text));
        *len = static_cast<int>(s.size());
        if (static_cast<int>(s.size()) + 1 > cap)
            throw qsim::DomainError("output buffer too small");
        std::memcpy(out, s.c_str(), s.size() + 1);
    });
}

// serialize(generate_random_circuit(...)) (circuit.cpp:50-100, 123-136).
int ref_serialize_random(int num_qubits, int depth, unsigned long long seed, char* out, int cap,
                         int* len) {
    return guarded([&] {
        const std::string s = qsim::serialize(
            qsim::generate_random_circuit({num_qubits, depth, seed, qsim::Topology::Linear}));
        *len = static_cast<int>(s.size());
        if (static_cast<int>(s.size()) + 1 > cap)
            throw qsim::DomainError("output buffer too small");
        std::memcpy(out, s.c_str(), s.size() + 1);
    });
}

// Distributed CPU baseline: the reference's own
// run_gate_ops over InProcessTransport with one thread per rank, timed by
// the reference itself (gate_seconds: clock started once all ranks are
// ready, stopped after the final global barrier, distributed.cpp:323-352).
// Allocation and zero-init are outside the clock; `reps` repetitions.
int ref_time_distributed(int num_qubits, int k, int strategy, int nops, const orc_op* ops, int workers,
                         int reps, double* seconds, unsigned long long* bytes_sent) {
    return guarded([&] {
        auto plan = qsim::partition(num_qubits, k, static_cast<qsim::Strategy>(strategy));
        std::vector<qsim::FlatGateOp> flat_ops;
        for (int i = 0; i < nops; ++i) {
            if (ops[i].kind != ORC_GATE) throw qsim::DomainError("distributed engine runs gates only");
            const auto controls = mask_to_controls(ops[i].ctrl_mask);
            flat_ops.push_back({qsim::detail::make_control_mask(num_qubits, controls, ops[i].target),
                                ops[i].target, to_matrix(ops[i])});
        }
        auto ranks = qsim::make_ranks(plan, qsim::Precision::Double);
        qsim::InProcessTransport transport(plan.rank_count());
        for (int r = 0; r < reps; ++r) {
            qsim::init_ranks_zero(ranks);
            double secs = 0.0;
            const auto stats = qsim::run_gate_ops(ranks, plan, flat_ops, transport, workers, nullptr, &secs);
            seconds[r] = secs;
            if (bytes_sent) *bytes_sent = stats.total_bytes();
        }
    });
}

} // extern "C"
