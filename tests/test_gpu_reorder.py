"""The library's default op ordering on the GPU: commutation-aware pass
scheduling (runtime.cpp `window_pass`, Env ordering 1).

Ops that commute are scheduled out of circuit order into fewer HBM passes,
so amplitudes equal the reference's up to rounding only. The bar is the
north star's: max-abs amplitude error <= 1e-12 against the reference (the
compiled reference where it is cheap, else its C restatement — both pinned
bit for bit to each other in tests/test_oracle.py), reductions within 1e-12,
single precision within 1e-5 of the double-precision reference. Every test
also checks that the schedule really was reordered (fewer passes than in
circuit order) where the circuit allows it.
"""
import os

import numpy as np
import pytest

import oracle
from paper_1802_08032_b200 import circuits as C
from paper_1802_08032_b200 import quest
from tests.harness import oracle_run, random_gate_circuit, to_oracle_ops

pytestmark = pytest.mark.gpu

TOL = 1e-12
WORKERS = os.cpu_count() or 1


def make_env(reorder=True, window=0, loopback=0):
    e = quest.Env.loopback(loopback) if loopback else quest.Env()
    e.set_ordering(reorder, window)
    return e


@pytest.fixture(scope="module")
def env():
    e = make_env()
    yield e
    e.destroy()


def run(env, circuit, density=False, init=None, precision="double"):
    q = quest.QuregHandle(env, circuit.num_qubits, density, precision=precision)
    try:
        if init is not None:
            q.set_state(init)
        C.apply_circuit(q, circuit)
        q.flush()
        return q.state(), q.pass_count()
    finally:
        q.destroy()


def max_err(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) if np.size(a) else 0.0


def test_default_ordering_is_reorder():
    e = quest.Env()
    try:
        e.set_ordering(True)  # conftest pins QGPU_ORDER=exact for the bit-exact suites
        assert e.reorder
        e.set_ordering(False)
        assert not e.reorder
    finally:
        e.destroy()


@pytest.mark.parametrize("n", [12, 14, 16, 20])
@pytest.mark.parametrize("window", [0, 48])
def test_random_gates(env, n, window):
    env.set_ordering(True, window or 512)
    try:
        c = random_gate_circuit(n, 400, seed=100 + n, max_controls=3)
        got, _ = run(env, c)
        assert max_err(got, oracle_run(c)) <= TOL
    finally:
        env.set_ordering(True, 512)


@pytest.mark.parametrize("n", [13, 17])
def test_random_state_in(env, n):
    rng = np.random.default_rng(n)
    init = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    init /= np.linalg.norm(init)
    c = random_gate_circuit(n, 300, seed=7 + n, max_controls=4)
    got, _ = run(env, c, init=init)
    assert max_err(got, oracle_run(c, init=init)) <= TOL


def test_layered_c1_against_reference_fewer_passes(env):
    """Config C1 (20 qubits, depth 20, seed 12345) vs the compiled reference;
    the reordered schedule needs at most a third of circuit order's passes."""
    c = C.layered_random_circuit(20, 20, 12345)
    want = oracle.ref_run(20, to_oracle_ops(c), workers=8) if oracle.ref_available() else oracle_run(c)
    got, passes = run(env, c)
    assert max_err(got, want) <= TOL
    ex = make_env(reorder=False)
    try:
        got_ex, passes_ex = run(ex, c)
    finally:
        ex.destroy()
    assert np.array_equal(got_ex, want) or not oracle.ref_available()
    assert passes * 3 <= passes_ex, (passes, passes_ex)


def test_qft_and_reference_generator(env):
    for c in (C.qft_circuit(18, mcpf_every=3), C.reference_random_circuit(18, 30, 2)):
        got, _ = run(env, c)
        assert max_err(got, oracle_run(c)) <= TOL


@pytest.mark.parametrize("N", [6, 7])
def test_density_matrix_with_channels(env, N):
    """Density matrices (2N >= 12 flat qubits: tile passes) with dephasing and
    depolarising channels between the gates."""
    c = random_gate_circuit(N, 250, seed=300 + N, max_controls=2, channels=True)
    got, _ = run(env, c, density=True)
    assert max_err(got, oracle_run(c, density=True)) <= TOL


@pytest.mark.slow
@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")
def test_density_c4_noisy_layered_against_reference(env):
    """Config C4 (14-qubit density matrix, noisy layered circuit)."""
    c = C.layered_random_circuit(14, 10, 12345, noise_pmax=0.05)
    want = oracle.ref_run(14, to_oracle_ops(c), density=True, workers=WORKERS)
    got, _ = run(env, c, density=True)
    assert max_err(got, want) <= TOL


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("swaps", [False, True])
def test_loopback_ranks(k, swaps):
    """2^k virtual ranks (16 - k >= 13 local qubits, tile passes): exchange
    gates and qubit swaps drain the window in order around them."""
    n = 16
    c = random_gate_circuit(n, 300, seed=500 + k, max_controls=2)
    want = oracle_run(c)
    e = make_env(loopback=1 << k)
    try:
        e.set_qubit_swaps(swaps)
        e.set_exchange_chunk(1 << 10)
        q = quest.QuregHandle(e, n)
        try:
            C.apply_circuit(q, c)
            for t in (0, 7, n - 1):
                assert abs(q.calcProbOfOutcome(t, 1) - oracle.orc_prob_of_outcome(want, n, t, 1)) <= TOL
            assert max_err(q.state(), want) <= TOL
        finally:
            q.destroy()
    finally:
        e.destroy()


@pytest.mark.parametrize("k", [1, 3])
def test_loopback_lightcone_drain(k):
    """Qubit swaps in the default ordering go through the light-cone drain
    (runtime.cpp drain_lightcone: ops that can run with the local qubits go
    first, global qubits are swapped in only when nothing can): a layered
    circuit (every qubit touched per layer) and a noisy density matrix
    (depolarising needs both of its qubits local) on 2^k virtual ranks,
    within 1e-12 of the oracle (the swap counts: tests/test_distributed_gloo.py)."""
    n = 17
    c = C.layered_random_circuit(n, 12, 12345)
    want = oracle_run(c)
    e = make_env(loopback=1 << k)
    try:
        e.set_qubit_swaps(True)
        q = quest.QuregHandle(e, n)
        try:
            C.apply_circuit(q, c)
            assert max_err(q.state(), want) <= TOL
        finally:
            q.destroy()
        d = C.layered_random_circuit(7, 4, 8, noise_pmax=0.1)
        dw = oracle_run(d, density=True)
        qd = quest.QuregHandle(e, 7, True)
        try:
            C.apply_circuit(qd, d)
            assert max_err(qd.state(), dw) <= TOL
        finally:
            qd.destroy()
    finally:
        e.destroy()


def test_measurement_and_collapse(env):
    n = 16
    c = random_gate_circuit(n, 200, seed=77, max_controls=2)
    want = oracle_run(c)
    q = quest.QuregHandle(env, n)
    try:
        C.apply_circuit(q, c)
        for t in range(n):
            assert abs(q.calcProbOfOutcome(t, 0) - oracle.orc_prob_of_outcome(want, n, t, 0)) <= TOL
        p = oracle.orc_prob_of_outcome(want, n, 3, 1)
        q.collapseToOutcome(3, 1)
        want = oracle.orc_collapse(want, n, 3, 1, p)
        C.apply_circuit(q, c)  # collapse, then more gates: the collapse sits in the window
        want = oracle_run(c, init=want)
        assert max_err(q.state(), want) <= TOL
        assert abs(q.calcTotalProb() - 1.0) <= 1e-12
    finally:
        q.destroy()


@pytest.mark.parametrize("n", [14, 20])
def test_jit_equals_interpreter(monkeypatch, n):
    """The same reordered schedule through the JIT kernels and the
    interpreter: bit-identical to each other (same handlers, same order).
    The phase limit is pinned: by default the interpreter cuts passes at two
    phases and the JIT at three, which schedules differently."""
    monkeypatch.setenv("QGPU_TILE_PHASES", "3")
    e = make_env()
    try:
        c = random_gate_circuit(n, 300, seed=900 + n, max_controls=3)
        out = {}
        for mode in (2, 0):
            quest.set_jit(mode)
            try:
                out[mode], _ = run(e, c)
            finally:
                quest.set_jit(1)
    finally:
        e.destroy()
    assert np.array_equal(out[2], out[0])
    assert max_err(out[2], oracle_run(c)) <= TOL


def test_single_precision(env):
    n = 18
    c = C.layered_random_circuit(n, 12, 4)
    got, _ = run(env, c, precision="single")
    assert max_err(got, oracle_run(c)) <= 1e-5


@pytest.mark.slow
@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")
def test_30q_bench_circuit_against_reference(env):
    """C2, the bench's workload in the default ordering: all 2^30 amplitudes
    within 1e-12 of the compiled reference (every pass shape JIT-compiled,
    as timed by bench.py), in at most 21 passes (circuit order: 66)."""
    n = 30
    c = C.layered_random_circuit(n, 20, 12345)
    want = oracle.ref_run(n, to_oracle_ops(c), workers=WORKERS)
    quest.set_jit(2)
    try:
        q = quest.QuregHandle(env, n)
        try:
            C.apply_circuit(q, c)
            q.flush()
            assert q.pass_count() <= 21
            err = 0.0
            chunk = 1 << 26
            for s in range(0, 1 << n, chunk):
                err = max(err, max_err(q.state(s, chunk), want[s:s + chunk]))
            assert err <= TOL, err
        finally:
            q.destroy()
    finally:
        quest.set_jit(1)


def test_scale_folding_paths(env):
    """Unit-coefficient normalization factors scalars out of uncontrolled
    H / Rx / Ry / Rz gates; they must be applied exactly once whatever the
    pass holds: a circuit whose last passes contain only controlled gates
    (the scalar is appended as its own elementwise op), a read in the middle
    (the window drains), and a register re-initialised with scalars pending."""
    n = 14
    c = C.Circuit(n, 0, [C.GateOp("H", q) for q in range(n)])
    c.ops += [C.GateOp("RX", q, angle=0.3 + q) for q in range(n)]
    c.ops += [C.GateOp("RZ", q, angle=1.1 * q) for q in range(n)]
    c.ops += [C.GateOp("X", (q + 1) % n, (q,)) for q in range(n)]
    c.ops += [C.GateOp("PHASE", q, ((q + 3) % n,), angle=0.7) for q in range(n)]
    want = oracle_run(c)
    q = quest.QuregHandle(env, n)
    try:
        C.apply_circuit(q, c)
        assert max_err(q.state(), want) <= TOL
        assert abs(q.calcTotalProb() - 1.0) <= 1e-12
        # gates, then a re-init: pending scalars are dropped with the ops
        C.apply_circuit(q, c)
        q.initZeroState()
        C.apply_circuit(q, c)
        assert max_err(q.state(), want) <= TOL
    finally:
        q.destroy()


@pytest.mark.parametrize("angle", [0.0, np.pi, np.pi / 2, 1e-300, np.pi - 1e-15])
def test_normalization_edge_angles(env, angle):
    """Rotations whose sine or cosine is zero or tiny (the pivot is the
    larger of the two, so the factored matrix stays bounded)."""
    n = 13
    c = C.Circuit(n, 0, [C.GateOp("H", q) for q in range(n)])
    for name in ("RX", "RY", "RZ", "PHASE"):
        c.ops += [C.GateOp(name, q, angle=angle * (1 + (q % 2))) for q in range(n)]
    got, _ = run(env, c)
    assert max_err(got, oracle_run(c)) <= TOL
