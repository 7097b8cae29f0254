"""Parity of the CUDA product (through the C-ABI) with the CPU checkers.

Bar: bit-identical amplitudes (np.array_equal, i.e. up to the sign of zero)
for every gate / channel path, since the kernels evaluate the reference's own
fma chain; reductions within 1e-12 (compensated sums in a different order).
"""
import math

import numpy as np
import pytest

import oracle
from paper_1802_08032_b200 import circuits as C
from paper_1802_08032_b200 import quest
from tests.harness import bits_equal, oracle_run, random_gate_circuit, to_oracle_ops

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def env():
    e = quest.Env()
    yield e
    e.destroy()


def run_product(env, circuit, density=False, init=None):
    q = quest.QuregHandle(env, circuit.num_qubits, density)
    try:
        if init is not None:
            q.set_state(init)
        C.apply_circuit(q, circuit)
        return q.state()
    finally:
        q.destroy()


def assert_parity(got, want):
    err = float(np.max(np.abs(got - want))) if got.size else 0.0
    assert err <= TOL, f"max-abs error {err}"
    assert bits_equal(got, want), f"not bit-identical (max-abs {err})"


FUSION = [(0, 48, 4), (0, 48, 3), (0, 48, 5), (0, 7, 2), (1, 0, 4), (2, 0, 0)]


@pytest.mark.parametrize("mode,max_ops,h", FUSION)
@pytest.mark.parametrize("n", [4, 7, 12])
def test_random_gates_all_fusion_modes(env, mode, max_ops, h, n):
    env.set_fusion(mode, max_ops if max_ops else 48, h if h else 4)
    try:
        c = random_gate_circuit(n, 150, seed=n * 31 + mode, max_controls=3)
        assert_parity(run_product(env, c), oracle_run(c))
    finally:
        env.set_fusion(0, 48, 4)


@pytest.mark.parametrize("n", [6, 11, 16])
def test_random_gates_from_random_state(env, n):
    rng = np.random.default_rng(n)
    init = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    c = random_gate_circuit(n, 200, seed=7 + n, max_controls=4)
    assert_parity(run_product(env, c, init=init), oracle_run(c, init=init))


def test_layered_circuit_c1_against_reference(env):
    """Config C1: 20 qubits, depth 20, seed 12345, vs the compiled reference."""
    c = C.layered_random_circuit(20, 20, 12345)
    want = oracle.ref_run(20, to_oracle_ops(c), workers=8) if oracle.ref_available() else oracle_run(c)
    assert_parity(run_product(env, c), want)


def test_reference_generator_circuit(env):
    c = C.reference_random_circuit(18, 30, 2)
    assert_parity(run_product(env, c), oracle_run(c))


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("N", [2, 4, 6])
def test_density_matrix_with_channels(env, mode, N):
    env.set_fusion(mode, 48, 4)
    try:
        c = random_gate_circuit(N, 120, seed=500 + N, max_controls=2, channels=True)
        assert_parity(run_product(env, c, density=True), oracle_run(c, density=True))
    finally:
        env.set_fusion(0, 48, 4)


def test_density_c4_noisy_layered(env):
    c = C.layered_random_circuit(7, 6, 99, noise_pmax=0.1)
    assert_parity(run_product(env, c, density=True), oracle_run(c, density=True))


@pytest.mark.parametrize("n", [5, 9, 14])
def test_every_target_and_control_placement(env, n):
    """Per-target sweep (SURVEY.md §8(d) C2 sweep) over every stride, with
    controls below / above the target."""
    c = C.Circuit(n, 0, [])
    rng = np.random.default_rng(n)
    for t in range(n):
        for name in ("H", "RX", "RY", "RZ", "PHASE", "X", "SX"):
            c.ops.append(C.GateOp(name, t, (), angle=float(rng.uniform(0, 6))))
        for cq in range(n):
            if cq != t:
                c.ops.append(C.GateOp("X", t, (cq,)))
                c.ops.append(C.GateOp("PHASE", t, (cq,), angle=float(rng.uniform(0, 6))))
    assert_parity(run_product(env, c), oracle_run(c))


def test_reductions(env):
    n = 13
    c = random_gate_circuit(n, 80, seed=3)
    want = oracle_run(c)
    q = quest.QuregHandle(env, n)
    C.apply_circuit(q, c)
    assert abs(q.calcTotalProb() - oracle.orc_norm_kahan(want)) < TOL
    for t in range(n):
        for o in (0, 1):
            assert abs(q.calcProbOfOutcome(t, o) - oracle.orc_prob_of_outcome(want, n, t, o)) < TOL
    q.destroy()
    N = 4
    c = random_gate_circuit(N, 60, seed=4, channels=True)
    want = oracle_run(c, density=True)
    q = quest.QuregHandle(env, N, density=True)
    C.apply_circuit(q, c)
    assert abs(q.calcTotalProb() - oracle.orc_trace(want, N).real) < TOL
    assert abs(q.calcPurity() - oracle.orc_norm_kahan(want)) < TOL
    for t in range(N):
        assert abs(q.calcProbOfOutcome(t, 1) - oracle.orc_prob_of_outcome(want, N, t, 1, density=True)) < TOL
    tr = quest.call("qgpuTrace", q.h)
    assert abs(complex(tr.real, tr.imag) - oracle.orc_trace(want, N)) < TOL
    q.destroy()


@pytest.mark.parametrize("density", [False, True])
def test_collapse_and_measure_match_restatement(env, density):
    n = 5 if density else 10
    c = random_gate_circuit(n, 60, seed=11)
    amps = oracle_run(c, density=density)
    q = quest.QuregHandle(env, n, density)
    C.apply_circuit(q, c)
    p = q.collapseToOutcome(2, 1)
    want_p = oracle.orc_prob_of_outcome(amps, n, 2, 1, density)
    assert abs(p - want_p) < TOL
    amps = oracle.orc_collapse(amps, n, 2, 1, p, density)
    got = q.state()
    assert np.max(np.abs(got - amps)) < TOL
    # measurement outcomes under a fixed seed match the restatement exactly
    env.seed(12345)
    st = oracle.orc_seed([12345])
    for t in (0, 3, 4):
        o = q.measure(t)
        ow, pw, amps, st = oracle.orc_measure(amps, n, t, st, density)
        assert o == ow
    assert np.max(np.abs(q.state() - amps)) < TOL
    q.destroy()


def test_qft_probabilities(env):
    """C5 analytic KAT: P(outcome) = 1/2 on every qubit after QFT of |x>."""
    n = 16
    q = quest.QuregHandle(env, n)
    q.initClassicalState(12345)
    C.apply_circuit(q, C.qft_circuit(n, mcpf_every=3))
    for t in range(n):
        assert abs(q.calcProbOfOutcome(t, 0) - 0.5) < TOL
    assert abs(q.calcTotalProb() - 1.0) < TOL
    q.destroy()


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("density", [False, True])
def test_loopback_distributed_equals_single(k, density):
    """2^k virtual ranks on one GPU through the sub-chunked exchange protocol
    == the single-rank result (acceptance 3)."""
    n = 4 if density else 11
    c = random_gate_circuit(n, 120, seed=40 + k, max_controls=2, channels=density)
    want = oracle_run(c, density=density)
    env = quest.Env.loopback(1 << k)
    env.set_exchange_chunk(16)
    try:
        got = run_product(env, c, density=density)
        assert_parity(got, want)
        q = quest.QuregHandle(env, n, density)
        C.apply_circuit(q, c)
        assert abs(q.calcTotalProb() - (oracle.orc_trace(want, n).real if density else oracle.orc_norm_kahan(want))) < TOL
        q.destroy()
    finally:
        env.destroy()


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("density", [False, True])
@pytest.mark.parametrize("chunk", [16, 1 << 24])
def test_qubit_swaps_equal_single(k, density, chunk):
    """Global<->local swaps (default) give the single-rank result bit for bit,
    including reductions, collapse and amplitude reads taken while qubits are
    displaced."""
    n = 4 if density else 11
    c = random_gate_circuit(n, 160, seed=90 + k, max_controls=2, channels=density)
    want = oracle_run(c, density=density)
    env = quest.Env.loopback(1 << k)
    env.set_exchange_chunk(chunk)
    try:
        q = quest.QuregHandle(env, n, density)
        C.apply_circuit(q, c)
        flat = 2 * n if density else n
        # probabilities before any read restores the layout
        for t in range(n):
            want_p = oracle.orc_prob_of_outcome(want, n, t, 1, density)
            assert abs(q.calcProbOfOutcome(t, 1) - want_p) < TOL
        a = q.getAmp(5) if not density else None
        got = q.state()
        assert_parity(got, want)
        if a is not None:
            assert a.real == want[5].real and a.imag == want[5].imag
        # keep going from a restored layout, then collapse while displaced
        C.apply_circuit(q, c)
        want2 = oracle_run(c, density=density, init=want)
        t = n - 1
        p = oracle.orc_prob_of_outcome(want2, n, t, 0, density)
        q.collapseToOutcome(t, 0)
        want3 = oracle.orc_collapse(want2, n, t, 0, p, density)
        assert np.max(np.abs(q.state() - want3)) < TOL
        q.destroy()
    finally:
        env.destroy()


def test_qubit_swaps_cut_exchange_traffic():
    """A layer of gates on the global qubits: per-gate exchanges move a whole
    partition per gate; swaps move half a partition once per qubit."""
    n, k = 12, 2
    c = C.layered_random_circuit(n, 6, 5)
    traffic = {}
    for swaps in (False, True):
        env = quest.Env.loopback(1 << k)
        env.set_qubit_swaps(swaps)
        q = quest.QuregHandle(env, n)
        C.apply_circuit(q, c)
        q.flush()
        traffic[swaps] = int(q.comm_stats(1 << k)[1].sum())
        q.destroy()
        env.destroy()
    assert 0 < traffic[True] < traffic[False] / 2, traffic


def test_loopback_comm_accounting():
    """Exchange accounting: a communicated gate moves exactly
    16 * 2^(n-k) bytes per rank, in 2^(n-k)/chunk messages; local gates none."""
    n, k = 10, 2
    env = quest.Env.loopback(1 << k)
    env.set_exchange_chunk(64)
    env.set_qubit_swaps(False)  # the reference's exchange per gate
    q = quest.QuregHandle(env, n)
    q.hadamard(3)
    q.flush()
    assert q.comm_stats(4)[1].sum() == 0
    q.hadamard(9)
    q.flush()
    msgs, byts = q.comm_stats(4)
    assert list(byts) == [16 * (1 << (n - k))] * 4
    assert list(msgs) == [(1 << (n - k)) // 64] * 4
    q.controlledNot(9, 8)  # control on rank bit 1: ranks 0, 1 skip
    q.flush()
    msgs2, byts2 = q.comm_stats(4)
    assert list(byts2 - byts) == [0, 0, 16 * 256, 16 * 256]
    q.destroy()
    env.destroy()


def test_validation_before_mutation(env):
    q = quest.QuregHandle(env, 5)
    q.hadamard(0)
    before = q.state()
    with pytest.raises(quest.DomainError, match="invalid target qubit 5"):
        q.hadamard(5)
    with pytest.raises(quest.DomainError, match="overlaps the target"):
        q.controlledNot(2, 2)
    arr, k = quest.int_array([1, 1, 3])
    with pytest.raises(quest.DomainError, match="duplicate control"):
        q.multiControlledPhaseFlip(arr, k)
    with pytest.raises(quest.DomainError, match="not unitary"):
        q.unitary(0, quest.cmatrix2([1, 0, 1, 0, 0, 0, 1, 0]))
    with pytest.raises(quest.DomainError, match="density-matrix"):
        q.mixDephasing(0, 0.1)
    with pytest.raises(quest.DomainError, match="finite"):
        q.set_state(np.array([np.nan + 0j]))
    with pytest.raises(quest.DomainError, match="out of range"):
        q.getAmp(32)
    assert bits_equal(q.state(), before)
    q.destroy()
    d = quest.QuregHandle(env, 2, density=True)
    with pytest.raises(quest.DomainError, match=r"\[0, 1/2\]"):
        d.mixDephasing(0, 0.6)
    with pytest.raises(quest.DomainError, match=r"\[0, 3/4\]"):
        d.mixDepolarising(1, 0.8)
    with pytest.raises(quest.DomainError, match="density matrix"):
        d.hadamard(2)
    d.destroy()


def test_init_and_amplitude_access(env):
    q = quest.QuregHandle(env, 6)
    q.initPlusState()
    assert abs(q.getAmp(17).real - 1 / 8) < 1e-15
    q.initClassicalState(5)
    assert q.getAmp(5).real == 1.0 and q.calcTotalProb() == 1.0
    rng = np.random.default_rng(1)
    a = rng.normal(size=64) + 1j * rng.normal(size=64)
    q.set_state(a)
    assert bits_equal(q.state(), a)
    q.initZeroState()
    assert q.getAmp(0).real == 1.0 and q.getProbAmp(1) == 0.0
    q.destroy()
    d = quest.QuregHandle(env, 3, density=True)
    d.initPlusState()
    assert abs(quest.call("getDensityAmp", d.h, 2, 5).real - 1 / 8) < 1e-15
    assert abs(d.calcTotalProb() - 1.0) < 1e-14
    d.destroy()


def test_kernels_actually_launch(env):
    before = quest.kernel_launches()
    q = quest.QuregHandle(env, 12)
    C.apply_circuit(q, C.layered_random_circuit(12, 4, 1))
    q.calcTotalProb()
    assert quest.kernel_launches() > before
    q.destroy()


@pytest.mark.slow
def test_30q_forward_inverse_property(env):
    """Config C2 size: layered 30-qubit circuit then its inverse returns |0>
    (size-independent property), and the norm stays 1."""
    n = 30
    c = C.layered_random_circuit(n, 4, 12345)
    q = quest.QuregHandle(env, n)
    C.apply_circuit(q, c)
    assert abs(q.calcTotalProb() - 1.0) < 1e-12
    C.apply_circuit(q, C.inverse_circuit(c))
    a0 = q.getAmp(0)
    assert abs(a0.real - 1.0) < 1e-12 and abs(a0.imag) < 1e-12
    assert abs(q.calcProbOfOutcome(n - 1, 0) - 1.0) < 1e-12
    q.destroy()


@pytest.mark.slow
def test_33q_config_c3a_forward_inverse(env):
    """Config C3a size (33 qubits = 128 GiB on one B200): a layered circuit
    and its inverse return |0>, the norm stays 1 (size-independent)."""
    n = 33
    c = C.layered_random_circuit(n, 2, 12345)
    q = quest.QuregHandle(env, n)
    try:
        C.apply_circuit(q, c)
        assert abs(q.calcTotalProb() - 1.0) < 1e-12
        C.apply_circuit(q, C.inverse_circuit(c))
        a0 = q.getAmp(0)
        assert abs(a0.real - 1.0) < 1e-12 and abs(a0.imag) < 1e-12
        assert abs(q.calcProbOfOutcome(n - 1, 1)) < 1e-12
    finally:
        q.destroy()


@pytest.mark.slow
def test_32q_config_c5_qft_measure_collapse(env):
    """Config C5 size (32 qubits): QFT of a basis state with multi-controlled
    phase flips; every qubit then reads P = 1/2 and collapsing four of them
    leaves a normalised state with those outcomes certain."""
    n = 32
    q = quest.QuregHandle(env, n)
    try:
        q.initClassicalState(0x5A5A5A5A)
        C.apply_circuit(q, C.qft_circuit(n, mcpf_every=3))
        for t in range(n):
            assert abs(q.calcProbOfOutcome(t, 0) - 0.5) < 1e-12
        for t, o in [(0, 1), (9, 0), (21, 1), (31, 0)]:
            assert abs(q.collapseToOutcome(t, o) - 0.5) < 1e-12
        assert abs(q.calcTotalProb() - 1.0) < 1e-12
        for t, o in [(0, 1), (9, 0), (21, 1), (31, 0)]:
            assert abs(q.calcProbOfOutcome(t, o) - 1.0) < 1e-12
        assert abs(q.calcProbOfOutcome(5, 0) - 0.5) < 1e-12
    finally:
        q.destroy()


@pytest.mark.slow
@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")
def test_14q_density_config_c4_against_reference(env):
    """Config C4 size (14-qubit density matrix = 28-qubit vector, 4 GiB):
    a noisy layered circuit, bit-identical to the compiled reference run with
    all host threads; trace 1 and purity below 1."""
    import os

    N = 14
    c = C.layered_random_circuit(N, 1, 7, noise_pmax=0.1)
    want = oracle.ref_run(N, to_oracle_ops(c), density=True, workers=os.cpu_count() or 1)
    q = quest.QuregHandle(env, N, density=True)
    try:
        C.apply_circuit(q, c)
        assert abs(q.calcTotalProb() - 1.0) < 1e-12
        assert q.calcPurity() < 1.0
        assert_parity(q.state(), want)
    finally:
        q.destroy()


@pytest.fixture
def jit_sync():
    quest.set_jit(2)  # compile every pass shape before its first launch
    yield
    quest.set_jit(1)


@pytest.mark.parametrize("n", [12, 14, 17])
def test_jit_passes_bit_identical(env, jit_sync, n):
    """Per-pass JIT kernels (straight-line handler calls) give the oracle's
    amplitudes bit for bit: random gates with controls anywhere (outer ones
    skip per tile), a layered circuit, and a noisy density matrix."""
    before = quest.jit_stats()[0]
    c = random_gate_circuit(n, 150, seed=300 + n, max_controls=3)
    assert_parity(run_product(env, c), oracle_run(c))
    lc = C.layered_random_circuit(n, 6, 31 + n)
    assert_parity(run_product(env, lc), oracle_run(lc))
    if n == 12:
        d = C.layered_random_circuit(6, 3, 8, noise_pmax=0.1)
        assert_parity(run_product(env, d, density=True), oracle_run(d, density=True))
    assert quest.jit_stats()[0] > before  # kernels were compiled and used
    assert quest.jit_stats()[1] == 0


def low_qubit_circuit(n, count, seed):
    """Random gates whose targets mostly sit on qubits 0-4 (the tile's lane
    qubits), with controls anywhere: runs of pair ops per lane qubit."""
    from tests.harness import random_unitary

    rng = np.random.default_rng(seed)
    names = ["H", "X", "SX", "RX", "RY", "RZ", "T", "U"]
    c = C.Circuit(n, 0, [])
    for _ in range(count):
        t = int(rng.integers(0, 5)) if rng.random() < 0.7 else int(rng.integers(n))
        others = [q for q in range(n) if q != t]
        k = int(rng.integers(0, 3)) if rng.random() < 0.3 else 0
        ctrls = tuple(int(x) for x in rng.choice(others, size=k, replace=False)) if k else ()
        name = str(rng.choice(names))
        if name == "U":
            c.ops.append(C.GateOp("U", t, ctrls, matrix=tuple(random_unitary(rng))))
        else:
            c.ops.append(C.GateOp(name, t, ctrls, angle=float(rng.uniform(-2 * np.pi, 2 * np.pi))))
    return c


@pytest.mark.parametrize("jit", [2, 0])
@pytest.mark.parametrize("n", [13, 18])
def test_lane_exchanges_bit_identical(monkeypatch, n, jit):
    """Runs of pair ops on a lane qubit go through lane <-> register
    exchanges (QGPU_XCHG=2, TC_LANE_XCHG: the qubit moves to a register bit
    and back, pure moves), so those ops run as register ops: circuit order
    stays bit for bit the oracle's, JIT (sync) and interpreter."""
    monkeypatch.setenv("QGPU_XCHG", "2")
    e = quest.Env()
    quest.set_jit(jit)
    try:
        before = quest.lane_exchanges()
        c = low_qubit_circuit(n, 240, seed=70 + n)
        assert_parity(run_product(e, c), oracle_run(c))
        assert quest.lane_exchanges() > before  # the exchanges were used
    finally:
        quest.set_jit(1)
        e.destroy()


@pytest.mark.parametrize("phases", ["3", "8"])
@pytest.mark.parametrize("n", [20, 22])
def test_jit_equals_interpreter_multi_phase(monkeypatch, n, phases):
    """Bigger registers with multi-phase passes: tiles where outer controls
    skip a middle phase must resync the whole CTA (regression: a group
    barrier computed for the skipped transition raced). JIT (sync) and the
    interpreter agree bit for bit, and match the oracle at n = 20."""
    monkeypatch.setenv("QGPU_TILE_PHASES", phases)
    e = quest.Env()
    try:
        c = C.layered_random_circuit(n, 4, 12345)
        out = {}
        for mode in (0, 2):
            quest.set_jit(mode)
            out[mode] = run_product(e, c)
        quest.set_jit(1)
        assert np.array_equal(out[0], out[2])
        if n == 20:
            assert_parity(out[2], oracle_run(c))
    finally:
        quest.set_jit(1)
        e.destroy()


@pytest.mark.parametrize("delay", [0.0, 0.02, 0.08])
@pytest.mark.parametrize("python_atexit", [True, False])
def test_exit_with_jit_compiles_pending(tmp_path, delay, python_atexit):
    """A process that exits while the JIT still has compiles queued or in
    flight shuts the compile threads down cleanly (regressions: a
    function-local static destroyed before the engine joined its threads;
    NVRTC's lazily built statics destroyed at exit under a running
    nvrtcCompileProgram — a segfault). Covered with the Python wrapper's
    atexit hook and with the library's own (hook removed)."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    script = (
        "import sys, time, atexit; sys.path.insert(0, %r)\n"
        "from paper_1802_08032_b200 import circuits as C, quest\n"
        "from tests.harness import random_gate_circuit\n"
        "env = quest.Env(); q = quest.QuregHandle(env, 18)\n"
        "%s"
        "C.apply_circuit(q, random_gate_circuit(18, 400, 5, max_controls=2))\n"
        "q.flush(); print('pending', quest.jit_stats()[2])\n"
        "t = time.time()\n"
        "while time.time() - t < %r: pass\n"
        % (str(root), "" if python_atexit else "atexit.unregister(quest.lib().qgpuJitShutdown)\n", delay))
    for _ in range(3):
        r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, timeout=300,
                           cwd=str(root), env={**__import__("os").environ, "QGPU_JIT_OPTS": "-DQGPU_X=1"})
        assert r.returncode == 0, r.stderr[-2000:]
        assert "corrupt" not in r.stderr and "free()" not in r.stderr, r.stderr[-2000:]


def _common_control_circuit(n, seed, ctrl):
    """Gates that all carry the controls `ctrl` (qubits outside most tiles),
    interleaved with outer diagonal gates (a == 1: T, S, phase shifts)."""
    rng = np.random.default_rng(seed)
    names = ["H", "X", "Y", "RX", "RY", "RZ", "T", "S", "PHASE", "U", "Z"]
    c = C.Circuit(n, 0, [])
    free = [q for q in range(n) if q not in ctrl]
    for _ in range(120):
        nm = names[int(rng.integers(len(names)))]
        t = int(free[int(rng.integers(len(free)))])
        ang = float(rng.uniform(0, 6.3))
        if nm == "U":
            from tests.harness import random_unitary

            c.ops.append(C.GateOp("U", t, controls=tuple(ctrl), matrix=tuple(random_unitary(rng))))
        else:
            c.ops.append(C.GateOp(nm, t, controls=tuple(ctrl), angle=ang))
    return c


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("ctrl", [(15,), (14, 15), (13,)])
def test_tile_skipping_common_outer_controls(env, mode, ctrl):
    """Passes whose every op needs the same qubits outside the tile at 1 visit
    only those tiles (TileParams.skip_ones); the rest of the state must come
    through untouched. Fused passes and one op per pass, bit for bit."""
    n = 16
    env.set_fusion(mode, 48, 4)
    try:
        rng = np.random.default_rng(3)
        init = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
        init /= np.linalg.norm(init)
        c = _common_control_circuit(n, 11 + len(ctrl), ctrl)
        c.ops += [C.GateOp("T", 15), C.GateOp("PHASE", 14, angle=0.4), C.GateOp("S", 13, controls=(15,))]
        assert_parity(run_product(env, c, init=init), oracle_run(c, init=init))
    finally:
        env.set_fusion(0, 48, 4)


@pytest.mark.parametrize("swaps", [False, True])
def test_tile_skipping_rank_bit_controls(swaps):
    """Controls on rank bits common to a whole pass skip the non-matching
    ranks' launches (distributed.cpp:143-145 at pass level)."""
    n, k = 15, 2
    c = _common_control_circuit(n, 5, (14,))
    c.ops += _common_control_circuit(n, 6, (13, 14)).ops
    want = oracle_run(c)
    e = quest.Env.loopback(1 << k)
    e.set_qubit_swaps(swaps)
    try:
        assert_parity(run_product(e, c), want)
    finally:
        e.destroy()


@pytest.mark.parametrize("density", [False, True])
def test_run_circuit_batch_equals_per_call(env, density):
    """qgpuRunCircuit (run_circuit, circuit.cpp:239-247, one C-ABI call) gives
    the per-call result and the oracle's, bit for bit; an invalid op anywhere
    in the array leaves the register untouched."""
    n = 6 if density else 14
    c = random_gate_circuit(n, 150, seed=77, max_controls=2, channels=density)
    q = quest.QuregHandle(env, n, density)
    try:
        C.run_circuit(q, c)
        got = q.state()
        assert_parity(got, oracle_run(c, density=density))
        assert_parity(got, run_product(env, c, density=density))
        bad = C.op_array(c)
        bad[len(bad) // 2]["target"] = n  # out of range, mid-array
        with pytest.raises(quest.DomainError, match="invalid"):
            q.run_ops(bad)
        chan = C.op_array(C.Circuit(n, 0, [C.GateOp("H", 0), C.GateOp("DEPOL", 1, prob=0.9)]))
        with pytest.raises(quest.DomainError):
            q.run_ops(chan)  # p > 3/4 (density) or a channel on a state vector
        assert np.array_equal(q.state(), got)
    finally:
        q.destroy()


@pytest.mark.parametrize("precision", ["double", "single"])
def test_nccl_environment_single_rank(precision):
    """The NCCL environment (qgpuCreateNcclEnv: communicator init, the NCCL
    transport, all-gathered reductions) on one rank — the multi-GPU
    plumbing runs on real hardware even with one GPU; results equal the
    oracle's bit for bit."""
    uid = quest.Env.nccl_unique_id()
    e = quest.Env.nccl(0, 1, 0, uid)
    try:
        assert e.num_ranks == 1 and e.rank == 0
        c = random_gate_circuit(14, 120, seed=123, max_controls=2)
        q = quest.QuregHandle(e, 14, precision=precision)
        C.run_circuit(q, c)
        got = q.state()
        ops = to_oracle_ops(c)
        if precision == "single":
            assert np.array_equal(got, oracle.orc_run_f(14, ops).astype(np.complex128))
        else:
            assert_parity(got, oracle_run(c))
        w = got.astype(np.complex128)
        assert abs(q.calcTotalProb() - float(np.sum(np.abs(w) ** 2))) < 1e-12
        assert abs(q.calcProbOfOutcome(3, 1) - float(np.sum(np.abs(w[((np.arange(1 << 14) >> 3) & 1) == 1]) ** 2))) < 1e-12
        q.destroy()
    finally:
        e.destroy()


def _product_matrix(env, apply):
    """The 2x2 matrix a C-ABI gate call applies, read off a 1-qubit register:
    column j = the state after the gate on |j> (pair_lo_out / pair_hi_out
    with a unit and a zero amplitude reproduce the coefficients exactly)."""
    cols = []
    for j in (0, 1):
        q = quest.QuregHandle(env, 1)
        try:
            q.initClassicalState(j)
            apply(q)
            cols.append(q.state())
        finally:
            q.destroy()
    (m00, m10), (m01, m11) = cols
    return [m00.real, m00.imag, m01.real, m01.imag, m10.real, m10.imag, m11.real, m11.imag]


@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")
def test_product_gate_matrices_equal_reference(env):
    """hadamard / pauliX/Y/Z / tGate / rotateX/Y/Z / rotateAroundAxis through
    the C-ABI apply exactly the reference's gate_matrix / rotation_matrix
    (gates.cpp:51-98) on random angles and unit axes."""
    ids = C.REF_GATE_IDS
    fixed = {"H": "hadamard", "X": "pauliX", "Y": "pauliY", "Z": "pauliZ", "T": "tGate"}
    for name, fn in fixed.items():
        got = _product_matrix(env, lambda q: getattr(q, fn)(0))
        assert got == list(oracle.ref_gate_matrix(ids[name])), name
    rng = np.random.default_rng(98)
    for a in list(rng.uniform(-4 * np.pi, 4 * np.pi, 12)) + [0.0, np.pi]:
        a = float(a)
        for name in ("RX", "RY", "RZ"):
            got = _product_matrix(env, lambda q: getattr(q, "rotate" + name[1])(0, a))
            assert got == list(oracle.ref_gate_matrix(ids[name], a)), (name, a)
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        got = _product_matrix(env, lambda q: q.rotateAroundAxis(0, a, quest.Vector(*map(float, v))))
        assert got == list(oracle.ref_rotation_matrix(v, a)), (v, a)


@pytest.mark.parametrize("init", ["initPlusState", "initStateFromAmps"])
def test_init_after_queued_gates_on_swapping_ranks(init):
    """Gates queued for swap planning (loopback ranks, qubit swaps on) are
    dropped by a whole-state initialiser, not applied on top of it."""
    lb = quest.Env.loopback(4)
    try:
        n = 8
        q = quest.QuregHandle(lb, n)
        for t in (7, 6, 0, 7):  # 6, 7 are global qubits: these wait in the swap window
            q.hadamard(t)
        q.rotateX(6, 0.3)
        if init == "initPlusState":
            q.initPlusState()
            want = np.full(1 << n, 1 / 16, dtype=np.complex128)
        else:
            rng = np.random.default_rng(3)
            want = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
            re, im = np.ascontiguousarray(want.real), np.ascontiguousarray(want.imag)
            quest.call("initStateFromAmps", q.h, re.ctypes.data, im.ctypes.data)
        assert np.array_equal(q.state(), want)
        a = q.getAmp(200)
        assert complex(a.real, a.imag) == complex(want[200])
        q.destroy()
    finally:
        lb.destroy()


def test_clone_needs_the_source_environment(env):
    q = quest.QuregHandle(env, 5)
    other = quest.Env.loopback(2)
    try:
        with pytest.raises(quest.DomainError):
            quest.call("createCloneQureg", q.h, other.h)
    finally:
        other.destroy()
        q.destroy()


@pytest.mark.parametrize("ranks", [1, 2, 4])
@pytest.mark.parametrize("precision", ["double", "single"])
def test_marginals_and_deferred_collapses(ranks, precision):
    """calcProbOfOutcome from the one-read marginals (>= 13 local qubits) and
    collapses deferred as selections: every probability within 1e-12 of the
    compensated restatement on the state the reference's sequence produces
    (collapse after collapse), measurement outcomes equal to the restated
    measure under the same seed, and the final amplitudes."""
    n = 16
    c = random_gate_circuit(n, 200, seed=123 + ranks, max_controls=2)
    env = quest.Env.loopback(ranks) if ranks > 1 else quest.Env()
    single = precision == "single"
    tol = 1e-6 if single else TOL
    try:
        q = quest.QuregHandle(env, n, precision=precision)
        C.apply_circuit(q, c)
        if not single:
            assert bits_equal(q.state(), oracle_run(c))
        # the product's state is the checker's input from here on (single
        # precision: the restatement then works on the widened floats)
        want = q.state()
        for t in range(n):
            for o in (0, 1):
                assert abs(q.calcProbOfOutcome(t, o) - oracle.orc_prob_of_outcome(want, n, t, o)) < tol
        cur = want
        for t, o in [(3, 1), (15, 0), (8, 1), (3, 1), (0, 0)]:
            p = oracle.orc_prob_of_outcome(cur, n, t, o)
            assert abs(q.collapseToOutcome(t, o) - p) < tol
            cur = oracle.orc_collapse(cur, n, t, o, p)
            for u in (1, 8, 12):
                assert abs(q.calcProbOfOutcome(u, 1) - oracle.orc_prob_of_outcome(cur, n, u, 1)) < tol
            assert abs(q.calcTotalProb() - oracle.orc_norm_kahan(cur)) < tol
        with pytest.raises(quest.DomainError):
            q.collapseToOutcome(15, 1)  # contradicts a pending collapse: probability 0
        env.seed(99, 7)
        st = oracle.orc_seed([99, 7])
        for t in (5, 9, 14):
            o, _, cur, st = oracle.orc_measure(cur, n, t, st)
            assert q.measure(t) == o
        assert np.max(np.abs(q.state() - cur)) < tol
        q.destroy()
    finally:
        env.destroy()
