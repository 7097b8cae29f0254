"""Single precision: Register(..., Precision::Single)
through the C-ABI against the float restatement (oracle.orc_run_f, pinned to
the compiled reference's Precision::Single run in tests/test_oracle.py).

Bar: bit-identical float amplitudes for every gate / channel path — the
kernels evaluate the reference's float fma chain on Mat2<float> coefficients
and narrowed channel factors (kernels.cpp:61-62, density.cpp:105-140), in the
tile pass (interpreter and JIT), the one-kernel-per-op path for small states,
the exchange combines and the qubit swaps. Reductions accumulate in double
(register.cpp:62-73), so they match a double sum of the widened floats to
1e-12.
"""
import numpy as np
import pytest

import oracle
from paper_1802_08032_b200 import circuits as C
from paper_1802_08032_b200 import quest
from tests.harness import bits_equal, random_gate_circuit, to_oracle_ops

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def env():
    e = quest.Env()
    yield e
    e.destroy()


def run_single(env, circuit, density=False):
    q = quest.QuregHandle(env, circuit.num_qubits, density, precision="single")
    try:
        assert q.precision == "single"
        C.apply_circuit(q, circuit)
        return q.state()
    finally:
        q.destroy()


def want_single(circuit, density=False):
    return oracle.orc_run_f(circuit.num_qubits, to_oracle_ops(circuit), density)


def assert_parity_f(got, want):
    want = np.asarray(want, dtype=np.complex64)
    # the host boundary widens exactly: every value is a float
    assert np.array_equal(got.astype(np.complex64).astype(np.complex128), got)
    err = float(np.max(np.abs(got - want))) if got.size else 0.0
    assert bits_equal(got, want), f"not bit-identical (max-abs {err})"


FUSION = [(0, 48, 4), (1, 0, 4), (2, 0, 0)]


@pytest.mark.parametrize("mode,max_ops,h", FUSION)
@pytest.mark.parametrize("n", [3, 9, 12, 15])
def test_single_random_gates_all_fusion_modes(env, mode, max_ops, h, n):
    env.set_fusion(mode, max_ops if max_ops else 48, h if h else 4)
    try:
        c = random_gate_circuit(n, 150, seed=n * 17 + mode, max_controls=3)
        assert_parity_f(run_single(env, c), want_single(c))
    finally:
        env.set_fusion(0, 48, 4)


@pytest.mark.parametrize("N", [2, 5, 7])
def test_single_density_matrix_with_channels(env, N):
    c = random_gate_circuit(N, 120, seed=700 + N, max_controls=2, channels=True)
    assert_parity_f(run_single(env, c, density=True), want_single(c, density=True))


def test_single_density_noisy_layered(env):
    """Fused depolarise handler (TC_DEPOL) in float: a 7-qubit noisy layered
    circuit (flat 14, tiled)."""
    c = C.layered_random_circuit(7, 6, 99, noise_pmax=0.1)
    assert_parity_f(run_single(env, c, density=True), want_single(c, density=True))


def test_single_layered_20q_against_reference(env):
    """Config C1's circuit in single precision vs the compiled reference's
    Precision::Single run (the float restatement when it is not built)."""
    c = C.layered_random_circuit(20, 20, 12345)
    ops = to_oracle_ops(c)
    want = oracle.ref_run_single(20, ops, workers=8) if oracle.ref_available() else oracle.orc_run_f(20, ops)
    assert_parity_f(run_single(env, c), want)


@pytest.fixture
def jit_sync():
    quest.set_jit(2)
    yield
    quest.set_jit(1)


@pytest.mark.parametrize("n", [12, 17, 20])
def test_single_jit_equals_interpreter_and_oracle(env, n):
    """The per-pass JIT's float kernels (namespace tile_f32) and the float
    interpreter agree bit for bit with the restatement."""
    c = C.layered_random_circuit(n, 5, 77 + n)
    out = {}
    try:
        for mode in (0, 2):
            quest.set_jit(mode)
            out[mode] = run_single(env, c)
    finally:
        quest.set_jit(1)
    assert np.array_equal(out[0], out[2])
    assert_parity_f(out[2], want_single(c))


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("swaps", [True, False])
@pytest.mark.parametrize("density", [False, True])
def test_single_loopback_distributed(k, swaps, density):
    """2^k virtual ranks: qubit swaps (default) or the reference's exchange per
    global-target gate (float combines) give the single-rank float result."""
    n = 5 if density else 13
    c = random_gate_circuit(n, 120, seed=60 + k, max_controls=2, channels=density)
    want = want_single(c, density)
    env = quest.Env.loopback(1 << k)
    env.set_exchange_chunk(64)
    env.set_qubit_swaps(swaps)
    try:
        q = quest.QuregHandle(env, n, density, precision="single")
        C.apply_circuit(q, c)
        w = want.astype(np.complex128)
        for t in range(n):
            mask = ((np.arange(1 << (2 * n if density else n)) >> t) & 1) == 1
            if density:
                dim = 1 << n
                diag = np.arange(dim) * (dim + 1)
                p = float(np.sum(w[diag][((np.arange(dim) >> t) & 1) == 1].real))
            else:
                p = float(np.sum(np.abs(w[mask]) ** 2))
            assert abs(q.calcProbOfOutcome(t, 1) - p) < 1e-9
        assert_parity_f(q.state(), want)
        q.destroy()
    finally:
        env.destroy()


def test_single_reductions_and_io(env):
    n = 14
    c = random_gate_circuit(n, 100, seed=5, max_controls=2)
    want = want_single(c).astype(np.complex128)
    q = quest.QuregHandle(env, n, precision="single")
    try:
        C.apply_circuit(q, c)
        # norm: double accumulation of the widened floats
        ref = float(np.sum(want.real * want.real + want.imag * want.imag))
        assert abs(q.calcTotalProb() - ref) < TOL
        for t in (0, 6, n - 1):
            sel = ((np.arange(1 << n) >> t) & 1) == 0
            assert abs(q.calcProbOfOutcome(t, 0) - float(np.sum(np.abs(want[sel]) ** 2))) < TOL
        a = q.getAmp(37)
        assert a.real == want[37].real and a.imag == want[37].imag
        # writes narrow to float (AmpVector::set)
        rng = np.random.default_rng(1)
        v = rng.normal(size=64) + 1j * rng.normal(size=64)
        q.set_state(v, start=128)
        got = q.state(128, 64)
        assert np.array_equal(got, v.astype(np.complex64).astype(np.complex128))
        # clones keep the precision; cloneQureg refuses a precision mismatch
        cl = quest.QuregHandle(env, n, precision="single")
        cl.cloneQureg(q.h)
        assert np.array_equal(cl.state(), q.state())
        cl.destroy()
        d = quest.QuregHandle(env, n)
        with pytest.raises(quest.DomainError):
            d.cloneQureg(q.h)
        d.destroy()
    finally:
        q.destroy()


def test_single_init_states(env):
    q = quest.QuregHandle(env, 13, precision="single")
    try:
        q.initPlusState()
        s = q.state()
        assert np.all(s == np.complex64(1.0 / np.sqrt(2.0 ** 13)))
        q.initClassicalState(77)
        s = q.state()
        assert s[77] == 1.0 and np.count_nonzero(s) == 1
        q.initZeroState()
        assert q.calcTotalProb() == 1.0
    finally:
        q.destroy()


def test_single_30q_forward_inverse_property(env):
    """Full size: a 30-qubit float register (8 GiB) through a layered circuit
    and its inverse returns to |0> within float rounding; the norm stays 1."""
    n = 30
    c = C.layered_random_circuit(n, 8, 4242)
    q = quest.QuregHandle(env, n, precision="single")
    try:
        C.apply_circuit(q, c)
        assert abs(q.calcTotalProb() - 1.0) < 1e-4
        C.apply_circuit(q, C.inverse_circuit(c))
        assert abs(q.calcProbOfOutcome(n - 1, 0) - 1.0) < 1e-4
        a = q.getAmp(0)
        assert abs(abs(complex(a.real, a.imag)) - 1.0) < 1e-4
    finally:
        q.destroy()


def test_single_qsim_mirror_register():
    """qsim.Register(n, kind, "single") (register.hpp:53-54) through the
    reference-named mirror: run_circuit then amps() as complex64, equal to the
    reference's data32() bit for bit."""
    from paper_1802_08032_b200 import qsim

    c = C.layered_random_circuit(13, 4, 21)
    r = qsim.Register(13, qsim.STATE_VECTOR, "single")
    try:
        assert r.precision() == "single"
        qsim.run_circuit(c, r)
        got = r.amps()
        assert got.dtype == np.complex64
        ops = to_oracle_ops(c)
        want = oracle.ref_run_single(13, ops) if oracle.ref_available() else oracle.orc_run_f(13, ops)
        assert np.array_equal(got, want)
    finally:
        r.destroy()


@pytest.mark.parametrize("n", [1, 2])
@pytest.mark.parametrize("density", [False, True])
def test_single_smallest_registers_and_empty_circuits(env, n, density):
    """The smallest registers (1-2 qubits; a 1-qubit density matrix is a
    2-qubit flat vector) in single precision, and empty op arrays (a no-op)."""
    c = random_gate_circuit(n, 40, seed=9 + n, max_controls=1 if n > 1 else 0, channels=density)
    q = quest.QuregHandle(env, n, density, precision="single")
    try:
        q.run_ops(C.op_array(C.Circuit(n, 0, [])))
        C.run_circuit(q, c)
        q.run_ops(C.op_array(C.Circuit(n, 0, [])))
        assert_parity_f(q.state(), want_single(c, density))
    finally:
        q.destroy()


@pytest.mark.parametrize("n", [9, 14])
def test_single_collapse_measure_and_purity(env, n):
    """collapseToOutcome / measure on float registers (tiled and small): the
    kept half is scaled by the narrowed 1/sqrt(P), the rest zeroed; the norm
    returns to 1 within float rounding. Purity of a float density matrix
    accumulates in double."""
    c = random_gate_circuit(n, 80, seed=31 + n, max_controls=1)
    want = want_single(c).astype(np.complex128)
    q = quest.QuregHandle(env, n, precision="single")
    try:
        C.run_circuit(q, c)
        idx = np.arange(1 << n)
        ps = [float(np.sum(np.abs(want[((idx >> k) & 1) == 1]) ** 2)) for k in range(n)]
        t = int(np.argmax([min(x, 1 - x) for x in ps]))  # the most mixed qubit
        sel = ((idx >> t) & 1) == 1
        p = ps[t]
        got_p = q.collapseToOutcome(t, 1)
        assert abs(got_p - p) < 1e-12
        exp = np.where(sel, want * np.float32(1.0 / np.sqrt(p)), 0)
        assert np.max(np.abs(q.state() - exp)) < 1e-6
        assert abs(q.calcTotalProb() - 1.0) < 1e-5
        o = q.measure(2)
        assert o in (0, 1) and abs(q.calcProbOfOutcome(2, o) - 1.0) < 1e-5
    finally:
        q.destroy()
    d = quest.QuregHandle(env, 5, density=True, precision="single")
    try:
        dc = random_gate_circuit(5, 60, seed=8, max_controls=1, channels=True)
        C.run_circuit(d, dc)
        rho = want_single(dc, density=True).astype(np.complex128)
        assert abs(d.calcPurity() - float(np.sum(np.abs(rho) ** 2))) < 1e-12
    finally:
        d.destroy()


@pytest.mark.slow
def test_single_34q_max_size_forward_inverse(env):
    """The largest single-precision register one B200 holds (34 qubits, 2^34
    amplitudes, 128 GiB; qgpuDeviceMaxQubits(single)): a layered circuit and
    its inverse return to |0> within float rounding, probabilities and the
    norm through the double-accumulated reductions."""
    n = 34
    free, _ = __import__("torch").cuda.mem_get_info()
    if free < quest.device_bytes_per_rank(n, 0, single=True):
        pytest.skip("not enough free HBM for 2^34 float amplitudes")
    c = C.layered_random_circuit(n, 2, 777)
    q = quest.QuregHandle(env, n, precision="single")
    try:
        C.run_circuit(q, c)
        assert abs(q.calcTotalProb() - 1.0) < 1e-4
        assert abs(q.calcProbOfOutcome(n - 1, 0) - 0.5) < 0.5
        C.run_circuit(q, C.inverse_circuit(c))
        a0 = q.getAmp(0)
        assert abs(a0.real - 1.0) < 1e-4 and abs(a0.imag) < 1e-4
        assert abs(q.calcProbOfOutcome(n - 1, 0) - 1.0) < 1e-4
    finally:
        q.destroy()
