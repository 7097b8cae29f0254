"""The reference's own C++ API, re-exposed by paper_1802_08032_b200.qsim on
the B200 C-ABI, against the SPEC.md examples the reference's (unshipped) tests
were written from. Reads like the reference's tests; runs on the GPU."""
import math

import numpy as np
import pytest

from paper_1802_08032_b200 import qsim

S = 1 / math.sqrt(2)


def test_memory_bytes_kats():  # CPU: pure arithmetic (register.cpp:140-151)
    assert qsim.memory_bytes(30) == 17_179_869_184
    assert qsim.memory_bytes(1, precision="single") == 16
    assert qsim.memory_bytes(15, qsim.DENSITY_MATRIX) == 16 * 2**30
    with pytest.raises(qsim.DomainError):
        qsim.memory_bytes(0)
    with pytest.raises(qsim.DomainError):
        qsim.memory_bytes(61)


def test_enumerate_pairs_kats():  # CPU: kernels.cpp:68-82
    assert qsim.enumerate_pairs(1, 0) == [(0, 1)]
    assert qsim.enumerate_pairs(3, 1) == [(0, 2), (1, 3), (4, 6), (5, 7)]
    assert qsim.enumerate_pairs(3, 2) == [(0, 4), (1, 5), (2, 6), (3, 7)]
    for n in range(1, 11):
        for t in range(n):
            flat = sorted(x for p in qsim.enumerate_pairs(n, t) for x in p)
            assert flat == list(range(1 << n))


def test_partition_rules():  # CPU: distributed.cpp:31-57 via the library planner
    plan = qsim.partition(34, 4)
    assert not qsim.needs_communication(plan, 29) and qsim.needs_communication(plan, 30)
    assert qsim.pair_rank(qsim.partition(3, 1), 0, 2) == 1
    assert qsim.pair_rank(qsim.partition(4, 2), 1, 3) == 3
    with pytest.raises(qsim.DomainError):
        qsim.pair_rank(qsim.partition(3, 1), 0, 0)
    with pytest.raises(qsim.DomainError):
        qsim.partition(3, 4)


def test_gate_matrix_unitarity():  # CPU: gates.cpp:16-98
    for name in ["H", "T", "X", "Y", "Z", "SX", "SY"]:
        assert qsim.is_unitary(qsim.gate_matrix(qsim.NamedGate(name)))
    sx = qsim.gate_matrix(qsim.NamedGate("SX"))
    x = sx * sx
    assert abs(x.m01 - 1) < 1e-15 and abs(x.m00) < 1e-15
    with pytest.raises(qsim.DomainError):
        qsim.rotation_matrix((1, 1, 0), 0.3)
    with pytest.raises(qsim.DomainError):
        qsim.GateMatrix.unitary_checked(1, 1, 0, 1)


pytestmark_gpu = pytest.mark.gpu


@pytest.mark.gpu
def test_register_create_and_access():
    r = qsim.Register(1)
    assert list(r.amps()) == [1, 0]
    d = qsim.Register(2, qsim.DENSITY_MATRIX)
    a = d.amps()
    assert a.size == 16 and a[0] == 1 and not a[1:].any()
    r.set_amplitude(0, 0)
    r.set_amplitude(1, 1)
    assert r.get_amplitude(1) == 1
    with pytest.raises(qsim.DomainError):
        r.set_amplitude(0, complex(float("nan"), 0))
    with pytest.raises(qsim.DomainError):
        r.get_amplitude(2)
    r.init_zero_state()
    r.init_zero_state()
    assert list(r.amps()) == [1, 0]  # SPEC.md:72-74 (idempotent)
    assert qsim.Register(12).norm_squared() == 1.0


@pytest.mark.gpu
def test_gate_kernel_kats():
    r = qsim.Register(1)
    qsim.apply_single_qubit_gate(r, 0, qsim.gate_matrix(qsim.NamedGate("X")))
    assert list(r.amps()) == [0, 1]
    r = qsim.Register(3)
    r.set_amps(np.eye(1, 8, 6, dtype=complex)[0])
    qsim.apply_controlled_gate(r, [1, 2], 0, qsim.gate_matrix(qsim.NamedGate("X")))
    assert r.get_amplitude(7) == 1  # SPEC.md:186 (Toffoli)
    r = qsim.Register(1)
    qsim.apply_single_qubit_rotation(r, 0, (1, 0, 0), math.pi)
    assert abs(r.get_amplitude(1) + 1j) < 1e-15
    with pytest.raises(qsim.DomainError):
        qsim.apply_controlled_gate(r, [0], 0, qsim.gate_matrix(qsim.NamedGate("X")))
    d = qsim.Register(1, qsim.DENSITY_MATRIX)
    with pytest.raises(qsim.DomainError):  # kernels.cpp:107-110
        qsim.apply_controlled_gate(d, [], 0, qsim.gate_matrix(qsim.NamedGate("X")))


@pytest.mark.gpu
def test_density_kats():
    d = qsim.Register(1, qsim.DENSITY_MATRIX)
    qsim.apply_named_gate(d, qsim.NamedGate("X"), [], 0)
    assert list(d.amps()) == [0, 0, 0, 1]
    d.set_amps(np.array([0.5, 0.5, 0.5, 0.5], dtype=complex))
    qsim.apply_dephasing(d, 0, 0.5)
    assert np.allclose(d.amps(), [0.5, 0, 0, 0.5], atol=0)
    d.set_amps(np.array([0.7, 0.2 - 0.1j, 0.2 + 0.1j, 0.3]))
    qsim.apply_depolarising(d, 0, 0.75)
    assert np.max(np.abs(d.amps() - [0.5, 0, 0, 0.5])) < 1e-15
    assert abs(qsim.trace(d) - 1) < 1e-15 and abs(qsim.purity(d) - 0.5) < 1e-15
    with pytest.raises(qsim.DomainError):
        qsim.apply_dephasing(d, 0, 0.51)
    with pytest.raises(qsim.DomainError):
        qsim.apply_depolarising(d, 1, 0.1)


@pytest.mark.gpu
def test_run_circuit_and_density_consistency():
    """SPEC.md:288 / acceptance 6: density evolution == outer product of the
    state-vector evolution."""
    c = qsim.generate_random_circuit(4, 10, 3)
    sv = qsim.Register(4)
    qsim.run_circuit(c, sv)
    dm = qsim.Register(4, qsim.DENSITY_MATRIX)
    qsim.run_circuit(c, dm)
    psi = sv.amps()
    rho = np.outer(psi, psi.conj())
    flat = rho.T.reshape(-1)  # rho_jk at j + 2^N k
    assert np.max(np.abs(dm.amps() - flat)) < 1e-12
    with pytest.raises(qsim.DomainError):
        qsim.run_circuit(c, qsim.Register(5))
