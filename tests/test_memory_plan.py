"""Memory plan: the reference's node model restated in
the C-ABI library agrees with the compiled reference (modeled_bytes_per_rank /
max_qubits, distributed.cpp:423-468) and its SPEC.md known answers; the device
model sizes registers for B200 HBM. CPU only: pure host calls."""
import ctypes

import pytest

import oracle
from paper_1802_08032_b200 import quest

GiB = 1 << 30
STRATS = ["full_clone", "half_exchange", "per_amplitude"]


def test_spec_kats():
    # max_qubits(64 GiB, 50 MiB, full_clone, double, k) = 30 + k, k in [0, 8]
    for k in range(9):
        assert quest.max_qubits(64 * GiB, k) == 30 + k
    # minimal node count for n = 38 at 64 GiB / full_clone is 2^8 (PAPER: 256 nodes)
    assert min(k for k in range(16) if quest.max_qubits(64 * GiB, k) >= 38) == 8
    # state-only bytes for n = 30: 16 GiB; full clone doubles it
    assert quest.modeled_bytes_per_rank(30, 0, "per_amplitude", block_amps=0) == 16 * GiB
    assert quest.modeled_bytes_per_rank(30, 0, "full_clone") == 32 * GiB
    assert quest.modeled_bytes_per_rank(30, 0, "half_exchange") == 24 * GiB


def test_monotone_in_node_bytes_and_ranks():
    # max_qubits is monotone non-decreasing in node_bytes and in k
    for s in STRATS:
        prev = [quest.max_qubits(b * GiB, 0, s) for b in (1, 2, 8, 64, 512)]
        assert prev == sorted(prev)
        ks = [quest.max_qubits(64 * GiB, k, s) for k in range(12)]
        assert ks == sorted(ks)


def test_invalid_inputs_raise():
    with pytest.raises(quest.DomainError):
        quest.modeled_bytes_per_rank(4, 5, "full_clone")
    with pytest.raises(quest.DomainError):
        quest.modeled_bytes_per_rank(70, 0, "full_clone")  # overflows 64 bits
    with pytest.raises(quest.DomainError):
        quest.max_qubits(64 * GiB, -1)
    assert quest.max_qubits(10 << 20, 0) == 0  # budget below the overhead


@pytest.mark.skipif(not oracle.ref_available(), reason="reference not built here")
@pytest.mark.parametrize("strategy", range(3))
@pytest.mark.parametrize("single", [0, 1])
def test_matches_compiled_reference(strategy, single):
    R = oracle.ref()
    for n, k, block in [(1, 0, 1), (10, 3, 7), (30, 0, 1), (33, 3, 1 << 24), (36, 3, 1 << 24), (50, 10, 5)]:
        want = ctypes.c_ulonglong()
        assert R.ref_modeled_bytes(n, k, strategy, single, block, ctypes.byref(want)) == 0
        got = ctypes.c_ulonglong()
        assert quest.lib().qgpuModeledBytesPerRank(n, k, strategy, single, block, ctypes.byref(got)) == 0
        assert got.value == want.value, (n, k, block)
    for node in (1 << 20, GiB, 64 * GiB, 180 * 10**9, 1 << 50):
        for k in (0, 1, 3, 8):
            want = ctypes.c_int()
            assert R.ref_max_qubits(node, 50 << 20, strategy, single, k, ctypes.byref(want)) == 0
            got = quest.lib().qgpuMaxQubits(node, 50 << 20, strategy, single, k)
            assert got == want.value, (node, k)


def test_device_plan_for_b200():
    hbm = 180 * 10**9  # usable HBM3e per B200, rounded down
    # one GPU: 33 qubits (128 GiB) fit, 34 (256 GiB) do not (BASELINE configs[2])
    assert quest.device_max_qubits(hbm, 0) == 33
    # eight GPUs: 36 qubits = 128 GiB per GPU + two 256 MiB exchange sub-chunks
    assert quest.device_max_qubits(hbm, 3) == 36
    per = quest.device_bytes_per_rank(36, 3)
    assert per == 128 * GiB + 2 * (1 << 24) * 16 + (592 + 8 + 1) * 16
    # a 14-qubit density matrix is a 28-qubit vector: 4 GiB
    assert quest.device_bytes_per_rank(28, 0) < 5 * GiB
    assert quest.device_max_qubits(hbm, 0, density=True) == 16
    # the sub-chunk buffers never exceed the partition
    assert quest.device_bytes_per_rank(10, 2, 1 << 24) == 16 * (1 << 8) * 3 + (592 + 4 + 1) * 16


def test_reference_named_mirror():
    from paper_1802_08032_b200 import qsim

    m = qsim.MemoryModel(node_bytes=64 * GiB)
    assert [qsim.max_qubits(m, k) for k in range(4)] == [30, 31, 32, 33]
    assert qsim.modeled_bytes_per_rank(30, 0, "half_exchange", "single") == 12 * GiB


def test_device_plan_single_precision():
    """Single-precision registers: 8 B amplitudes and exchange sub-chunks (the
    reduction scratch stays double-double), so one more qubit fits."""
    hbm = 180 * 10**9
    assert quest.device_max_qubits(hbm, 0, single=True) == 34
    assert quest.device_max_qubits(hbm, 3, single=True) == 37
    per = quest.device_bytes_per_rank(36, 3, single=True)
    assert per == 64 * GiB + 2 * (1 << 24) * 8 + (592 + 8 + 1) * 16
