"""Pins the CPU restatement (oracle/qsim_oracle.c) to the UNMODIFIED
reference compiled in place (oracle/_ref), bit for bit. CPU only."""
import numpy as np
import pytest

import oracle
from paper_1802_08032_b200 import circuits as C
from tests.harness import bits_equal, oracle_run, random_gate_circuit, to_oracle_ops

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="reference not built here")


@needs_ref
@pytest.mark.parametrize("seed", [1, 2, 12345])
def test_restatement_matches_reference_generator_circuits(seed):
    ops, _ = oracle.ref_random_circuit(10, 12, seed)
    assert bits_equal(oracle.ref_run(10, ops, workers=3), oracle.orc_run(10, ops))


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_restatement_matches_reference_random_unitaries(seed):
    c = random_gate_circuit(9, 120, seed, max_controls=3)
    ops = to_oracle_ops(c)
    assert bits_equal(oracle.ref_run(9, ops, workers=4), oracle.orc_run(9, ops))


@needs_ref
@pytest.mark.parametrize("seed", range(4))
def test_restatement_matches_reference_density_with_channels(seed):
    c = random_gate_circuit(4, 80, 100 + seed, max_controls=2, channels=True)
    ops = to_oracle_ops(c)
    assert bits_equal(oracle.ref_run(4, ops, density=True, workers=2),
                      oracle.orc_run(4, ops, density=True))


@needs_ref
def test_restatement_matches_reference_layered_circuit():
    c = C.layered_random_circuit(12, 8, 12345)
    ops = to_oracle_ops(c)
    assert bits_equal(oracle.ref_run(12, ops, workers=8), oracle.orc_run(12, ops))


@needs_ref
def test_restatement_from_random_initial_state():
    rng = np.random.default_rng(3)
    init = rng.normal(size=1 << 8) + 1j * rng.normal(size=1 << 8)
    c = random_gate_circuit(8, 60, 77)
    ops = to_oracle_ops(c)
    assert bits_equal(oracle.ref_run(8, ops, init=init), oracle.orc_run(8, ops, init=init))


@needs_ref
def test_reductions_against_reference():
    c = random_gate_circuit(3, 40, 5, channels=True)
    amps = oracle_run(c, density=True)
    norm, tr, pur = oracle.ref_reductions(3, amps, density=True)
    assert abs(oracle.orc_norm_kahan(amps) - norm) < 1e-14
    assert abs(oracle.orc_trace(amps, 3) - tr) < 1e-14
    assert abs(pur - norm) == 0.0


def test_kahan_beats_naive_sum():
    rng = np.random.default_rng(0)
    a = rng.normal(size=1 << 20) + 1j * rng.normal(size=1 << 20)
    a /= np.sqrt(np.sum(np.abs(a) ** 2, dtype=np.longdouble))
    exact = float(np.sum(a.real.astype(np.longdouble) ** 2 + a.imag.astype(np.longdouble) ** 2))
    assert abs(oracle.orc_norm_kahan(a) - exact) <= 4e-16


def test_prob_collapse_measure_restated():
    c = C.qft_circuit(6)
    amps = oracle_run(c, init=np.eye(1, 64, 13, dtype=np.complex128)[0])
    for q in range(6):
        assert abs(oracle.orc_prob_of_outcome(amps, 6, q, 0) - 0.5) < 1e-14
    col = oracle.orc_collapse(amps, 6, 2, 1, 0.5)
    assert abs(oracle.orc_norm_kahan(col) - 1.0) < 1e-14
    st = oracle.orc_seed([12345])
    o1, p1, a1, s1 = oracle.orc_measure(amps, 6, 0, st)
    o2, p2, a2, s2 = oracle.orc_measure(amps, 6, 0, st)
    assert (o1, p1, s1) == (o2, p2, s2) and bits_equal(a1, a2)


def test_splitmix_matches_python_generator():
    st = oracle.ctypes_state = None
    import ctypes

    s = ctypes.c_uint64(42)
    py = C.SplitMix64(42)
    for _ in range(100):
        assert oracle.restated().orc_splitmix64_next(ctypes.byref(s)) == py.next()


@needs_ref
@pytest.mark.parametrize("strategy", ["full_clone", "half_exchange", "per_amplitude"])
def test_combine_restatement_matches_reference_distributed(strategy):
    """Single-rank restatement + orc_combine protocol == reference run_gate_ops."""
    n, k = 8, 2
    c = random_gate_circuit(n, 50, 9, max_controls=2)
    ops = to_oracle_ops(c)
    ref_out, msgs, byts, rounds = oracle.ref_run_distributed(n, ops, k, strategy, block_amps=16)
    assert bits_equal(ref_out, oracle.orc_run(n, ops))
    # protocol restated on 4 rank chunks with orc_combine for global targets
    L = 1 << (n - k)
    chunks = [oracle.zero_state(n)[r * L:(r + 1) * L].copy() for r in range(1 << k)]
    for op in ops:
        t, mask = int(op["target"]), int(op["ctrl_mask"])
        rank_mask, low = mask >> (n - k), mask & (L - 1)
        new = []
        for r in range(1 << k):
            if (r & rank_mask) != rank_mask:
                new.append(chunks[r])
                continue
            if t < n - k:
                x = chunks[r].copy()
                oracle.restated().orc_apply_gate(x.ctypes.data, n - k, t, low, op["m"].ctypes.data)
                new.append(x)
            else:
                peer = r ^ (1 << (t - (n - k)))
                own_lo = not ((r >> (t - (n - k))) & 1)
                new.append(oracle.orc_combine(chunks[r], chunks[peer], low, own_lo, op["m"]))
        chunks = new
    assert bits_equal(np.concatenate(chunks), ref_out)


@pytest.mark.skipif(not oracle.ref_available(), reason="reference not built here")
@pytest.mark.parametrize("n,density,seed", [(8, False, 1), (11, False, 2), (5, True, 3), (13, False, 4)])
def test_single_precision_restatement_matches_reference(n, density, seed):
    """The float restatement (Mat2<float>, float fma chain, narrowed channel
    factors) equals the reference's Precision::Single run bit for bit."""
    import numpy as np

    from tests.harness import random_gate_circuit, to_oracle_ops

    ops = to_oracle_ops(random_gate_circuit(n, 200, seed, max_controls=2, channels=density))
    got = oracle.orc_run_f(n, ops, density)
    want = oracle.ref_run_single(n, ops, density)
    assert got.dtype == np.complex64 and np.array_equal(got, want)
