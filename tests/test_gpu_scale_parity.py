"""Amplitude parity at the headline sizes (BASELINE.json configs[1], [2]).

The north star's correctness bar is "all amplitudes within 1e-12 of the CPU
reference" on the bench's own configuration. These tests run the bench's
exact workload through the C-ABI and compare every amplitude:

* C2, 30 qubits (2^30 amplitudes, 16 GiB): the layered circuit of bench.py
  (depth 20, seed 12345, 875 gates) against the UNMODIFIED reference compiled
  from /root/reference (``oracle.ref_run``: ``qsim::Register`` +
  ``apply_controlled_gate``, kernels.cpp:105-112, on every host core), once
  with every pass shape JIT-compiled (the kernels the bench times) and once
  on the interpreter; plus a per-target sweep (H, Rx, CNOT with the control
  above and below, CPhase) on every target 0..29 (SURVEY.md §8(d) C2 sweep).
  The bar is bit-identity (np.array_equal), which implies the 1e-12 bound.
* C3a, 33 qubits (2^33 amplitudes, 128 GiB): two copies do not fit one
  B200, and the reference needs 2 x 128 GiB of host RAM (the GPU box has
  196 GB), so the single-GPU run is compared with the reference's own
  distributed protocol on 8 loopback ranks (``rank_apply_op`` per gate,
  distributed.cpp:128-233, swaps off; and the swap scheduler) through
  per-chunk 64-bit checksums of the raw amplitude bits (a random-weight
  linear hash: any difference changes it with probability ~1 - 2^-60).

Host RAM and time: C2 needs ~48 GiB of host memory and ~4 min of the
reference on 16 cores; C3a ~3 x 128 GiB of device passes and ~1 min of
hashing. Marked slow.
"""
import os

import numpy as np
import pytest

import oracle
from paper_1802_08032_b200 import circuits as C
from paper_1802_08032_b200 import quest
from tests.harness import to_oracle_ops

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CHUNK = 1 << 26  # amplitudes per host readback (1 GiB)
WORKERS = os.cpu_count() or 1


def _jit_run(env, n, circuit, jit_mode):
    """Runs `circuit` on a fresh register with the given JIT mode (0 off =
    interpreter, 2 sync = every pass shape compiled before its first launch)
    and returns the register (caller destroys)."""
    quest.set_jit(jit_mode)
    try:
        q = quest.QuregHandle(env, n)
        C.apply_circuit(q, circuit)
        q.flush()
        env.sync()
        return q
    finally:
        quest.set_jit(1)


def _compare_chunks(q, want):
    n_amp = want.size
    max_err = 0.0
    for s in range(0, n_amp, CHUNK):
        got = q.state(s, min(CHUNK, n_amp - s))
        ref = want[s:s + got.size]
        err = float(np.max(np.abs(got - ref)))
        max_err = max(max_err, err)
        assert np.array_equal(got, ref), f"amplitudes [{s}, {s + got.size}) differ (max-abs {err})"
    return max_err


@pytest.fixture(scope="module")
def env():
    e = quest.Env()
    yield e
    e.destroy()


def _sweep_circuit(n, seed=2024):
    """H on every qubit, then for every target t: H, Rx(theta), CNOT with
    the control above t, CNOT with the control below t, CPhase(theta) with a
    far control -- every stride, both control orders."""
    rng = np.random.default_rng(seed)
    c = C.Circuit(n, 0, [C.GateOp("H", q) for q in range(n)])
    for t in range(n):
        c.ops.append(C.GateOp("H", t))
        c.ops.append(C.GateOp("RX", t, angle=float(rng.uniform(0, 2 * np.pi))))
        c.ops.append(C.GateOp("X", t, ((t + 1) % n,)))
        c.ops.append(C.GateOp("X", t, ((t - 1) % n,)))
        c.ops.append(C.GateOp("PHASE", t, ((t + n // 2) % n,), angle=float(rng.uniform(0, 2 * np.pi))))
    return c


@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")
def test_30q_bench_circuit_against_reference(env):
    """C2: bench.py's workload (30 qubits, depth 20, seed 12345), every one of
    the 2^30 amplitudes bit-identical to the compiled reference, for the JIT
    kernels the bench times and for the interpreter."""
    n = 30
    c = C.layered_random_circuit(n, 20, 12345)
    assert len(c.ops) == 875
    want = oracle.ref_run(n, to_oracle_ops(c), workers=WORKERS)
    for mode in (2, 0):
        q = _jit_run(env, n, c, mode)
        try:
            assert _compare_chunks(q, want) <= 1e-12
        finally:
            q.destroy()


@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")
def test_30q_per_target_sweep_against_reference(env):
    """C2 sweep: H / Rx / CNOT (control above, below) / CPhase on every
    target 0..29 of a 30-qubit state, bit-identical to the compiled reference
    (JIT and interpreter)."""
    n = 30
    c = _sweep_circuit(n)
    want = oracle.ref_run(n, to_oracle_ops(c), workers=WORKERS)
    for mode in (2, 0):
        q = _jit_run(env, n, c, mode)
        try:
            assert _compare_chunks(q, want) <= 1e-12
        finally:
            q.destroy()


_W = None


def _chunk_hashes(q, n_amp, chunk=CHUNK):
    """64-bit random-weight linear hash of each chunk's raw amplitude bits."""
    global _W
    if _W is None or _W.size != 2 * chunk:
        _W = np.random.default_rng(0xC0FFEE).integers(0, 2**64, size=2 * chunk, dtype=np.uint64) | np.uint64(1)
    out = []
    for s in range(0, n_amp, chunk):
        a = q.state(s, min(chunk, n_amp - s))
        bits = a.view(np.uint64)
        with np.errstate(over="ignore"):
            out.append(int(np.sum(bits * _W[:bits.size], dtype=np.uint64)))
    return out


@pytest.mark.parametrize("swaps", [False, True])
def test_33q_single_gpu_equals_loopback_8(env, swaps):
    """C3a (33 qubits, 128 GiB): the single-GPU state equals, bit for bit,
    the state produced over 8 loopback ranks (30 local qubits each; gates on
    qubits 30-32 exchange with the partner rank as in rank_apply_op,
    distributed.cpp:128-233, or move through global<->local qubit swaps)."""
    n = 33
    c = C.layered_random_circuit(n, 3, 12345)
    q = quest.QuregHandle(env, n)
    try:
        C.apply_circuit(q, c)
        single = _chunk_hashes(q, 1 << n)
        assert abs(q.calcTotalProb() - 1.0) < 1e-12
    finally:
        q.destroy()
    lb = quest.Env.loopback(8)
    try:
        lb.set_qubit_swaps(swaps)
        q8 = quest.QuregHandle(lb, n)
        try:
            C.apply_circuit(q8, c)
            multi = _chunk_hashes(q8, 1 << n)
            assert abs(q8.calcTotalProb() - 1.0) < 1e-12
        finally:
            q8.destroy()
    finally:
        lb.destroy()
    diff = [i for i, (a, b) in enumerate(zip(single, multi)) if a != b]
    assert not diff, f"{len(diff)} of {len(single)} 1 GiB chunks differ (first {diff[:4]})"
