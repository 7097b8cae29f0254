"""The reorder scheduler on the host (qgpuPlanPasses dry runs, no GPU).

Env ordering 1 (the library default) cuts passes by commutation instead of
by circuit position (runtime.cpp `window_pass`). These tests pin, on CPU:

* every executed order respects "must precede": ops that share a qubit on
  which either acts non-diagonally keep their circuit order;
* replaying the executed order through the C restatement of the reference
  (oracle/qsim_oracle.c, the reference's fma chain) gives the circuit-order
  state within 1e-12 (commuting ops reorder only the rounding);
* ordering 0 executes the circuit order exactly;
* the bench circuit (30 qubits, depth 20, seed 12345) needs 3x fewer HBM
  passes than in circuit order.
"""
import numpy as np
import pytest

import oracle
from paper_1802_08032_b200 import circuits as C
from paper_1802_08032_b200 import quest
from tests.harness import random_gate_circuit, to_oracle_ops

DIAG = {"Z", "S", "T", "RZ", "PHASE"}


def flat_ops(circuit: C.Circuit, density: bool = False):
    """The physical ops the C-ABI queues (api.cpp: a density-matrix gate is G
    at t and conj(G) at t + N with the controls shifted, density.cpp:85-116)."""
    n = circuit.num_qubits
    out = []
    for op in circuit.ops:
        if op.name == "DEPHASE":
            out.append((1, op.target, op.target + n, 0, None))
        elif op.name == "DEPOL":
            out.append((2, op.target, op.target + n, 0, None))
        else:
            m = op.m8()
            out.append((0, op.target, -1, op.ctrl_mask(), m))
            if density:
                conj = [m[0], -m[1], m[2], -m[3], m[4], -m[5], m[6], -m[7]]
                out.append((0, op.target + n, -1, op.ctrl_mask() << n, conj))
    return out


def acts(op):
    """(non-diagonal, X-type, diagonal) qubit masks of an op: two ops commute
    when every qubit they share is diagonal in both or X-type ([[a, b], [b,
    a]]: X / CNOT targets, Rx) in both (runtime.cpp op_qubits)."""
    kind, q0, q1, cmask, m = op
    nd, nx, dg = 0, 0, 0
    if kind == 0:
        dg = cmask
        diag = m[2] == 0 and m[3] == 0 and m[4] == 0 and m[5] == 0
        if diag:
            dg |= 1 << q0
        elif m[0] == m[6] and m[1] == m[7] and m[2] == m[4] and m[3] == m[5]:
            nx |= 1 << q0
        else:
            nd |= 1 << q0
    elif kind == 2:
        nd = (1 << q0) | (1 << q1)
    else:
        dg = (1 << q0) | ((1 << q1) if q1 >= 0 else 0)
    return nd, nx, dg


def commute(a, b):
    nda, nxa, dga = a
    ndb, nxb, dgb = b
    return not ((nda & (ndb | nxb | dgb)) or (nxa & (ndb | dgb)) or (dga & (ndb | nxb)))


def assert_respects_dependencies(ops, order):
    pos = np.empty(len(ops), dtype=np.int64)
    pos[order] = np.arange(len(ops))
    a = [acts(o) for o in ops]
    for j in range(len(ops)):
        for i in range(j):
            if not commute(a[i], a[j]):
                assert pos[i] < pos[j], f"op {j} ran before op {i} it does not commute with"


def circuits():
    yield "layered16", C.layered_random_circuit(16, 12, 7), False
    yield "random14", random_gate_circuit(14, 300, seed=5, max_controls=3), False
    yield "random13_channels", random_gate_circuit(7, 200, seed=9, max_controls=2, channels=True), True
    yield "qft16", C.qft_circuit(16, mcpf_every=3), False
    yield "refgen18", C.reference_random_circuit(18, 20, 3), False


@pytest.mark.parametrize("window", [8, 64, 512])
@pytest.mark.parametrize("name,circuit,density", list(circuits()), ids=[c[0] for c in circuits()])
def test_plan_respects_dependencies(name, circuit, density, window):
    ops = flat_ops(circuit, density)
    flat = circuit.num_qubits * (2 if density else 1)
    order, passes, phases = quest.plan_passes(flat, ops, reorder=True, window=window)
    assert sorted(order.tolist()) == list(range(len(ops)))
    assert_respects_dependencies(ops, order)
    # passes and phases are contiguous and non-decreasing in execution order
    assert np.all(np.diff(passes) >= 0)
    same = np.diff(passes) == 0
    assert np.all(np.diff(phases)[same] >= 0)
    assert phases.max() < 3


@pytest.mark.parametrize("name,circuit,density", [c for c in circuits() if not c[2]],
                         ids=[c[0] for c in circuits() if not c[2]])
def test_plan_replay_matches_circuit_order(name, circuit, density):
    ops = flat_ops(circuit)
    order, _, _ = quest.plan_passes(circuit.num_qubits, ops, reorder=True)
    orc = to_oracle_ops(circuit)
    want = oracle.orc_run(circuit.num_qubits, orc)
    got = oracle.orc_run(circuit.num_qubits, orc[order])
    assert float(np.max(np.abs(got - want))) <= 1e-12


def test_exact_ordering_keeps_circuit_order():
    c = random_gate_circuit(15, 400, seed=3, max_controls=3)
    order, passes, _ = quest.plan_passes(15, flat_ops(c), reorder=False)
    assert order.tolist() == list(range(len(c.ops)))


def test_bench_circuit_needs_fewer_passes():
    c = C.layered_random_circuit(30, 20, 12345)
    ops = flat_ops(c)
    _, p_exact, _ = quest.plan_passes(30, ops, reorder=False)
    _, p_reorder, _ = quest.plan_passes(30, ops, reorder=True)
    n_exact, n_reorder = int(p_exact.max()) + 1, int(p_reorder.max()) + 1
    assert n_exact == 66
    assert n_reorder <= 21, n_reorder
