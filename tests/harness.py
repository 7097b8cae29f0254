"""Test harness: converts circuits to the checkers' op records and drives the
product through the C-ABI. Used only by tests/ (and smoke())."""
from __future__ import annotations

import numpy as np

import oracle
from paper_1802_08032_b200 import circuits as C


def to_oracle_ops(circuit: C.Circuit) -> np.ndarray:
    ops = np.zeros(len(circuit.ops), dtype=oracle.OP_DTYPE)
    for i, op in enumerate(circuit.ops):
        if op.name == "DEPHASE":
            ops[i] = (oracle.DEPHASE, op.target, 0, np.zeros(8), op.prob, 0.0)
        elif op.name == "DEPOL":
            ops[i] = (oracle.DEPOLARISE, op.target, 0, np.zeros(8), op.prob, 0.0)
        else:
            ops[i] = (oracle.GATE, op.target, op.ctrl_mask(), np.array(op.m8()), 0.0, 0.0)
    return ops


def random_unitary(rng: np.random.Generator) -> list[float]:
    z = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
    q, r = np.linalg.qr(z)
    q = q * (np.diag(r) / np.abs(np.diag(r)))
    return [q[0, 0].real, q[0, 0].imag, q[0, 1].real, q[0, 1].imag,
            q[1, 0].real, q[1, 0].imag, q[1, 1].real, q[1, 1].imag]


def random_gate_circuit(n: int, count: int, seed: int, max_controls: int = 2,
                        channels: bool = False, names=None) -> C.Circuit:
    """Random mix of named gates, random unitaries ("U") and controls."""
    rng = np.random.default_rng(seed)
    names = names or ["H", "X", "Y", "Z", "T", "S", "SX", "SY", "RX", "RY", "RZ", "PHASE", "U"]
    c = C.Circuit(n, 0, [])
    for _ in range(count):
        t = int(rng.integers(n))
        if channels and rng.random() < 0.25:
            if rng.random() < 0.5:
                c.ops.append(C.GateOp("DEPHASE", t, prob=float(rng.uniform(0, 0.5))))
            else:
                c.ops.append(C.GateOp("DEPOL", t, prob=float(rng.uniform(0, 0.75))))
            continue
        others = [q for q in range(n) if q != t]
        k = int(rng.integers(0, min(max_controls, len(others)) + 1))
        ctrls = tuple(int(x) for x in rng.choice(others, size=k, replace=False)) if k else ()
        name = str(rng.choice(names))
        angle = float(rng.uniform(-2 * np.pi, 2 * np.pi))
        if name == "U":
            c.ops.append(C.GateOp("U", t, ctrls, matrix=tuple(random_unitary(rng))))
        else:
            c.ops.append(C.GateOp(name, t, ctrls, angle=angle))
    return c


def oracle_run(circuit: C.Circuit, density: bool = False, init=None) -> np.ndarray:
    return oracle.orc_run(circuit.num_qubits, to_oracle_ops(circuit), density=density, init=init)


def bits_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """Bit-identical up to the sign of zero."""
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return bool(np.array_equal(a, b))
