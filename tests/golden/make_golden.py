"""Generates the committed golden fixtures under tests/golden/ by running the
UNMODIFIED reference (oracle/_ref, compiled from /root/reference/proj by
oracle/Makefile). Run here (where /root/reference exists):

    python tests/golden/make_golden.py

Outputs
  spec_kats.json  SPEC.md known-answer examples on the hot path: each case's
                  expected amplitudes are written from the SPEC statement
                  (analytic) and asserted against the reference before saving.
  ref_vectors.npz reference outputs for small seeded workloads (state vector,
                  density matrix with channels, distributed accounting).
"""
from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_1802_08032_b200 import circuits as C  # noqa: E402
from tests.harness import random_gate_circuit, to_oracle_ops  # noqa: E402

HERE = Path(__file__).resolve().parent
S = 1 / math.sqrt(2)


def op(name, t, controls=(), angle=0.0, prob=0.0, matrix=None):
    return {"name": name, "target": t, "controls": list(controls), "angle": angle, "prob": prob,
            "matrix": matrix}


def amps(pairs, size):
    a = np.zeros(size, dtype=np.complex128)
    for i, v in pairs:
        a[i] = v
    return a


def kats():
    """(source, n, density, init, ops, expected, tol)."""
    cases = []
    add = lambda *c: cases.append(c)  # noqa: E731
    # core-state / gate-kernels examples
    add("SPEC.md:63 create (1, sv)", 1, False, None, [], amps([(0, 1)], 2), 0.0)
    add("SPEC.md:64 create (2, dm)", 2, True, None, [], amps([(0, 1)], 16), 0.0)
    add("SPEC.md:83 H then amp 1", 1, False, None, [op("H", 0)], amps([(0, S), (1, S)], 2), 0.0)
    add("SPEC.md:175 X on |0>", 1, False, None, [op("X", 0)], amps([(1, 1)], 2), 0.0)
    add("SPEC.md:176 H on |0>", 1, False, None, [op("H", 0)], amps([(0, S), (1, S)], 2), 0.0)
    bell = amps([(0, S), (3, S)], 4)
    add("SPEC.md:184 CZ on Bell", 2, False, bell, [op("Z", 0, (1,))], amps([(0, S), (3, -S)], 4), 0.0)
    add("SPEC.md:185 CNOT |10>", 2, False, amps([(2, 1)], 4), [op("X", 0, (1,))], amps([(3, 1)], 4), 0.0)
    add("SPEC.md:186 Toffoli |110>", 3, False, amps([(6, 1)], 8), [op("X", 0, (1, 2))], amps([(7, 1)], 8), 0.0)
    add("SPEC.md:193 T on |1>", 1, False, amps([(1, 1)], 2), [op("T", 0)],
        amps([(1, complex(math.cos(math.pi / 4), math.sin(math.pi / 4)))], 2), 0.0)
    add("SPEC.md:194 SX twice on |0>", 1, False, None, [op("SX", 0), op("SX", 0)], amps([(1, 1)], 2), 1e-12)
    rng = np.random.default_rng(195)
    psi = rng.normal(size=8) + 1j * rng.normal(size=8)
    add("SPEC.md:195 Rz(0) identity", 3, False, psi, [op("RZ", 1, angle=0.0)], psi, 1e-15)
    add("SPEC.md:202 angle 0 identity", 3, False, psi, [op("RX", 2, angle=0.0)], psi, 1e-15)
    add("SPEC.md:203 Rx(pi) |0> = -i|1>", 1, False, None, [op("RX", 0, angle=math.pi)], amps([(1, -1j)], 2), 1e-15)
    # density-noise examples
    add("SPEC.md:248 DM X on |0><0|", 1, True, None, [op("X", 0)], amps([(3, 1)], 4), 0.0)
    plus = amps([(0, 0.5), (1, 0.5), (2, 0.5), (3, 0.5)], 4)
    add("SPEC.md:257 dephase 1/2 on |+><+|", 1, True, plus, [op("DEPHASE", 0, prob=0.5)],
        amps([(0, 0.5), (3, 0.5)], 4), 0.0)
    add("SPEC.md:256 dephase 0 identity", 1, True, plus, [op("DEPHASE", 0, prob=0.0)], plus, 0.0)
    rho = np.array([0.7, 0.2 - 0.1j, 0.2 + 0.1j, 0.3], dtype=np.complex128)
    add("SPEC.md:266 depolarise 3/4 -> I/2", 1, True, rho, [op("DEPOL", 0, prob=0.75)],
        amps([(0, 0.5), (3, 0.5)], 4), 1e-15)
    add("SPEC.md:265 depolarise 0 identity", 1, True, rho, [op("DEPOL", 0, prob=0.0)], rho, 0.0)
    add("SPEC.md:247 DM identity gate", 2, True, None, [op("U", 1, matrix=[1, 0, 0, 0, 0, 0, 1, 0])],
        amps([(0, 1)], 16), 0.0)
    return cases


def to_circuit(n, ops_):
    c = C.Circuit(n, 0, [])
    for o in ops_:
        c.ops.append(C.GateOp(o["name"], o["target"], tuple(o["controls"]), angle=o["angle"],
                              matrix=tuple(o["matrix"]) if o["matrix"] else None, prob=o["prob"]))
    return c


def single_workloads():
    """name -> (num_qubits, density, circuit) for the single-precision vectors
    (shared with tests/test_golden.py)."""
    return {
        "sp_layered_n13_d5_s3": (13, False, C.layered_random_circuit(13, 5, 3)),
        "sp_random_n5_s99": (5, False, random_gate_circuit(5, 60, 99, max_controls=2)),
        "sp_dm_noisy_n6_d3_s5": (6, True, C.layered_random_circuit(6, 3, 5, noise_pmax=0.2)),
    }


def main():
    assert oracle.ref_available(), "build the reference first: make -C oracle ref"
    out = []
    for src, n, density, init, ops_, expected, tol in kats():
        got = oracle.ref_run(n, to_oracle_ops(to_circuit(n, ops_)), density=density, init=init)
        err = float(np.max(np.abs(got - expected)))
        assert err <= max(tol, 0.0) + 1e-16, (src, err)
        out.append({
            "source": src, "num_qubits": n, "density": density,
            "init": None if init is None else [[float(z.real), float(z.imag)] for z in init],
            "ops": ops_, "expected": [[float(z.real), float(z.imag)] for z in expected], "tol": tol,
        })
    (HERE / "spec_kats.json").write_text(json.dumps(out, indent=1))

    vec = {}
    c = C.layered_random_circuit(8, 6, 1)
    vec["sv_layered_n8_d6_s1"] = oracle.ref_run(8, to_oracle_ops(c))
    ops_, _ = oracle.ref_random_circuit(7, 10, 2)
    vec["sv_refgen_n7_d10_s2"] = oracle.ref_run(7, ops_)
    c = random_gate_circuit(6, 80, 424242, max_controls=3)
    vec["sv_random_n6_s424242"] = oracle.ref_run(6, to_oracle_ops(c))
    c = C.layered_random_circuit(3, 4, 5, noise_pmax=0.2)
    vec["dm_noisy_n3_d4_s5"] = oracle.ref_run(3, to_oracle_ops(c), density=True)
    c = random_gate_circuit(8, 40, 77, max_controls=2)
    st, msgs, byts, rounds = oracle.ref_run_distributed(8, to_oracle_ops(c), 2, "full_clone")
    vec["dist_n8_k2_s77_state"] = st
    vec["dist_n8_k2_s77_bytes"] = byts
    vec["dist_n8_k2_s77_msgs"] = msgs
    # Precision::Single (complex64): tiled (13 qubits; a 6-qubit density
    # matrix = 12 flat qubits) and small-state workloads
    for name, (n, density, c) in single_workloads().items():
        vec[name] = oracle.ref_run_single(n, to_oracle_ops(c), density=density)
    np.savez_compressed(HERE / "ref_vectors.npz", **vec)
    print(f"wrote {len(out)} KATs and {len(vec)} reference vectors")


if __name__ == "__main__":
    main()
