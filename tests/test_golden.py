"""Committed golden fixtures (tests/golden/, made by make_golden.py from the
compiled reference): SPEC.md known answers and reference output vectors.
CPU: the oracle restatement reproduces them. GPU: the product does."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_1802_08032_b200 import circuits as C
from tests.harness import random_gate_circuit, to_oracle_ops

GOLD = Path(__file__).resolve().parent / "golden"
KATS = json.loads((GOLD / "spec_kats.json").read_text())
VEC = dict(np.load(GOLD / "ref_vectors.npz"))


def _c(a):
    return None if a is None else np.array([complex(x, y) for x, y in a], dtype=np.complex128)


def _circuit(case):
    c = C.Circuit(case["num_qubits"], 0, [])
    for o in case["ops"]:
        c.ops.append(C.GateOp(o["name"], o["target"], tuple(o["controls"]), angle=o["angle"],
                              matrix=tuple(o["matrix"]) if o["matrix"] else None, prob=o["prob"]))
    return c


def _workloads():
    """name -> (num_qubits, density, circuit-or-ops)."""
    ops_refgen, _ = (None, None)
    return {
        "sv_layered_n8_d6_s1": (8, False, C.layered_random_circuit(8, 6, 1)),
        "sv_refgen_n7_d10_s2": (7, False, C.reference_random_circuit(7, 10, 2)),
        "sv_random_n6_s424242": (6, False, random_gate_circuit(6, 80, 424242, max_controls=3)),
        "dm_noisy_n3_d4_s5": (3, True, C.layered_random_circuit(3, 4, 5, noise_pmax=0.2)),
    }


@pytest.mark.parametrize("case", KATS, ids=[k["source"] for k in KATS])
def test_oracle_reproduces_spec_kats(case):
    got = oracle.orc_run(case["num_qubits"], to_oracle_ops(_circuit(case)), density=case["density"],
                         init=_c(case["init"]))
    assert np.max(np.abs(got - _c(case["expected"]))) <= case["tol"] + 1e-16


@pytest.mark.parametrize("name", list(_workloads()))
def test_oracle_reproduces_reference_vectors(name):
    n, density, c = _workloads()[name]
    assert np.array_equal(oracle.orc_run(n, to_oracle_ops(c), density=density), VEC[name])


def test_distributed_accounting_vector():
    # full_clone: one message of 16 * 2^(n-k) bytes per rank per communicated gate
    c = random_gate_circuit(8, 40, 77, max_controls=2)
    assert np.array_equal(oracle.orc_run(8, to_oracle_ops(c)), VEC["dist_n8_k2_s77_state"])
    assert set(VEC["dist_n8_k2_s77_bytes"] % (16 * 64)) == {0}


@pytest.mark.gpu
@pytest.mark.parametrize("case", KATS, ids=[k["source"] for k in KATS])
def test_product_reproduces_spec_kats(case):
    from paper_1802_08032_b200 import quest

    env = quest.Env()
    try:
        q = quest.QuregHandle(env, case["num_qubits"], case["density"])
        if case["init"] is not None:
            q.set_state(_c(case["init"]))
        C.apply_circuit(q, _circuit(case))
        assert np.max(np.abs(q.state() - _c(case["expected"]))) <= case["tol"] + 1e-16
        q.destroy()
    finally:
        env.destroy()


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(_workloads()))
def test_product_reproduces_reference_vectors(name):
    from paper_1802_08032_b200 import quest

    n, density, c = _workloads()[name]
    env = quest.Env()
    try:
        q = quest.QuregHandle(env, n, density)
        C.apply_circuit(q, c)
        assert np.array_equal(q.state(), VEC[name])
        q.destroy()
    finally:
        env.destroy()


@pytest.mark.gpu
def test_product_distributed_vector_loopback():
    from paper_1802_08032_b200 import quest

    env = quest.Env.loopback(4)
    try:
        q = quest.QuregHandle(env, 8)
        C.apply_circuit(q, random_gate_circuit(8, 40, 77, max_controls=2))
        assert np.array_equal(q.state(), VEC["dist_n8_k2_s77_state"])
        q.destroy()
    finally:
        env.destroy()


def _single_workloads():
    import importlib.util

    spec = importlib.util.spec_from_file_location("make_golden", GOLD / "make_golden.py")
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    return mg.single_workloads()


@pytest.mark.parametrize("name", ["sp_layered_n13_d5_s3", "sp_random_n5_s99", "sp_dm_noisy_n6_d3_s5"])
def test_oracle_reproduces_single_precision_vectors(name):
    """The float restatement reproduces the reference's Precision::Single
    outputs committed in tests/golden (complex64, bit for bit)."""
    n, density, c = _single_workloads()[name]
    assert VEC[name].dtype == np.complex64
    assert np.array_equal(oracle.orc_run_f(n, to_oracle_ops(c), density), VEC[name])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["sp_layered_n13_d5_s3", "sp_random_n5_s99", "sp_dm_noisy_n6_d3_s5"])
def test_product_reproduces_single_precision_vectors(name):
    from paper_1802_08032_b200 import quest

    n, density, c = _single_workloads()[name]
    env = quest.Env()
    try:
        q = quest.QuregHandle(env, n, density, precision="single")
        C.run_circuit(q, c)
        assert np.array_equal(q.state(), VEC[name].astype(np.complex128))
        q.destroy()
    finally:
        env.destroy()
