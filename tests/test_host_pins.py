"""Host-side pieces pinned to the compiled reference (CPU only).

* Gate matrices: ``circuits.gate_matrix`` / ``rotation_matrix`` equal the
  reference's ``gate_matrix`` / ``rotation_matrix`` (gates.cpp:51-98) double
  for double, on the fixed gates and on random angles and axes.
* Text format: ``circuits.serialize`` / ``parse`` against the reference's
  ``serialize`` / ``parse`` (circuit.cpp:123-237) on the same text -- the
  SPEC.md:459-461 known answers, round trips of generated circuits, and a
  seeded corpus of malformed and edge-case lines whose error messages
  ("line N: ...") must match the reference's exactly.
"""
import math

import numpy as np
import pytest

import oracle
from paper_1802_08032_b200 import circuits as C

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not present")


def _same(a, b):
    return all(x == y and math.copysign(1, x) == math.copysign(1, y) for x, y in zip(a, b))


@needs_ref
def test_fixed_gate_matrices_equal_reference():
    for name, gid in C.REF_GATE_IDS.items():
        if name in ("RX", "RY", "RZ"):
            continue
        assert _same(C.gate_matrix(name), oracle.ref_gate_matrix(gid)), name


@needs_ref
def test_rotation_matrices_equal_reference_on_random_angles():
    rng = np.random.default_rng(85)
    angles = list(rng.uniform(-4 * np.pi, 4 * np.pi, 200)) + [0.0, -0.0, np.pi, -np.pi, 2 * np.pi, 1e-300, 1e300]
    for a in angles:
        for name, axis in (("RX", (1, 0, 0)), ("RY", (0, 1, 0)), ("RZ", (0, 0, 1))):
            want = oracle.ref_gate_matrix(C.REF_GATE_IDS[name], float(a))
            assert _same(C.gate_matrix(name, float(a)), want), (name, a)
            assert _same(C.rotation_matrix(axis, float(a)), want), (name, a)
    for _ in range(200):  # arbitrary unit axes (apply_single_qubit_rotation)
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        a = float(rng.uniform(-10, 10))
        assert _same(C.rotation_matrix(v, a), oracle.ref_rotation_matrix(v, a))


# ------------------------------------------------------------ text format

def _ours(text):
    """serialize(parse(text)) or the parse error message."""
    try:
        return C.serialize(C.parse(text))
    except C.ParseError as e:
        return "ERR " + str(e)


def _theirs(text):
    try:
        return oracle.ref_parse_serialize(text)
    except oracle.OracleError as e:
        assert e.code == 4, e  # ParseError
        return "ERR " + e.msg


def test_spec_known_answers():
    # SPEC.md:459-461
    c = C.parse("qubits 2 depth 1\nH 0\nCZ 0 1\n")
    assert c.num_qubits == 2 and c.depth == 1 and len(c.ops) == 2
    assert c.ops[1] == C.GateOp("CZ", 0, (1,))
    with pytest.raises(C.ParseError, match=r"^line 2: "):
        C.parse("qubits 2 depth 1\nH 9\n")
    rng = np.random.default_rng(5)  # round trip of a random n=5 circuit
    c = C.Circuit(5, 3, [])
    for _ in range(40):
        name = str(rng.choice(sorted(C._TEXT_NAMES)))
        t = int(rng.integers(5))
        ctrl = tuple(int(q) for q in rng.choice([q for q in range(5) if q != t], size=int(rng.integers(0, 3)),
                                                replace=False))
        angle = float(rng.uniform(-7, 7)) if name in C.HAS_ANGLE else 0.0
        c.ops.append(C.GateOp(name, t, ctrl, angle))
    assert C.parse(C.serialize(c)) == c


@needs_ref
@pytest.mark.parametrize("n,d,seed", [(2, 1, 0), (5, 10, 1), (7, 13, 12345), (30, 100, 2)])
def test_serialize_generated_circuit_equals_reference(n, d, seed):
    text = oracle.ref_serialize_random(n, d, seed)
    assert C.serialize(C.reference_random_circuit(n, d, seed)) == text
    assert C.serialize(C.parse(text)) == text


EDGE = [
    "", "\n", "\n\n", "# only a comment\n", "qubits 2 depth 1", "qubits 2 depth 1\n",
    "qubits 0 depth 1\n", "qubits -3 depth 1\n", "qubits 2 depth -5\n", "qubits +2 depth 1\n",
    "qubits 2 depth 99999999999\n", "qubits 2 depth 2147483647\n", "qubits 2 depth -2147483648\n",
    "qubits 2 depth 1.0\n", "qubits 2 depth 0x1\n", "qubits 2\n", "qubits 2 depth 1 extra\n",
    "qubit 2 depth 1\n", "  qubits\t2 depth\v1 # c\nH 0\n", "qubits 2 depth 1 #x\nH 1#c\n",
    "qubits 2 depth 1\nH 9\n", "qubits 2 depth 1\nH -1\n", "qubits 2 depth 1\nH\n", "qubits 2 depth 1\nRX 1\n",
    "qubits 2 depth 1\nFOO 1\n", "qubits 2 depth 1\nh 1\n", "qubits 2 depth 1\nH 1 0 1\n",
    "qubits 2 depth 1\nH 1 1\n", "qubits 2 depth 1\nCZ 0 7\n", "qubits 3 depth 1\nCZ 0 1 2\n",
    "qubits 2 depth 1\nRX 1 0 0.5\n", "qubits 2 depth 1\r\nH 0\r\n", "qubits 2 depth 1\n\n\nH 0\n\nFOO\n",
    "qubits 2 depth 1\nH 0\nqubits 2 depth 1\n", "qubits 2 depth 1\nH 00001\n", "qubits 2 depth 1\nH +1\n",
    "qubits 2 depth 1\nH 0x1\n", "qubits 2 depth 1\nH 1.0\n",
] + ["qubits 2 depth 1\nRX 1 " + v + "\n" for v in [
    "0.5", "-0", "-0.0", "1e308", "1.8e308", "1e999", "1e999x", "1e-310", "4.9e-324", "1e-400", "0e-999",
    "2.2250738585072014e-308", "2.2250738585072011e-308", "1.7976931348623158e308", "+0x1p3", "0X.8P1",
    "0x1p-1074", "0x1p-1080", "0x1p1024", "0x1.fffffffffffffp1023", "0x", "0x.", "0xp1", "1e", "1e+", "1e+5x",
    ".", "1.", ".5e+1", "00012", "1_0", "inf", "INF", "inFinity", "-inf", "infx", "infinit", "nan", "-nan",
    "+nan", "nan()", "nan(a_b)", "nan(a-b)", "NaN(123)", "1e5", "1E5", "6.283185307179586", "0.1", "1/2",
    "--1", "+-1", "١", "3.14159265358979323846264338327950288",
]]


@needs_ref
@pytest.mark.parametrize("text", EDGE)
def test_parse_edge_cases_match_reference(text):
    assert _ours(text) == _theirs(text)


@needs_ref
def test_parse_fuzz_matches_reference():
    """Seeded mutations of valid circuits: same output or same error."""
    rng = np.random.default_rng(1802)
    alphabet = list("0123456789 \t\n#-+.eEpPxXinfaINFA_HTCZSXYRrz()")
    base = C.serialize(C.reference_random_circuit(6, 6, 3)) + "RX 2 0.25\nRY 3 1 -1.5e-3\nRZ 0 2 4 3.0\n"
    for _ in range(400):
        t = list(base)
        for _ in range(int(rng.integers(1, 4))):
            i = int(rng.integers(len(t)))
            r = rng.random()
            if r < 0.4:
                t[i] = str(rng.choice(alphabet))
            elif r < 0.7:
                del t[i]
            else:
                t.insert(i, str(rng.choice(alphabet)))
        text = "".join(t)
        assert _ours(text) == _theirs(text), repr(text)
