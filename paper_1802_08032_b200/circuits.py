"""Circuit IR, gate matrices and the seeded workload generators.

Workload plumbing around the hot path:

* ``gate_matrix`` / ``rotation_matrix`` restate gates.cpp:51-98 with the same
  expressions, so the doubles equal the reference's (pinned in
  tests/test_host_pins.py against the compiled reference).
* ``reference_random_circuit`` restates the reference generator
  (circuit.cpp:16-100: SplitMix64, H layer, period-3 CZ pattern, T/SX/SY with
  the first-T and no-repeat rules).
* ``layered_random_circuit`` is BASELINE.json config C1/C2 — H layer, then per
  layer a brickwork of alternating CNOT / CPhase(theta) and Rx/Ry/Rz(theta)
  on every qubit, theta = 2 pi u, u = (x >> 11) 2^-53 from the SplitMix64
  stream.
* ``qft_circuit`` is config C5.
* ``serialize`` / ``parse`` restate the reference text format
  (circuit.cpp:123-237).
* ``apply_circuit`` drives a register through the C-ABI, one QuEST call per op.
"""
from __future__ import annotations

import math
import re
from dataclasses import dataclass, field
from fractions import Fraction

MASK64 = (1 << 64) - 1


class SplitMix64:
    """circuit.cpp:16-34."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def below(self, n: int) -> int:
        return self.next() % n

    def uniform(self) -> float:
        return (self.next() >> 11) * 2.0 ** -53


# ------------------------------------------------------------------ matrices

def rotation_matrix(axis, angle: float) -> list[float]:
    """gates.cpp:85-98: cos(a/2) I - i sin(a/2) (n . sigma), as 8 doubles."""
    nx, ny, nz = (float(a) for a in axis)
    c, s = math.cos(angle / 2), math.sin(angle / 2)
    return [c, -s * nz, -s * ny, -s * nx, s * ny, -s * nx, c, s * nz]


def gate_matrix(name: str, angle: float = 0.0) -> list[float]:
    """gates.cpp:51-83 (+ S and PHASE, QuEST's sGate / phaseShift)."""
    if name == "H":
        s = 1.0 / math.sqrt(2.0)
        return [s, 0.0, s, 0.0, s, 0.0, -s, 0.0]
    if name == "T":
        return [1.0, 0.0, 0.0, 0.0, 0.0, 0.0, math.cos(math.pi / 4), math.sin(math.pi / 4)]
    if name == "X":
        return [0.0, 0.0, 1.0, 0.0, 1.0, 0.0, 0.0, 0.0]
    if name == "Y":
        return [0.0, 0.0, 0.0, -1.0, 0.0, 1.0, 0.0, 0.0]
    if name in ("Z", "CZ"):
        return [1.0, 0.0, 0.0, 0.0, 0.0, 0.0, -1.0, 0.0]
    if name == "S":
        return [1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 1.0]
    if name == "SX":
        return [0.5, 0.5, 0.5, -0.5, 0.5, -0.5, 0.5, 0.5]
    if name == "SY":
        return [0.5, 0.5, -0.5, -0.5, 0.5, 0.5, 0.5, 0.5]
    if name == "RX":
        return rotation_matrix((1, 0, 0), angle)
    if name == "RY":
        return rotation_matrix((0, 1, 0), angle)
    if name == "RZ":
        return rotation_matrix((0, 0, 1), angle)
    if name == "PHASE":
        return [1.0, 0.0, 0.0, 0.0, 0.0, 0.0, math.cos(angle), math.sin(angle)]
    raise ValueError(f"unknown gate name '{name}'")


# reference enum order (gates.hpp:30) for the compiled reference's gate ids
REF_GATE_IDS = {"H": 0, "T": 1, "CZ": 2, "SX": 3, "SY": 4, "RX": 5, "RY": 6, "RZ": 7, "X": 8, "Y": 9, "Z": 10}
HAS_ANGLE = {"RX", "RY", "RZ", "PHASE"}
CHANNELS = {"DEPHASE", "DEPOL"}


@dataclass
class GateOp:
    name: str
    target: int
    controls: tuple[int, ...] = ()
    angle: float = 0.0
    matrix: tuple[float, ...] | None = None  # name == "U"
    prob: float = 0.0  # channels

    def m8(self) -> list[float]:
        return list(self.matrix) if self.name == "U" else gate_matrix(self.name, self.angle)

    def ctrl_mask(self) -> int:
        m = 0
        for c in self.controls:
            m |= 1 << c
        return m


@dataclass
class Circuit:
    num_qubits: int
    depth: int = 0
    ops: list[GateOp] = field(default_factory=list)

    def __len__(self):
        return len(self.ops)


# ---------------------------------------------------------------- generators

def cz_layer_pairs(num_qubits: int, layer: int) -> list[tuple[int, int]]:
    """circuit.cpp:40-48."""
    if layer < 1:
        return []
    phase = (layer - 1) % 3
    return [(i, i + 1) for i in range(phase, num_qubits - 1, 3)]


def reference_random_circuit(num_qubits: int, depth: int, seed: int) -> Circuit:
    """circuit.cpp:50-100."""
    if num_qubits < 2:
        raise ValueError("random circuits need at least 2 qubits for the linear CZ pattern")
    if depth < 1:
        raise ValueError("circuit depth must be at least 1")
    rng = SplitMix64(seed)
    c = Circuit(num_qubits, depth, [GateOp("H", q) for q in range(num_qubits)])
    singles = ("T", "SX", "SY")
    prev = [-1] * num_qubits
    had_first_t = [False] * num_qubits
    for layer in range(1, depth):
        busy = [False] * num_qubits
        for a, b in cz_layer_pairs(num_qubits, layer):
            c.ops.append(GateOp("CZ", a, (b,)))
            busy[a] = busy[b] = True
        nxt = [-1] * num_qubits
        for q in range(num_qubits):
            if busy[q]:
                continue
            if not had_first_t[q]:
                choice = 0
                had_first_t[q] = True
            elif prev[q] == -1:
                choice = rng.below(3)
            else:
                choice = rng.below(2)
                if choice >= prev[q]:
                    choice += 1
            c.ops.append(GateOp(singles[choice], q))
            nxt[q] = choice
        prev = nxt
    return c


def layered_random_circuit(num_qubits: int, depth: int, seed: int, noise_pmax: float = 0.0) -> Circuit:
    """BASELINE.json C1/C2: layer 0 = H on every qubit;
    layer d >= 1 = brickwork on (q, q+1), q = d mod 2, q += 2, alternating
    CNOT(control q, target q+1) and CPhase(q, q+1, theta), then Rx/Ry/Rz(theta)
    on every qubit (kind = next() mod 3, theta = 2 pi u).

    noise_pmax > 0 gives config C4: after every layer, mixDephasing and
    mixDepolarising on every qubit with p = noise_pmax * u from a second
    SplitMix64 stream seeded with seed ^ 0xD1B54A32D192ED03."""
    rng = SplitMix64(seed)
    nrng = SplitMix64(seed ^ 0xD1B54A32D192ED03)
    c = Circuit(num_qubits, depth, [])

    def noise():
        if noise_pmax > 0:
            for q in range(num_qubits):
                c.ops.append(GateOp("DEPHASE", q, prob=noise_pmax * nrng.uniform()))
                c.ops.append(GateOp("DEPOL", q, prob=noise_pmax * nrng.uniform()))

    c.ops.extend(GateOp("H", q) for q in range(num_qubits))
    noise()
    for d in range(1, depth):
        for j, q in enumerate(range(d % 2, num_qubits - 1, 2)):
            if j % 2 == 0:
                c.ops.append(GateOp("X", q + 1, (q,)))
            else:
                c.ops.append(GateOp("PHASE", q, (q + 1,), angle=2 * math.pi * rng.uniform()))
        for q in range(num_qubits):
            kind = ("RX", "RY", "RZ")[rng.next() % 3]
            c.ops.append(GateOp(kind, q, angle=2 * math.pi * rng.uniform()))
        noise()
    return c


def qft_circuit(num_qubits: int, mcpf_every: int = 0, seed: int = 1) -> Circuit:
    """Config C5: QFT (H + controlledPhaseShift(pi / 2^k) ladder, no final
    swaps); optionally a multiControlledPhaseFlip on 3-5 seeded qubits after
    every `mcpf_every` stages."""
    rng = SplitMix64(seed)
    c = Circuit(num_qubits, 0, [])
    for stage, j in enumerate(range(num_qubits - 1, -1, -1)):
        c.ops.append(GateOp("H", j))
        for k in range(j - 1, -1, -1):
            c.ops.append(GateOp("PHASE", j, (k,), angle=math.pi / (1 << (j - k))))
        if mcpf_every and (stage + 1) % mcpf_every == 0 and num_qubits >= 5:
            m = 3 + rng.below(3)
            qs = []
            while len(qs) < m:
                q = rng.below(num_qubits)
                if q not in qs:
                    qs.append(q)
            c.ops.append(GateOp("Z", qs[-1], tuple(qs[:-1])))
    return c


def gate_counts(circuit: Circuit) -> tuple[int, int]:
    """circuit.cpp:102-111: (single, controlled)."""
    single = sum(1 for op in circuit.ops if not op.controls and op.name not in CHANNELS)
    return single, sum(1 for op in circuit.ops if op.controls)


# ------------------------------------------------------------- text format

_TEXT_NAMES = {"H", "T", "CZ", "SX", "SY", "RX", "RY", "RZ", "X", "Y", "Z"}


class ParseError(ValueError):
    pass


def _format_angle(x: float) -> str:
    """circuit.cpp:104-110: printf("%.17g"); glibc prints a NaN's sign."""
    if math.isnan(x):
        return "-nan" if math.copysign(1.0, x) < 0 else "nan"
    return "%.17g" % x


def serialize(circuit: Circuit) -> str:
    """circuit.cpp:123-136 (reference gate set only)."""
    lines = [f"qubits {circuit.num_qubits} depth {circuit.depth}"]
    for op in circuit.ops:
        if op.name not in _TEXT_NAMES:
            raise ValueError(f"gate {op.name} has no text form")
        parts = [op.name, str(op.target), *map(str, op.controls)]
        if op.name in HAS_ANGLE:
            parts.append(_format_angle(float(op.angle)))
        lines.append(" ".join(parts))
    return "\n".join(lines) + "\n"


# std::from_chars<int> (circuit.cpp:144-151): optional '-', ASCII digits, int32
_INT_RE = re.compile(r"-?[0-9]+")
# std::stod = strtod's longest prefix (circuit.cpp:153-167): hex, decimal,
# inf/infinity, nan(n-char-sequence); ERANGE (overflow, or a tiny inexact
# result) -> out_of_range; no prefix -> invalid_argument; a prefix shorter
# than the token -> "expected a number"
_STOD_RES = (
    re.compile(r"[+-]?0[xX](?:[0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)(?:[pP][+-]?[0-9]+)?"),
    re.compile(r"[+-]?(?:[0-9]+\.?[0-9]*|\.[0-9]+)(?:[eE][+-]?[0-9]+)?"),
    re.compile(r"[+-]?inf(?:inity)?", re.IGNORECASE),
    re.compile(r"[+-]?nan(?:\([0-9A-Za-z_]*\))?", re.IGNORECASE),
)
_DBL_MIN = Fraction(2) ** -1022


def _exact_hex(tok: str) -> Fraction:
    sign = -1 if tok[0] == "-" else 1
    body = tok.lstrip("+-")[2:]
    mant, _, exp = body.replace("P", "p").partition("p")
    whole, _, frac = mant.partition(".")
    digits = whole + frac
    return sign * Fraction(int(digits, 16)) * Fraction(2) ** (int(exp or 0) - 4 * len(frac))


def _parse_int(tok: str, line: int) -> int:
    if not _INT_RE.fullmatch(tok) or not -(1 << 31) <= int(tok) < (1 << 31):
        raise ParseError(f"line {line}: expected an integer, got '{tok}'")
    return int(tok)


def _parse_double(tok: str, line: int) -> float:
    m = None
    for r in _STOD_RES:
        m = r.match(tok)
        if m:
            break
    if not m:
        raise ParseError(f"line {line}: expected a number, got '{tok}'")
    pre = m.group(0)
    low = pre.lower().lstrip("+-")
    erange = False
    if low.startswith("inf") or low.startswith("nan"):
        value = float(pre.split("(")[0])
    else:
        hexa = low.startswith("0x")
        exact = _exact_hex(pre) if hexa else Fraction(pre)
        try:
            value = float.fromhex(pre) if hexa else float(pre)
        except OverflowError:
            value, erange = math.inf, True
        if math.isinf(value):
            erange = True
        elif exact != 0 and abs(exact) < _DBL_MIN and Fraction(value) != exact:
            erange = True
    if erange:
        raise ParseError(f"line {line}: number out of range: '{tok}'")
    if len(pre) != len(tok):
        raise ParseError(f"line {line}: expected a number, got '{tok}'")
    return value


def parse(text: str) -> Circuit:
    """circuit.cpp:172-237: std::getline lines ('\\n' only), tokens split on
    C-locale whitespace, '#' starts a comment only at a token's start; the
    reference's messages and check order."""
    circuit = None
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    line_no = 0
    for line_no, line in enumerate(lines, 1):
        toks = []
        for t in re.split(r"[ \t\n\v\f\r]+", line):
            if not t:
                continue
            if t.startswith("#"):
                break
            toks.append(t)
        if not toks:
            continue
        if circuit is None:
            if len(toks) != 4 or toks[0] != "qubits" or toks[2] != "depth":
                raise ParseError(f"line {line_no}: expected header 'qubits N depth D'")
            n = _parse_int(toks[1], line_no)
            d = _parse_int(toks[3], line_no)
            if n < 1:
                raise ParseError(f"line {line_no}: qubit count must be positive")
            circuit = Circuit(n, d, [])
            continue
        name = toks[0]
        if name not in _TEXT_NAMES:
            raise ParseError(f"line {line_no}: unknown gate name '{name}'")
        angled = name in HAS_ANGLE
        if len(toks) < 2 or (angled and len(toks) < 3):
            raise ParseError(f"line {line_no}: missing operands for {name}")
        target = _parse_int(toks[1], line_no)
        ctrl_end = len(toks) - (1 if angled else 0)
        controls = tuple(_parse_int(t, line_no) for t in toks[2:ctrl_end])
        angle = _parse_double(toks[-1], line_no) if angled else 0.0
        if not 0 <= target < circuit.num_qubits:
            raise ParseError(f"line {line_no}: target {target} out of range for {circuit.num_qubits} qubits")
        for c in controls:
            if not 0 <= c < circuit.num_qubits:
                raise ParseError(f"line {line_no}: control {c} out of range")
            if c == target:
                raise ParseError(f"line {line_no}: control overlaps target")
        circuit.ops.append(GateOp(name, target, controls, angle))
    if circuit is None:
        raise ParseError(f"line {line_no + 1}: missing 'qubits N depth D' header")
    return circuit


# ------------------------------------------------------- C-ABI application

def apply_op(q, op: GateOp):
    """One QuEST call per op on a ``quest.QuregHandle`` (QuEST names)."""
    from . import quest

    n, t, cs = op.name, op.target, op.controls
    if n == "DEPHASE":
        return q.mixDephasing(t, op.prob)
    if n == "DEPOL":
        return q.mixDepolarising(t, op.prob)
    if not cs:
        simple = {"H": "hadamard", "X": "pauliX", "Y": "pauliY", "Z": "pauliZ", "T": "tGate", "S": "sGate"}
        if n in simple:
            return getattr(q, simple[n])(t)
        if n in ("RX", "RY", "RZ"):
            return getattr(q, "rotate" + n[1])(t, op.angle)
        if n == "PHASE":
            return q.phaseShift(t, op.angle)
        return q.unitary(t, quest.cmatrix2(op.m8()))
    if len(cs) == 1:
        c = cs[0]
        if n == "X":
            return q.controlledNot(c, t)
        if n == "Y":
            return q.controlledPauliY(c, t)
        if n in ("Z", "CZ"):
            return q.controlledPhaseFlip(t, c)
        if n == "PHASE":
            return q.controlledPhaseShift(t, c, op.angle)
        if n in ("RX", "RY", "RZ"):
            return getattr(q, "controlledRotate" + n[1])(c, t, op.angle)
        return q.controlledUnitary(c, t, quest.cmatrix2(op.m8()))
    arr, k = quest.int_array(list(cs) + [t])
    if n in ("Z", "CZ"):
        return q.multiControlledPhaseFlip(arr, k)
    if n == "PHASE":
        return q.multiControlledPhaseShift(arr, k, op.angle)
    carr, kc = quest.int_array(list(cs))
    return q.multiControlledUnitary(carr, kc, t, quest.cmatrix2(op.m8()))


def apply_circuit(q, circuit: Circuit):
    """One QuEST C-ABI call per op (the per-gate entry points)."""
    for op in circuit.ops:
        apply_op(q, op)


# qgpuOp (include/qgpu.h): 96-byte records, kind 0 gate / 1 dephase / 2 depolarise
OP_DTYPE = [("kind", "<i4"), ("target", "<i4"), ("ctrl_mask", "<u8"), ("m", "<f8", (8,)),
            ("prob", "<f8"), ("reserved", "<f8")]


def op_array(circuit: Circuit):
    """The circuit as a qgpuOp array for qgpuRunCircuit."""
    import numpy as np

    a = np.zeros(len(circuit.ops), dtype=np.dtype(OP_DTYPE, align=False))
    for i, op in enumerate(circuit.ops):
        if op.name == "DEPHASE":
            a[i] = (1, op.target, 0, np.zeros(8), op.prob, 0.0)
        elif op.name == "DEPOL":
            a[i] = (2, op.target, 0, np.zeros(8), op.prob, 0.0)
        else:
            a[i] = (0, op.target, op.ctrl_mask(), np.array(op.m8()), 0.0, 0.0)
    return a


def run_circuit(q, circuit: Circuit):
    """run_circuit (circuit.cpp:239-247) as one C-ABI call
    (qgpuRunCircuit): all ops validated first, then queued."""
    q.run_ops(op_array(circuit))


def dagger(op: GateOp) -> GateOp:
    """The inverse gate (same controls)."""
    if op.name in ("H", "X", "Y", "Z", "CZ"):
        return op
    if op.name in ("RX", "RY", "RZ", "PHASE"):
        return GateOp(op.name, op.target, op.controls, angle=-op.angle)
    m = op.m8()
    # conjugate transpose of [[a, b], [c, d]]
    inv = [m[0], -m[1], m[4], -m[5], m[2], -m[3], m[6], -m[7]]
    return GateOp("U", op.target, op.controls, matrix=tuple(inv))


def inverse_circuit(circuit: Circuit) -> Circuit:
    if any(op.name in CHANNELS for op in circuit.ops):
        raise ValueError("channels have no inverse")
    return Circuit(circuit.num_qubits, circuit.depth, [dagger(op) for op in reversed(circuit.ops)])
