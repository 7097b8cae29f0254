"""The reference's C++ operation names (namespace qsim, /root/reference/proj)
re-exposed over the B200 C-ABI, so code and tests written against the
reference read the same here. Every call goes to libqgpu.so; nothing here
computes amplitudes.

    reg = Register(12)                              # register.hpp:51-86
    apply_named_gate(reg, NamedGate("H"), [], 0)    # kernels.cpp:114-122
    apply_controlled_gate(reg, [3], 0, gate_matrix(NamedGate("X")))
    run_circuit(generate_random_circuit(12, 10, 1), reg)

Errors mirror the reference's exception classes (types.hpp:31-55) and are
raised before any mutation.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import circuits as C
from . import quest
from .quest import CommError, DomainError, ResourceError  # noqa: F401

STATE_VECTOR = "statevector"
DENSITY_MATRIX = "density"

_default_env: quest.Env | None = None


def default_env() -> quest.Env:
    global _default_env
    if _default_env is None:
        _default_env = quest.Env()
    return _default_env


# ------------------------------------------------------------------ gates

@dataclass
class GateMatrix:
    """gates.hpp:12-27: a 2x2 complex matrix with an optional unitary tag."""
    m00: complex = 1
    m01: complex = 0
    m10: complex = 0
    m11: complex = 1
    unitary: bool = False

    @staticmethod
    def from_m8(m8, unitary=False) -> "GateMatrix":
        return GateMatrix(complex(m8[0], m8[1]), complex(m8[2], m8[3]), complex(m8[4], m8[5]),
                          complex(m8[6], m8[7]), unitary)

    @staticmethod
    def unitary_checked(a, b, c, d, tol=1e-12) -> "GateMatrix":
        g = GateMatrix(complex(a), complex(b), complex(c), complex(d))
        if not is_unitary(g, tol):
            raise DomainError("matrix is not unitary within tolerance")
        g.unitary = True
        return g

    def m8(self) -> list[float]:
        return [self.m00.real, self.m00.imag, self.m01.real, self.m01.imag,
                self.m10.real, self.m10.imag, self.m11.real, self.m11.imag]

    def dagger(self) -> "GateMatrix":
        c = complex.conjugate
        return GateMatrix(c(self.m00), c(self.m10), c(self.m01), c(self.m11), self.unitary)

    def conjugate(self) -> "GateMatrix":
        c = complex.conjugate
        return GateMatrix(c(self.m00), c(self.m01), c(self.m10), c(self.m11), self.unitary)

    def __mul__(self, r: "GateMatrix") -> "GateMatrix":
        return GateMatrix(self.m00 * r.m00 + self.m01 * r.m10, self.m00 * r.m01 + self.m01 * r.m11,
                          self.m10 * r.m00 + self.m11 * r.m10, self.m10 * r.m01 + self.m11 * r.m11)


def is_unitary(g: GateMatrix, tol: float = 1e-12) -> bool:
    """gates.cpp:16-24."""
    c = complex.conjugate
    e00 = c(g.m00) * g.m00 + c(g.m10) * g.m10
    e01 = c(g.m00) * g.m01 + c(g.m10) * g.m11
    e10 = c(g.m01) * g.m00 + c(g.m11) * g.m10
    e11 = c(g.m01) * g.m01 + c(g.m11) * g.m11
    mx = lambda z: max(abs(z.real), abs(z.imag))  # noqa: E731
    return mx(e00 - 1) <= tol and mx(e01) <= tol and mx(e10) <= tol and mx(e11 - 1) <= tol


@dataclass
class NamedGate:
    """gates.hpp:31-40 (names: H T CZ SX SY RX RY RZ X Y Z)."""
    gate: str = "H"
    angle: float = 0.0


def gate_matrix(g: NamedGate) -> GateMatrix:
    """gates.cpp:51-83."""
    return GateMatrix.from_m8(C.gate_matrix(g.gate, g.angle), unitary=True)


def rotation_matrix(axis, angle: float) -> GateMatrix:
    """gates.cpp:85-98 (throws unless |axis| = 1 within 1e-12)."""
    if abs(sum(float(a) ** 2 for a in axis) - 1.0) > 1e-12:
        raise DomainError("rotation axis must be a unit vector")
    return GateMatrix.from_m8(C.rotation_matrix(axis, angle), unitary=True)


# ------------------------------------------------------------- registers

def memory_bytes(num_qubits: int, kind: str = STATE_VECTOR, precision: str = "double") -> int:
    """register.cpp:140-151 (pure arithmetic)."""
    if num_qubits < 1:
        raise DomainError(f"register needs at least 1 qubit, got {num_qubits}")
    shift = (2 * num_qubits if kind == DENSITY_MATRIX else num_qubits) + (3 if precision == "single" else 4)
    if shift >= 64:
        raise DomainError(f"memory byte count overflows 64 bits for {num_qubits} qubits")
    return 1 << shift


class Register:
    """register.hpp:51-86 on HBM: N-qubit state vector (2^N amplitudes) or
    density matrix (2^(2N), rho_jk at j + 2^N k)."""

    def __init__(self, num_qubits: int, kind: str = STATE_VECTOR, precision: str = "double",
                 env: quest.Env | None = None):
        if precision not in ("single", "double"):
            raise DomainError(f"unknown precision {precision!r}")
        if kind not in (STATE_VECTOR, DENSITY_MATRIX):
            raise DomainError(f"unknown register kind {kind!r}")
        self.env = env or default_env()
        self._q = quest.QuregHandle(self.env, num_qubits, kind == DENSITY_MATRIX, precision=precision)
        self._kind = kind
        self._precision = precision

    # register.hpp accessors
    def num_qubits(self) -> int:
        return self._q.num_qubits

    def kind(self) -> str:
        return self._kind

    def precision(self) -> str:
        return self._precision

    def flat_qubits(self) -> int:
        return self._q.flat_qubits

    def size(self) -> int:
        return 1 << self.flat_qubits()

    def init_zero_state(self):
        self._q.initZeroState()

    def get_amplitude(self, index: int) -> complex:
        if not 0 <= index < self.size():
            raise DomainError(f"amplitude index {index} out of range [0, {self.size()})")
        return complex(self._q.state(index, 1)[0])

    def set_amplitude(self, index: int, value: complex):
        if not 0 <= index < self.size():
            raise DomainError(f"amplitude index {index} out of range [0, {self.size()})")
        self._q.set_state(np.array([value], dtype=np.complex128), index)

    def norm_squared(self) -> float:
        return quest.call("qgpuNormSquared", self._q.h)

    def amps(self) -> np.ndarray:
        """Host copy of the whole flat vector (for tests and result export):
        complex128, or complex64 for a single-precision register (the
        reference's data32(), register.hpp:30)."""
        a = self._q.state()
        return a.astype(np.complex64) if self._precision == "single" else a

    def set_amps(self, amps: np.ndarray):
        self._q.set_state(amps)

    @property
    def handle(self) -> quest.QuregHandle:
        return self._q

    def destroy(self):
        self._q.destroy()

    def __del__(self):
        try:
            self._q.destroy()
        except Exception:
            pass


def _mask(controls) -> int:
    m = 0
    for c in controls:
        if not 0 <= c < 64:
            raise DomainError(f"invalid control qubit {c}")
        if m >> c & 1:
            raise DomainError(f"duplicate control qubit {c}")
        m |= 1 << c
    return m


def _as_matrix(g) -> GateMatrix:
    return g if isinstance(g, GateMatrix) else GateMatrix.from_m8(g)


# --------------------------------------------------------------- kernels

def enumerate_pairs(num_qubits: int, target: int) -> list[tuple[int, int]]:
    """kernels.cpp:68-82 (host-side index arithmetic, Eq. (1))."""
    if num_qubits < 1:
        raise DomainError("need at least 1 qubit")
    if not 0 <= target < num_qubits:
        raise DomainError(f"invalid target qubit {target} for {num_qubits} qubits")
    i = np.arange(1 << (num_qubits - 1), dtype=np.uint64)
    low = np.uint64((1 << target) - 1)
    base = ((i & ~low) << np.uint64(1)) | (i & low)
    return list(zip(base.tolist(), (base + np.uint64(1 << target)).tolist()))


def apply_single_qubit_gate(reg: Register, target: int, g):
    """kernels.cpp:100-103."""
    apply_controlled_gate(reg, [], target, g)


def apply_controlled_gate(reg: Register, controls, target: int, g):
    """kernels.cpp:105-112 (state vectors only)."""
    if reg.kind() != STATE_VECTOR:
        raise DomainError("state-vector kernel invoked on a density matrix; use the density evolution path")
    reg.handle.apply_matrix(target, _mask(controls), _as_matrix(g).m8())


def apply_named_gate(reg: Register, gate, controls, target: int):
    """kernels.cpp:114-122: density registers route to the density path."""
    g = gate_matrix(gate if isinstance(gate, NamedGate) else NamedGate(gate))
    if reg.kind() == DENSITY_MATRIX:
        apply_gate_to_density(reg, controls, target, g)
    else:
        apply_controlled_gate(reg, controls, target, g)


def apply_single_qubit_rotation(reg: Register, target: int, axis, angle: float):
    """kernels.cpp:124-132."""
    g = rotation_matrix(axis, angle)
    if reg.kind() == DENSITY_MATRIX:
        apply_gate_to_density(reg, [], target, g)
    else:
        apply_controlled_gate(reg, [], target, g)


# --------------------------------------------------------------- density

def apply_gate_to_density(reg: Register, controls, target: int, g):
    """density.cpp:85-116: G at ket qubit t, conj(G) at bra qubit t + N."""
    if reg.kind() != DENSITY_MATRIX:
        raise DomainError("gate conjugation requires a density-matrix register")
    reg.handle.apply_matrix(target, _mask(controls), _as_matrix(g).m8())


def apply_dephasing(reg: Register, target: int, prob: float):
    """density.cpp:118-130."""
    reg.handle.mixDephasing(target, prob)


def apply_depolarising(reg: Register, target: int, prob: float):
    """density.cpp:132-145."""
    reg.handle.mixDepolarising(target, prob)


def trace(reg: Register) -> complex:
    """density.cpp:147-154."""
    t = quest.call("qgpuTrace", reg.handle.h)
    return complex(t.real, t.imag)


def purity(reg: Register) -> float:
    """density.cpp:156-159."""
    return reg.handle.calcPurity()


# --------------------------------------------------------------- circuits

def generate_random_circuit(num_qubits: int, depth: int, seed: int) -> C.Circuit:
    """circuit.cpp:50-100."""
    return C.reference_random_circuit(num_qubits, depth, seed)


def run_circuit(circuit: C.Circuit, reg: Register):
    """circuit.cpp:239-247, as one C-ABI call (qgpuRunCircuit)."""
    if reg.num_qubits() != circuit.num_qubits:
        raise DomainError(f"circuit is for {circuit.num_qubits} qubits but the register has {reg.num_qubits()}")
    C.run_circuit(reg.handle, circuit)


gate_counts = C.gate_counts
serialize = C.serialize
parse = C.parse


# ------------------------------------------------------------ distributed

@dataclass
class PartitionPlan:
    """distributed.hpp:30-44."""
    num_qubits: int
    rank_count_log2: int

    def rank_count(self) -> int:
        return 1 << self.rank_count_log2

    def local_qubits(self) -> int:
        return self.num_qubits - self.rank_count_log2

    def local_len(self) -> int:
        return 1 << self.local_qubits()

    def global_lo(self, rank: int) -> int:
        return rank * self.local_len()


def partition(num_qubits: int, rank_count_log2: int) -> PartitionPlan:
    """distributed.cpp:31-42."""
    if num_qubits < 1:
        raise DomainError("partition needs at least 1 qubit")
    if rank_count_log2 < 0 or rank_count_log2 > num_qubits:
        raise DomainError(f"rank count 2^{rank_count_log2} invalid for {num_qubits} qubits (need 0 <= k <= n)")
    return PartitionPlan(num_qubits, rank_count_log2)


def needs_communication(plan: PartitionPlan, target: int) -> bool:
    """distributed.cpp:44-48."""
    if not 0 <= target < plan.num_qubits:
        raise DomainError(f"invalid target qubit {target}")
    return target >= plan.local_qubits()


def pair_rank(plan: PartitionPlan, rank: int, target: int) -> int:
    """distributed.cpp:50-57, via the library's planner."""
    if not 0 <= rank < plan.rank_count():
        raise DomainError(f"invalid rank {rank}")
    if not needs_communication(plan, target):
        raise DomainError(f"gate on qubit {target} is rank-local; no pair rank exists")
    kind, peer, _, _ = quest.plan_gate(plan.num_qubits, plan.rank_count_log2, rank, target, 0)
    return peer


# ------------------------------------------------------------ memory model

@dataclass
class MemoryModel:
    """distributed.hpp:145-150 (node budget for a strategy / precision)."""

    node_bytes: int = 0
    overhead_bytes: int = 50 << 20
    strategy: str = "full_clone"
    precision: str = "double"


def modeled_bytes_per_rank(num_qubits: int, rank_count_log2: int, strategy: str = "full_clone",
                           precision: str = "double", block_amps: int = 1) -> int:
    """distributed.cpp:436-446 over qgpuModeledBytesPerRank."""
    return quest.modeled_bytes_per_rank(num_qubits, rank_count_log2, strategy, precision == "single",
                                        block_amps)


def max_qubits(model: MemoryModel, rank_count_log2: int) -> int:
    """distributed.cpp:448-468 over qgpuMaxQubits."""
    return quest.max_qubits(model.node_bytes, rank_count_log2, model.strategy,
                            model.precision == "single", model.overhead_bytes)
