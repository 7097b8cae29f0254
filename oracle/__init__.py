"""CPU checkers for the state-vector / density-matrix gate path.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package; the product (``paper_1802_08032_b200``) never does, and fails loudly
when its own CUDA library is missing instead of falling back here.

Two libraries, same op-record layout (``oracle_ops.h``):

* ``ref()``      -> ``oracle/_ref/libqsimref_shim.so``: the unmodified reference
  C++ library (``/root/reference/proj/src/*.cpp`` compiled in place by
  ``oracle/Makefile``) behind ``ref_shim.cpp``.
* ``restated()`` -> ``oracle/_build/libqsim_oracle.so``: the plain-C
  restatement ``qsim_oracle.c`` (each function cites the reference file:line it
  follows), pinned bit-for-bit against ``ref()`` in ``tests/test_oracle.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SO = HERE / "_ref" / "libqsimref_shim.so"
ORACLE_SO = HERE / "_build" / "libqsim_oracle.so"

OP_DTYPE = np.dtype(
    [
        ("kind", "<i4"),
        ("target", "<i4"),
        ("ctrl_mask", "<u8"),
        ("m", "<f8", (8,)),
        ("param", "<f8"),
        ("pad", "<f8"),
    ],
    align=False,
)
assert OP_DTYPE.itemsize == 96

GATE, DEPHASE, DEPOLARISE = 0, 1, 2
STRATEGIES = {"full_clone": 0, "half_exchange": 1, "per_amplitude": 2}

_u64 = ctypes.c_uint64
_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


def build(reference: bool | None = None) -> None:
    """Compile the restatement, and the reference when /root/reference exists."""
    targets = ["restated"]
    if reference is None:
        reference = Path("/root/reference/proj/src").is_dir()
    if reference:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


_ref_lib = None
_orc_lib = None


def ref_available() -> bool:
    return REF_SO.exists()


def ref():
    global _ref_lib
    if _ref_lib is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle ref` where /root/reference exists")
        _ref_lib = ctypes.CDLL(str(REF_SO))
        L = _ref_lib
        L.ref_last_error.argtypes = [ctypes.c_char_p, ctypes.c_int]
        L.ref_kernel_invocations.restype = ctypes.c_ulonglong
        L.ref_run_ops.argtypes = [ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp, ctypes.c_int, _vp]
        L.ref_run_ops_single.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, _vp]
        L.ref_count_kernel_calls.argtypes = [ctypes.c_int, ctypes.c_int, _vp, ctypes.POINTER(ctypes.c_ulonglong)]
        L.ref_set_get.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, ctypes.c_double, ctypes.c_double, _dp, _dp]
        L.ref_reductions.argtypes = [ctypes.c_int, ctypes.c_int, _vp, _dp, _dp, _dp, _dp]
        L.ref_run_distributed.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong,
            ctypes.c_int, _vp, ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.POINTER(ctypes.c_int),
        ]
        L.ref_random_circuit.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, ctypes.c_int, _vp, _vp, ctypes.POINTER(ctypes.c_int)]
        L.ref_gate_matrix.argtypes = [ctypes.c_int, ctypes.c_double, _vp]
        L.ref_rotation_matrix.argtypes = [ctypes.c_double] * 4 + [_vp]
        L.ref_is_unitary.argtypes = [_vp, ctypes.c_double, ctypes.POINTER(ctypes.c_int)]
        L.ref_memory_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong)]
        L.ref_modeled_bytes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, ctypes.POINTER(ctypes.c_ulonglong)]
        L.ref_max_qubits.argtypes = [ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.ref_partition_info.argtypes = [ctypes.c_int] * 4 + [ctypes.POINTER(ctypes.c_int)] * 2
        L.ref_enumerate_pairs.argtypes = [ctypes.c_int, ctypes.c_int, _vp]
        L.ref_time_ops.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, _dp]
        L.ref_parse_serialize.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.ref_serialize_random.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_ulonglong, ctypes.c_char_p, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_int)]
        L.ref_time_distributed.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int,
                                           ctypes.c_int, _dp, ctypes.POINTER(ctypes.c_ulonglong)]
        L.ref_time_ops_prec.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int, _dp]
    return _ref_lib


def restated():
    global _orc_lib
    if _orc_lib is None:
        if not ORACLE_SO.exists():
            build(reference=False)
        _orc_lib = ctypes.CDLL(str(ORACLE_SO))
        L = _orc_lib
        L.orc_pair_base_index.restype = _u64
        L.orc_pair_base_index.argtypes = [_u64, ctypes.c_int]
        L.orc_apply_gate.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _u64, _vp]
        L.orc_run_ops_f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp]
        L.orc_run_ops_f.restype = ctypes.c_int
        L.orc_apply_dm_gate.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _u64, _vp]
        L.orc_dephase.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_double]
        L.orc_depolarise.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_double]
        L.orc_run_ops.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp, _vp]
        L.orc_norm_naive.restype = ctypes.c_double
        L.orc_norm_naive.argtypes = [_vp, _u64]
        L.orc_norm_kahan.restype = ctypes.c_double
        L.orc_norm_kahan.argtypes = [_vp, _u64]
        L.orc_trace.argtypes = [_vp, ctypes.c_int, _dp, _dp]
        L.orc_prob_of_outcome.restype = ctypes.c_double
        L.orc_prob_of_outcome.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.orc_collapse.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double]
        L.orc_splitmix64_next.restype = _u64
        L.orc_splitmix64_next.argtypes = [ctypes.POINTER(_u64)]
        L.orc_uniform.restype = ctypes.c_double
        L.orc_uniform.argtypes = [ctypes.POINTER(_u64)]
        L.orc_seed.restype = _u64
        L.orc_seed.argtypes = [ctypes.POINTER(_u64), ctypes.c_int]
        L.orc_measure.restype = ctypes.c_int
        L.orc_measure.argtypes = [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_u64), _dp]
        L.orc_combine.argtypes = [_vp, _vp, _u64, _u64, ctypes.c_int, _vp]
    return _orc_lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _check(code: int):
    if code != 0:
        buf = ctypes.create_string_buffer(1024)
        ref().ref_last_error(buf, 1024)
        raise OracleError(code, buf.value.decode())


def as_ops(ops) -> np.ndarray:
    if isinstance(ops, np.ndarray) and ops.dtype == OP_DTYPE:
        return np.ascontiguousarray(ops)
    arr = np.zeros(len(ops), dtype=OP_DTYPE)
    for i, op in enumerate(ops):
        arr[i] = op
    return arr


def zero_state(nq: int, density: bool = False) -> np.ndarray:
    flat = 2 * nq if density else nq
    a = np.zeros(1 << flat, dtype=np.complex128)
    a[0] = 1.0
    return a


# ----------------------------------------------------------- reference (pinned)

def ref_run(nq: int, ops, density: bool = False, init: np.ndarray | None = None, workers: int = 1) -> np.ndarray:
    ops = as_ops(ops)
    flat = 2 * nq if density else nq
    out = np.empty(1 << flat, dtype=np.complex128)
    init_p = None
    if init is not None:
        init = np.ascontiguousarray(init, dtype=np.complex128)
        init_p = _ptr(init)
    _check(ref().ref_run_ops(nq, int(density), init_p, len(ops), _ptr(ops) if len(ops) else None, workers, _ptr(out)))
    return out


def ref_run_distributed(nq: int, ops, k: int, strategy: str = "full_clone", block_amps: int = 1,
                        density: bool = False, workers: int = 1):
    ops = as_ops(ops)
    flat = 2 * nq if density else nq
    out = np.empty(1 << flat, dtype=np.complex128)
    msgs = np.zeros(1 << k, dtype=np.uint64)
    byts = np.zeros(1 << k, dtype=np.uint64)
    nflat = len(ops) * (2 if density else 1)
    rounds = np.zeros(max(nflat, 1), dtype=np.uint32)
    nf = ctypes.c_int(0)
    _check(ref().ref_run_distributed(nq, int(density), k, STRATEGIES[strategy], block_amps, len(ops),
                                     _ptr(ops) if len(ops) else None, workers, _ptr(out), _ptr(msgs),
                                     _ptr(byts), _ptr(rounds), ctypes.byref(nf)))
    return out, msgs, byts, rounds[: nf.value]


def ref_random_circuit(nq: int, depth: int, seed: int):
    cap = nq * depth + nq + 16
    ops = np.zeros(cap, dtype=OP_DTYPE)
    names = np.zeros(cap, dtype=np.int32)
    n = ctypes.c_int(0)
    _check(ref().ref_random_circuit(nq, depth, seed, cap, _ptr(ops), _ptr(names), ctypes.byref(n)))
    return ops[: n.value].copy(), names[: n.value].copy()


def ref_gate_matrix(gate: int, angle: float = 0.0) -> np.ndarray:
    m = np.zeros(8)
    _check(ref().ref_gate_matrix(gate, angle, _ptr(m)))
    return m


def ref_rotation_matrix(axis, angle: float) -> np.ndarray:
    m = np.zeros(8)
    _check(ref().ref_rotation_matrix(float(axis[0]), float(axis[1]), float(axis[2]), angle, _ptr(m)))
    return m


def ref_time_distributed(nq: int, ops, k: int, workers: int, reps: int, strategy: str = "full_clone"):
    """Seconds of the reference's run_gate_ops (its own clock) per rep, and
    the bytes its ranks sent in one rep."""
    ops = as_ops(ops)
    secs = (ctypes.c_double * reps)()
    b = ctypes.c_ulonglong(0)
    _check(ref().ref_time_distributed(nq, k, STRATEGIES[strategy], len(ops), _ptr(ops), workers, reps, secs,
                                      ctypes.byref(b)))
    return list(secs), b.value


def ref_parse_serialize(text: str) -> str:
    """serialize(parse(text)) by the reference (circuit.cpp:123-237); raises
    OracleError (code 4, the reference's "line N: ..." message) on a parse error."""
    cap = 64 + 4 * len(text) + (1 << 16)
    buf = ctypes.create_string_buffer(cap)
    n = ctypes.c_int(0)
    _check(ref().ref_parse_serialize(text.encode(), buf, cap, ctypes.byref(n)))
    return buf.value.decode()


def ref_serialize_random(nq: int, depth: int, seed: int) -> str:
    cap = 64 * (nq * depth + nq + 16) + 64
    buf = ctypes.create_string_buffer(cap)
    n = ctypes.c_int(0)
    _check(ref().ref_serialize_random(nq, depth, seed, buf, cap, ctypes.byref(n)))
    return buf.value.decode()


def ref_reductions(nq: int, amps: np.ndarray, density: bool = False):
    amps = np.ascontiguousarray(amps, dtype=np.complex128)
    norm, tr, ti, pur = (ctypes.c_double() for _ in range(4))
    _check(ref().ref_reductions(nq, int(density), _ptr(amps), ctypes.byref(norm), ctypes.byref(tr),
                                ctypes.byref(ti), ctypes.byref(pur)))
    return norm.value, complex(tr.value, ti.value), pur.value


def ref_time_ops(nq: int, ops, workers: int, reps: int, density: bool = False,
                 single: bool = False) -> list[float]:
    ops = as_ops(ops)
    secs = (ctypes.c_double * reps)()
    _check(ref().ref_time_ops_prec(nq, int(density), int(single), len(ops), _ptr(ops), workers, reps, secs))
    return list(secs)


# ------------------------------------------------------------------ restated

def orc_run(nq: int, ops, density: bool = False, init: np.ndarray | None = None) -> np.ndarray:
    ops = as_ops(ops)
    amps = zero_state(nq, density) if init is None else np.array(init, dtype=np.complex128, copy=True)
    rc = restated().orc_run_ops(nq, int(density), len(ops), _ptr(ops) if len(ops) else None, _ptr(amps))
    if rc:
        raise OracleError(rc, "op invalid for register kind")
    return amps


def orc_norm_kahan(amps: np.ndarray) -> float:
    amps = np.ascontiguousarray(amps, dtype=np.complex128)
    return restated().orc_norm_kahan(_ptr(amps), amps.size)


def orc_prob_of_outcome(amps: np.ndarray, nq: int, target: int, outcome: int, density: bool = False) -> float:
    amps = np.ascontiguousarray(amps, dtype=np.complex128)
    return restated().orc_prob_of_outcome(_ptr(amps), nq, int(density), target, outcome)


def orc_trace(amps: np.ndarray, nq: int) -> complex:
    amps = np.ascontiguousarray(amps, dtype=np.complex128)
    re, im = ctypes.c_double(), ctypes.c_double()
    restated().orc_trace(_ptr(amps), nq, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


def orc_collapse(amps: np.ndarray, nq: int, target: int, outcome: int, prob: float, density: bool = False) -> np.ndarray:
    out = np.array(amps, dtype=np.complex128, copy=True)
    restated().orc_collapse(_ptr(out), nq, int(density), target, outcome, prob)
    return out


def orc_seed(seeds) -> int:
    arr = (_u64 * len(seeds))(*[int(s) for s in seeds])
    return restated().orc_seed(arr, len(seeds))


def orc_measure(amps: np.ndarray, nq: int, target: int, rng_state: int, density: bool = False):
    """Returns (outcome, prob, collapsed amps, new rng state)."""
    out = np.array(amps, dtype=np.complex128, copy=True)
    st = _u64(rng_state)
    p = ctypes.c_double()
    o = restated().orc_measure(_ptr(out), nq, int(density), target, ctypes.byref(st), ctypes.byref(p))
    return o, p.value, out, st.value


def orc_combine(mine: np.ndarray, theirs: np.ndarray, low_mask: int, own_lo: bool, m) -> np.ndarray:
    out = np.array(mine, dtype=np.complex128, copy=True)
    theirs = np.ascontiguousarray(theirs, dtype=np.complex128)
    m = np.ascontiguousarray(m, dtype=np.float64)
    restated().orc_combine(_ptr(out), _ptr(theirs), out.size, low_mask, int(own_lo), _ptr(m))
    return out


def zero_state_f(nq: int, density: bool = False) -> np.ndarray:
    """Single-precision zero state (complex64)."""
    n = 1 << (2 * nq if density else nq)
    a = np.zeros(n, dtype=np.complex64)
    a[0] = 1.0
    return a


def orc_run_f(nq: int, ops, density: bool = False) -> np.ndarray:
    """The single-precision restatement (complex64 result)."""
    ops = as_ops(ops)
    amps = zero_state_f(nq, density)
    _check(restated().orc_run_ops_f(nq, int(density), len(ops), _ptr(ops), _ptr(amps)))
    return amps


def ref_run_single(nq: int, ops, density: bool = False, workers: int = 1) -> np.ndarray:
    """The compiled reference in Precision::Single (complex64 result)."""
    ops = as_ops(ops)
    out = np.zeros(1 << (2 * nq if density else nq), dtype=np.complex64)
    _check(ref().ref_run_ops_single(nq, int(density), len(ops), _ptr(ops), workers, _ptr(out)))
    return out
