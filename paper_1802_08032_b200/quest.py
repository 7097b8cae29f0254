"""ctypes binding of the C-ABI (include/QuEST.h, include/qgpu.h).

This is plumbing for Python callers (tests, bench, the reference-named mirror
in ``qsim.py``); the product is ``_lib/libqgpu.so``. Loading fails loudly when
the library has not been built — there is no CPU fallback.

Every wrapper checks the library's thread-local error after the call and
raises the Python twin of the reference's exception class (types.hpp:31-55).
"""
from __future__ import annotations

import atexit
import ctypes
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("QGPU_LIB") or Path(__file__).resolve().parent / "_lib" / "libqgpu.so")


class QuESTError(RuntimeError):
    code = -1


class DomainError(QuESTError, ValueError):
    """qsim::DomainError — invalid argument; the call had no effect."""
    code = 1


class ResourceError(QuESTError, MemoryError):
    """qsim::ResourceError — allocation failure; the message names the bytes."""
    code = 2


class CommError(QuESTError):
    """qsim::CommError — transport failure; the message names the ranks."""
    code = 3


class DeviceError(QuESTError):
    code = 4


_ERRORS = {1: DomainError, 2: ResourceError, 3: CommError, 4: DeviceError}


class Complex(ctypes.Structure):
    _fields_ = [("real", ctypes.c_double), ("imag", ctypes.c_double)]


class ComplexMatrix2(ctypes.Structure):
    _fields_ = [("real", (ctypes.c_double * 2) * 2), ("imag", (ctypes.c_double * 2) * 2)]


class Vector(ctypes.Structure):
    _fields_ = [("x", ctypes.c_double), ("y", ctypes.c_double), ("z", ctypes.c_double)]


class QuESTEnv(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("numRanks", ctypes.c_int), ("impl", ctypes.c_void_p)]


class Qureg(ctypes.Structure):
    _fields_ = [
        ("isDensityMatrix", ctypes.c_int),
        ("numQubitsRepresented", ctypes.c_int),
        ("numQubitsInStateVec", ctypes.c_int),
        ("numAmpsPerChunk", ctypes.c_longlong),
        ("numAmpsTotal", ctypes.c_longlong),
        ("chunkId", ctypes.c_int),
        ("numChunks", ctypes.c_int),
        ("impl", ctypes.c_void_p),
    ]


_lib = None
_I, _D, _LL, _ULL, _VP = ctypes.c_int, ctypes.c_double, ctypes.c_longlong, ctypes.c_ulonglong, ctypes.c_void_p
_IP = ctypes.POINTER(ctypes.c_int)

# name -> (restype, argtypes)
_SIGS = {
    "createQuESTEnv": (QuESTEnv, []),
    "qgpuCreateLoopbackEnv": (QuESTEnv, [_I]),
    "qgpuCreateNcclEnv": (QuESTEnv, [_I, _I, _I, ctypes.c_char_p]),
    "qgpuGetNcclUniqueId": (_I, [ctypes.c_char_p]),
    "qgpuCreatePeerEnv": (QuESTEnv, [_I, _I, _I, ctypes.c_char_p]),
    "qgpuPeerUniqueId": (_I, [ctypes.c_char_p]),
    "qgpuPeerProbe": (_I, [ctypes.c_char_p, _I, _I, _I, _I]),
    "destroyQuESTEnv": (None, [QuESTEnv]),
    "syncQuESTEnv": (None, [QuESTEnv]),
    "reportQuESTEnv": (None, [QuESTEnv]),
    "seedQuEST": (None, [ctypes.POINTER(QuESTEnv), ctypes.POINTER(ctypes.c_ulong), _I]),
    "seedQuESTDefault": (None, [ctypes.POINTER(QuESTEnv)]),
    "createQureg": (Qureg, [_I, QuESTEnv]),
    "createDensityQureg": (Qureg, [_I, QuESTEnv]),
    "createCloneQureg": (Qureg, [Qureg, QuESTEnv]),
    "destroyQureg": (None, [Qureg, QuESTEnv]),
    "getNumQubits": (_I, [Qureg]),
    "getNumAmps": (_LL, [Qureg]),
    "initZeroState": (None, [Qureg]),
    "initPlusState": (None, [Qureg]),
    "initClassicalState": (None, [Qureg, _LL]),
    "initStateFromAmps": (None, [Qureg, _VP, _VP]),
    "setAmps": (None, [Qureg, _LL, _VP, _VP, _LL]),
    "cloneQureg": (None, [Qureg, Qureg]),
    "getAmp": (Complex, [Qureg, _LL]),
    "getRealAmp": (_D, [Qureg, _LL]),
    "getImagAmp": (_D, [Qureg, _LL]),
    "getProbAmp": (_D, [Qureg, _LL]),
    "getDensityAmp": (Complex, [Qureg, _LL, _LL]),
    "hadamard": (None, [Qureg, _I]),
    "pauliX": (None, [Qureg, _I]),
    "pauliY": (None, [Qureg, _I]),
    "pauliZ": (None, [Qureg, _I]),
    "sGate": (None, [Qureg, _I]),
    "tGate": (None, [Qureg, _I]),
    "phaseShift": (None, [Qureg, _I, _D]),
    "rotateX": (None, [Qureg, _I, _D]),
    "rotateY": (None, [Qureg, _I, _D]),
    "rotateZ": (None, [Qureg, _I, _D]),
    "rotateAroundAxis": (None, [Qureg, _I, _D, Vector]),
    "compactUnitary": (None, [Qureg, _I, Complex, Complex]),
    "unitary": (None, [Qureg, _I, ComplexMatrix2]),
    "controlledNot": (None, [Qureg, _I, _I]),
    "controlledPauliY": (None, [Qureg, _I, _I]),
    "controlledPhaseFlip": (None, [Qureg, _I, _I]),
    "controlledPhaseShift": (None, [Qureg, _I, _I, _D]),
    "multiControlledPhaseFlip": (None, [Qureg, _IP, _I]),
    "multiControlledPhaseShift": (None, [Qureg, _IP, _I, _D]),
    "controlledRotateX": (None, [Qureg, _I, _I, _D]),
    "controlledRotateY": (None, [Qureg, _I, _I, _D]),
    "controlledRotateZ": (None, [Qureg, _I, _I, _D]),
    "controlledRotateAroundAxis": (None, [Qureg, _I, _I, _D, Vector]),
    "controlledCompactUnitary": (None, [Qureg, _I, _I, Complex, Complex]),
    "controlledUnitary": (None, [Qureg, _I, _I, ComplexMatrix2]),
    "multiControlledUnitary": (None, [Qureg, _IP, _I, _I, ComplexMatrix2]),
    "calcTotalProb": (_D, [Qureg]),
    "calcProbOfOutcome": (_D, [Qureg, _I, _I]),
    "collapseToOutcome": (_D, [Qureg, _I, _I]),
    "measure": (_I, [Qureg, _I]),
    "measureWithStats": (_I, [Qureg, _I, ctypes.POINTER(ctypes.c_double)]),
    "calcPurity": (_D, [Qureg]),
    "mixDephasing": (None, [Qureg, _I, _D]),
    "mixDepolarising": (None, [Qureg, _I, _D]),
    "qgpuGetLastError": (_I, [ctypes.c_char_p, _I]),
    "qgpuClearError": (None, []),
    "qgpuVersion": (ctypes.c_char_p, []),
    "qgpuKernelLaunches": (_ULL, []),
    "qgpuTransferBytes": (None, [ctypes.POINTER(ctypes.c_ulonglong), ctypes.POINTER(ctypes.c_ulonglong)]),
    "qgpuPassCount": (_ULL, [Qureg]),
    "qgpuFlush": (None, [Qureg]),
    "qgpuSetFusion": (None, [QuESTEnv, _I, _I, _I]),
    "qgpuGetStream": (_VP, [QuESTEnv]),
    "qgpuGetDevice": (_I, [QuESTEnv]),
    "qgpuCopyStateToHost": (None, [Qureg, _LL, _LL, _VP]),
    "qgpuCopyStateFromHost": (None, [Qureg, _LL, _LL, _VP]),
    "qgpuApplyMatrix": (None, [Qureg, _I, _ULL, _VP]),
    "qgpuNormSquared": (_D, [Qureg]),
    "qgpuTrace": (Complex, [Qureg]),
    "qgpuSetExchangeChunk": (None, [QuESTEnv, _LL]),
    "qgpuSetQubitSwaps": (None, [QuESTEnv, _I]),
    "qgpuSetOrdering": (None, [QuESTEnv, _I, _I]),
    "qgpuGetOrdering": (_I, [QuESTEnv]),
    "qgpuPlanPasses": (_I, [_I, _I, _VP, _VP, _VP, _VP, _VP, _I, _I, _I, _VP, _VP, _VP]),
    "qgpuPlanSwaps": (_I, [_I, _I, _ULL, _I, _VP, _VP, _VP, _I]),
    "qgpuPlanDistributed": (_I, [_I, _I, _I, _VP, _VP, _VP, _VP, _VP, _I, _VP, _VP, _I]),
    "qgpuCommStats": (None, [Qureg, _VP, _VP]),
    "qgpuPlanGate": (_I, [_I, _I, _I, _I, _ULL, _IP, _IP, ctypes.POINTER(ctypes.c_ulonglong)]),
    "qgpuPlanChunks": (_I, [_ULL, _ULL, ctypes.POINTER(ctypes.c_ulonglong)]),
    "qgpuModeledBytesPerRank": (_I, [_I, _I, _I, _I, _ULL, ctypes.POINTER(ctypes.c_ulonglong)]),
    "qgpuMaxQubits": (_I, [_ULL, _ULL, _I, _I, _I]),
    "qgpuDeviceBytesPerRank": (_ULL, [_I, _I, _ULL, _I]),
    "qgpuDeviceMaxQubits": (_I, [_ULL, _I, _ULL, _I, _I]),
    "qgpuCreateQuregPrecision": (Qureg, [_I, QuESTEnv, _I, _I]),
    "qgpuGetPrecision": (_I, [Qureg]),
    "qgpuSetJit": (None, [_I]),
    "qgpuGetJit": (_I, []),
    "qgpuJitWait": (None, []),
    "qgpuJitShutdown": (None, []),
    "qgpuRunCircuit": (None, [Qureg, _VP, _I]),
    "qgpuJitStats": (None, [_VP, _VP, _VP]),
    "qgpuLaneExchanges": (ctypes.c_ulonglong, []),
    "qgpuJitSelfTest": (_I, [ctypes.c_char_p, _I, ctypes.POINTER(ctypes.c_double)]),
    "qgpuProfileStart": (None, [QuESTEnv]),
    "qgpuProfileStop": (_I, [QuESTEnv, _VP, _VP, _I]),
    "qgpuProfileInfo": (_I, [QuESTEnv, _VP, _I]),
}

# Every symbol include/QuEST.h and include/qgpu.h declare.
EXPORTED = sorted(set(_SIGS) | {"syncQuESTSuccess", "invalidQuESTInputError", "qgpuSetErrorHandler"})


def lib():
    """Load libqgpu.so (raises ImportError if it has not been built)."""
    global _lib
    if _lib is None:
        path = LIB_PATH
        if os.environ.get("QGPU_LIB"):  # an A/B variant build (build.py QGPU_VARIANT)
            path = Path(os.environ["QGPU_LIB"])
        if not path.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1802_08032_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
        # compiles still queued at interpreter exit are dropped and the compile
        # threads joined before any library tears down (qgpuJitShutdown)
        atexit.register(L.qgpuJitShutdown)
    return _lib


def last_error() -> tuple[int, str]:
    buf = ctypes.create_string_buffer(2048)
    code = lib().qgpuGetLastError(buf, 2048)
    return code, buf.value.decode()


def check():
    code, msg = last_error()
    if code:
        lib().qgpuClearError()
        raise _ERRORS.get(code, QuESTError)(msg)


def call(name: str, *args):
    r = getattr(lib(), name)(*args)
    check()
    return r


def cmatrix2(m8) -> ComplexMatrix2:
    u = ComplexMatrix2()
    m8 = [float(x) for x in m8]
    for k, (i, j) in enumerate([(0, 0), (0, 1), (1, 0), (1, 1)]):
        u.real[i][j] = m8[2 * k]
        u.imag[i][j] = m8[2 * k + 1]
    return u


def int_array(xs):
    arr = (ctypes.c_int * max(len(xs), 1))(*xs)
    return arr, len(xs)


# ------------------------------------------------------------- Python shells

class Env:
    """Owns a QuESTEnv. ``Env()`` = one GPU; ``Env.loopback(2**k)`` = 2^k
    virtual ranks on one GPU; ``Env.peer(rank, n, device, uid)`` = one
    process per GPU of one node over peer memory; ``Env.nccl(rank, n, device, uid)`` = one
    process per GPU."""

    def __init__(self, _handle: QuESTEnv | None = None):
        self.h = _handle if _handle is not None else call("createQuESTEnv")

    @classmethod
    def loopback(cls, num_ranks: int) -> "Env":
        return cls(call("qgpuCreateLoopbackEnv", num_ranks))

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        call("qgpuGetNcclUniqueId", buf)
        return buf.raw

    @classmethod
    def nccl(cls, rank: int, num_ranks: int, device: int, uid: bytes) -> "Env":
        return cls(call("qgpuCreateNcclEnv", rank, num_ranks, device, uid))

    @staticmethod
    def peer_unique_id() -> bytes:
        """Rank 0 only: creates the peer group's shared-memory control
        segment and returns its 128-byte id for the other ranks."""
        buf = ctypes.create_string_buffer(128)
        call("qgpuPeerUniqueId", buf)
        return buf.raw

    @classmethod
    def peer(cls, rank: int, num_ranks: int, device: int, uid: bytes) -> "Env":
        """One process per GPU of one node over peer memory (qgpu.h)."""
        return cls(call("qgpuCreatePeerEnv", rank, num_ranks, device, uid))

    @property
    def rank(self) -> int:
        return self.h.rank

    @property
    def num_ranks(self) -> int:
        return self.h.numRanks

    def sync(self):
        call("syncQuESTEnv", self.h)

    def seed(self, *seeds: int):
        arr = (ctypes.c_ulong * len(seeds))(*seeds)
        call("seedQuEST", ctypes.byref(self.h), arr, len(seeds))

    def set_fusion(self, mode: int = 0, max_ops: int = 0, reg_qubits: int = 0):
        call("qgpuSetFusion", self.h, mode, max_ops, reg_qubits)

    def set_exchange_chunk(self, amps: int):
        call("qgpuSetExchangeChunk", self.h, amps)

    def set_qubit_swaps(self, enable: bool):
        """Global<->local qubit swaps (True, default) or the reference's
        exchange per global-target gate (False)."""
        call("qgpuSetQubitSwaps", self.h, int(enable))

    def set_ordering(self, reorder: bool, window: int = 0):
        """Commutation-aware pass scheduling (True, default: within 1e-12 of
        the reference) or circuit order (False: bit-identical)."""
        call("qgpuSetOrdering", self.h, int(reorder), int(window))

    @property
    def reorder(self) -> bool:
        return bool(call("qgpuGetOrdering", self.h))

    @property
    def stream(self) -> int:
        return call("qgpuGetStream", self.h) or 0

    @property
    def device(self) -> int:
        return call("qgpuGetDevice", self.h)

    def profile_start(self):
        call("qgpuProfileStart", self.h)

    def profile_stop(self, max_records: int = 1 << 16):
        """-> (durations_ms, kinds) of every hot launch since profile_start."""
        ms = np.zeros(max_records, dtype=np.float64)
        kinds = np.zeros(max_records, dtype=np.int32)
        n = call("qgpuProfileStop", self.h, ms.ctypes.data, kinds.ctypes.data, max_records)
        n = min(n, max_records)
        info = np.zeros(max_records, dtype=np.int32)
        call("qgpuProfileInfo", self.h, info.ctypes.data, max_records)
        self.last_info = info[:n].copy()  # fused passes: ops | phases << 8 | fp64/amp x4 << 16
        return ms[:n].copy(), kinds[:n].copy()

    def destroy(self):
        if self.h is not None and self.h.impl:
            call("destroyQuESTEnv", self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.destroy()


class QuregHandle:
    """Owns a Qureg; thin methods with QuEST names and a numpy state view."""

    def __init__(self, env: Env, num_qubits: int, density: bool = False, precision: str = "double"):
        """precision "double" (createQureg / createDensityQureg) or "single"
        (Register(..., Precision::Single), register.hpp:53-54)."""
        self.env = env
        if precision == "double":
            self.h = call("createDensityQureg" if density else "createQureg", num_qubits, env.h)
        elif precision == "single":
            self.h = call("qgpuCreateQuregPrecision", num_qubits, env.h, int(density), 1)
        else:
            raise DomainError(f"precision must be 'single' or 'double', got {precision!r}")

    @property
    def precision(self) -> str:
        return "single" if call("qgpuGetPrecision", self.h) == 1 else "double"

    @property
    def num_qubits(self) -> int:
        return self.h.numQubitsRepresented

    @property
    def flat_qubits(self) -> int:
        return self.h.numQubitsInStateVec

    @property
    def is_density(self) -> bool:
        return bool(self.h.isDensityMatrix)

    def __getattr__(self, name):
        # qureg.hadamard(3) -> hadamard(qureg, 3)
        if name in _SIGS and _SIGS[name][1] and _SIGS[name][1][0] is Qureg:
            return lambda *a: call(name, self.h, *a)
        raise AttributeError(name)

    def state(self, start: int = 0, num: int | None = None) -> np.ndarray:
        total = 1 << self.flat_qubits
        num = total - start if num is None else num
        out = np.empty(num, dtype=np.complex128)
        call("qgpuCopyStateToHost", self.h, start, num, out.ctypes.data)
        return out

    def set_state(self, amps: np.ndarray, start: int = 0):
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        call("qgpuCopyStateFromHost", self.h, start, a.size, a.ctypes.data)

    def run_ops(self, ops: np.ndarray):
        """qgpuRunCircuit over a circuits.op_array() record array."""
        a = np.ascontiguousarray(ops)
        if a.dtype.itemsize != 96:
            raise DomainError("op records must be 96-byte qgpuOp")
        call("qgpuRunCircuit", self.h, a.ctypes.data, a.size)

    def apply_matrix(self, target: int, ctrl_mask: int, m8):
        m = np.ascontiguousarray(m8, dtype=np.float64)
        call("qgpuApplyMatrix", self.h, target, ctrl_mask, m.ctypes.data)

    def flush(self):
        call("qgpuFlush", self.h)

    def pass_count(self) -> int:
        return call("qgpuPassCount", self.h)

    def comm_stats(self, n: int):
        msgs = np.zeros(n, dtype=np.uint64)
        byts = np.zeros(n, dtype=np.uint64)
        call("qgpuCommStats", self.h, msgs.ctypes.data, byts.ctypes.data)
        return msgs, byts

    def destroy(self):
        if self.h is not None and self.h.impl:
            call("destroyQureg", self.h, self.env.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.destroy()


def transfer_bytes() -> tuple[int, int]:
    """(host->device, device->host) bytes the library moved since load."""
    a, b = ctypes.c_ulonglong(0), ctypes.c_ulonglong(0)
    call("qgpuTransferBytes", ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def kernel_launches() -> int:
    return call("qgpuKernelLaunches")


def plan_gate(flat: int, rank_log2: int, rank: int, target: int, ctrl_mask: int):
    """Pure host planner (qgpuPlanGate): ('local'|'skip'|'exchange', peer, own_lo, low_mask)."""
    peer, own_lo, low = ctypes.c_int(), ctypes.c_int(), ctypes.c_ulonglong()
    r = lib().qgpuPlanGate(flat, rank_log2, rank, target, ctrl_mask, ctypes.byref(peer),
                           ctypes.byref(own_lo), ctypes.byref(low))
    if r < 0:
        raise DomainError("invalid plan request")
    return ("local", "skip", "exchange")[r], peer.value, bool(own_lo.value), low.value


def plan_chunks(local_len: int, chunk: int):
    c = ctypes.c_ulonglong()
    n = lib().qgpuPlanChunks(local_len, chunk, ctypes.byref(c))
    return n, c.value


STRATEGIES = {"full_clone": 0, "half_exchange": 1, "per_amplitude": 2}


def modeled_bytes_per_rank(n: int, k: int, strategy: str = "full_clone", single: bool = False,
                           block_amps: int = 1) -> int:
    """qgpuModeledBytesPerRank (the reference's node model)."""
    out = ctypes.c_ulonglong()
    r = lib().qgpuModeledBytesPerRank(n, k, STRATEGIES[strategy], int(single), block_amps, ctypes.byref(out))
    if r < 0:
        check()
    return out.value


def max_qubits(node_bytes: int, k: int, strategy: str = "full_clone", single: bool = False,
               overhead: int = 50 << 20) -> int:
    """qgpuMaxQubits (the reference's max_qubits)."""
    r = lib().qgpuMaxQubits(node_bytes, overhead, STRATEGIES[strategy], int(single), k)
    if r < 0:
        check()
    return r


def device_bytes_per_rank(flat: int, k: int, chunk_amps: int = 1 << 24, single: bool = False) -> int:
    r = lib().qgpuDeviceBytesPerRank(flat, k, chunk_amps, int(single))
    if r == 0:
        check()
    return r


def device_max_qubits(device_bytes: int, k: int, chunk_amps: int = 1 << 24, density: bool = False,
                      single: bool = False) -> int:
    r = lib().qgpuDeviceMaxQubits(device_bytes, k, chunk_amps, int(density), int(single))
    if r < 0:
        check()
    return r


def plan_swaps(flat: int, rank_log2: int, ops, chunk_amps: int = 1 << 24):
    """qgpuPlanSwaps over [(target, is_pair), ...]: [(op index, global pos, local pos)]."""
    import numpy as np

    t = np.array([o[0] for o in ops], dtype=np.int32)
    pr = np.array([int(o[1]) for o in ops], dtype=np.int32)
    out = np.zeros(3 * max(1, len(ops)), dtype=np.int32)
    n = lib().qgpuPlanSwaps(flat, rank_log2, chunk_amps, len(ops), t.ctypes.data, pr.ctypes.data,
                            out.ctypes.data, len(ops))
    if n < 0:
        check()
    return [tuple(int(x) for x in out[3 * i:3 * i + 3]) for i in range(n)]


def plan_distributed(flat: int, rank_log2: int, ops, reorder: bool = True):
    """qgpuPlanDistributed (host only): ops as for plan_passes, on logical
    qubits of a register over 2^rank_log2 ranks. Returns (passes, [(global
    position, local position) per swap])."""
    import numpy as np

    n = len(ops)
    kinds = np.array([o[0] for o in ops], dtype=np.int32)
    q0 = np.array([o[1] for o in ops], dtype=np.int32)
    q1 = np.array([o[2] for o in ops], dtype=np.int32)
    cm = np.array([o[3] for o in ops], dtype=np.uint64)
    mats = np.zeros((max(1, n), 8), dtype=np.float64)
    for i, o in enumerate(ops):
        if o[0] == 0:
            mats[i] = o[4]
    passes = np.zeros(1, dtype=np.int32)
    cap = 4 * max(1, n)
    sw = np.zeros(2 * cap, dtype=np.int32)
    r = lib().qgpuPlanDistributed(flat, rank_log2, n, kinds.ctypes.data, q0.ctypes.data, q1.ctypes.data,
                                  cm.ctypes.data, mats.ctypes.data, int(reorder), passes.ctypes.data,
                                  sw.ctypes.data, cap)
    if r < 0:
        check()
    return int(passes[0]), [(int(sw[2 * i]), int(sw[2 * i + 1])) for i in range(min(r, cap))]


def plan_passes(flat: int, ops, reorder: bool = True, window: int = 0, max_phases: int = 3):
    """qgpuPlanPasses (host only): ops = [(kind, q0, q1, cmask, m8)], kind 0
    gate (m8: a, b, c, d as interleaved re / im), 1 dephasing, 2
    depolarising, 3 collapse. Returns (order, pass, phase) arrays over the
    executed ops: the input index, pass and phase of each, in execution
    order."""
    import numpy as np

    n = len(ops)
    kinds = np.array([o[0] for o in ops], dtype=np.int32)
    q0 = np.array([o[1] for o in ops], dtype=np.int32)
    q1 = np.array([o[2] for o in ops], dtype=np.int32)
    cm = np.array([o[3] for o in ops], dtype=np.uint64)
    mats = np.zeros((max(1, n), 8), dtype=np.float64)
    for i, o in enumerate(ops):
        if o[0] == 0:
            mats[i] = o[4]
    order = np.zeros(max(1, n), dtype=np.int32)
    pas = np.zeros(max(1, n), dtype=np.int32)
    phase = np.zeros(max(1, n), dtype=np.int32)
    r = lib().qgpuPlanPasses(flat, n, kinds.ctypes.data, q0.ctypes.data, q1.ctypes.data, cm.ctypes.data,
                             mats.ctypes.data, int(reorder), window, max_phases, order.ctypes.data,
                             pas.ctypes.data, phase.ctypes.data)
    if r < 0:
        check()
    return order[:n], pas[:n], phase[:n]


def set_jit(mode: int):
    """Per-pass JIT: 0 off, 1 background compiles (default), 2 compile before first use."""
    call("qgpuSetJit", mode)


def jit_wait():
    call("qgpuJitWait")


def lane_exchanges() -> int:
    """Lane <-> register exchange ops emitted by tile passes so far."""
    return int(lib().qgpuLaneExchanges())


def jit_stats() -> tuple[int, int, int]:
    """(compiled kernels, failed compiles, pending compiles)."""
    import numpy as np

    out = np.zeros(3, dtype=np.uint64)
    lib().qgpuJitStats(out[0:].ctypes.data, out[1:].ctypes.data, out[2:].ctypes.data)
    return int(out[0]), int(out[1]), int(out[2])


def jit_selftest() -> tuple[int, str, float]:
    """Host-only NVRTC compile of a sample pass: (cubin bytes or -1, log, seconds)."""
    buf = ctypes.create_string_buffer(1 << 16)
    sec = ctypes.c_double()
    n = lib().qgpuJitSelfTest(buf, len(buf), ctypes.byref(sec))
    return n, buf.value.decode(errors="replace"), sec.value
