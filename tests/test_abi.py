"""The C-ABI library loads and exports every symbol include/*.h declares; the
pure-host planner agrees with the reference's partition rules. CPU only (no
compute calls)."""
import re
from pathlib import Path

import pytest

import oracle
from paper_1802_08032_b200 import quest

ROOT = Path(__file__).resolve().parent.parent


def declared_functions():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in re.finditer(r"^([A-Za-z_][\w\s\*]*?)\b([A-Za-z_]\w*)\s*\(", text, flags=re.M):
            if m.group(1).startswith("typedef"):
                continue
            names.add(m.group(2))
    return sorted(names)


def test_headers_declare_the_north_star_calls():
    names = set(declared_functions())
    for n in ["createQureg", "destroyQureg", "createDensityQureg", "hadamard", "compactUnitary",
              "unitary", "rotateX", "rotateY", "rotateZ", "controlledNot", "controlledPhaseShift",
              "multiControlledPhaseFlip", "calcProbOfOutcome", "calcTotalProb", "collapseToOutcome",
              "mixDephasing", "mixDepolarising", "initZeroState", "getAmp", "setAmps", "measure"]:
        assert n in names, n


def test_library_exports_every_declared_symbol():
    lib = quest.lib()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(quest.EXPORTED) <= set(declared_functions())


def test_version_and_launch_counter_without_gpu():
    assert b"sm_100a" in quest.lib().qgpuVersion()
    assert quest.kernel_launches() >= 0


@pytest.mark.skipif(not oracle.ref_available(), reason="reference not built here")
@pytest.mark.parametrize("n,k", [(3, 1), (4, 2), (6, 3), (10, 3), (34, 4)])
def test_planner_matches_reference_partition(n, k):
    import ctypes

    for t in range(n):
        for rank in range(1 << k):
            kind, peer, own_lo, low = quest.plan_gate(n, k, rank, t, 0)
            nc, p = ctypes.c_int(), ctypes.c_int()
            assert oracle.ref().ref_partition_info(n, k, t, rank, ctypes.byref(nc), ctypes.byref(p)) == 0
            assert (kind == "exchange") == bool(nc.value)
            if nc.value:
                assert peer == p.value
                assert own_lo == (not ((rank >> (t - (n - k))) & 1))


def test_planner_rank_control_skip():
    # (n=4, k=2, CZ controls={3}, target=2): ranks without bit 3 skip
    for rank in range(4):
        kind, peer, own_lo, low = quest.plan_gate(4, 2, rank, 2, 1 << 3)
        if rank & 0b10:
            assert kind == "exchange" and peer == rank ^ 1
        else:
            assert kind == "skip"
    assert quest.plan_gate(4, 2, 0, 1, 0b1001)[0] == "skip"
    assert quest.plan_gate(4, 2, 2, 1, 0b1001)[0] == "local"
    assert quest.plan_gate(4, 2, 2, 1, 0b1001)[3] == 0b0001


def test_planner_rejects_bad_input():
    with pytest.raises(quest.DomainError):
        quest.plan_gate(4, 5, 0, 1, 0)
    with pytest.raises(quest.DomainError):
        quest.plan_gate(4, 2, 0, 1, 0b10)  # control == target


def test_chunk_plan():
    assert quest.plan_chunks(1 << 20, 1 << 16) == (16, 1 << 16)
    assert quest.plan_chunks(1 << 10, 1 << 16) == (1, 1 << 10)


def test_jit_compiles_sample_pass_for_sm100a():
    """The per-pass JIT's generated code (register, lane, diagonal, controlled
    and channel handlers over two phases) compiles with NVRTC for sm_100a —
    host only, no GPU."""
    n, log, sec = quest.jit_selftest()
    assert n > 0, log


def test_qgpu_op_records_match_the_checkers_layout():
    """circuits.op_array (qgpuOp, include/qgpu.h) is byte-identical to the
    oracle's 96-byte op records for gates, controls and both channels."""
    import oracle
    from paper_1802_08032_b200 import circuits as C
    from tests.harness import random_gate_circuit, to_oracle_ops

    c = random_gate_circuit(6, 80, seed=4, max_controls=3, channels=True)
    a = C.op_array(c)
    assert a.dtype.itemsize == 96 == oracle.OP_DTYPE.itemsize
    assert a.tobytes() == to_oracle_ops(c).tobytes()
