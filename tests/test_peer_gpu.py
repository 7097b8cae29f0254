"""Multi-process peer-memory transport on the GPU (qgpuCreatePeerEnv):
2 or 4 processes, one rank each, their partitions mapped into each other
through CUDA IPC. On this one-GPU box every rank sits on device 0 (the
mappings, interprocess events and fences are the same calls as across
NVLink/NVSwitch peers), so the cross-process protocol -- fused exchange
combines, staging-free qubit swaps, distributed depolarising, mailbox
reductions and amplitude reads, the broadcast RNG seed -- is checked bit
for bit against the oracle before it meets an 8-GPU box.

Bar: every rank's partition bit-identical to the corresponding slice of the
oracle's state; probabilities within 1e-12 of the compensated restatement;
measurement outcomes identical on every rank and equal to the restated
measure under the same seed."""
import multiprocessing as mp
import time

import numpy as np
import pytest

import oracle
from paper_1802_08032_b200 import circuits as C
from paper_1802_08032_b200 import quest
from tests import peer_worker
from tests.harness import oracle_run, random_gate_circuit, to_oracle_ops

pytestmark = pytest.mark.gpu
TOL = 1e-12


def launch(spec, nranks, limit=240.0):
    uid = quest.Env.peer_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=peer_worker.run, args=(spec, uid, r, nranks, q)) for r in range(nranks)]
    for p in procs:
        p.start()
    outs = {}
    t0 = time.time()
    try:
        while len(outs) < nranks and time.time() - t0 < limit:
            try:
                o = q.get(timeout=0.5)
                outs[o["rank"]] = o
            except Exception:
                pass
            if all(not p.is_alive() for p in procs) and q.empty():
                break
    finally:
        for p in procs:
            p.join(timeout=10)
            if p.is_alive():
                p.kill()
                p.join()
    return outs, [p.exitcode for p in procs]


def circuit_of(spec):
    if spec.get("layered"):
        return C.layered_random_circuit(spec["n"], spec["layered"], spec["seed"])
    return random_gate_circuit(spec["n"], spec["gates"], seed=spec["seed"], max_controls=2,
                               channels=spec["density"])


def check(spec, nranks):
    outs, codes = launch(spec, nranks)
    errs = {r: o for r, o in outs.items() if "error" in o}
    assert not errs, {r: o["trace"] for r, o in errs.items()}
    assert sorted(outs) == list(range(nranks)) and codes == [0] * nranks, codes
    n, density = spec["n"], spec["density"]
    c = circuit_of(spec)
    single = spec.get("precision") == "single"
    if single:
        want = oracle.orc_run_f(n, to_oracle_ops(c), density=density).astype(np.complex128)
    else:
        want = oracle_run(c, density=density)
    got = np.concatenate([np.frombuffer(outs[r]["shard"], dtype=np.complex128) for r in range(nranks)])
    if spec.get("reorder"):  # commutation-aware schedule: the north star's 1e-12, not bit for bit
        assert np.max(np.abs(got - want)) <= TOL, f"max-abs {np.max(np.abs(got - want))}"
    else:
        assert np.array_equal(got, want), f"max-abs {np.max(np.abs(got - want))}"
    wd = want.astype(np.complex128)
    norm = oracle.orc_trace(wd, n).real if density else oracle.orc_norm_kahan(wd)
    ptol = 1e-6 if single else TOL
    for o in outs.values():
        assert abs(o["total"] - norm) < ptol
        for t in range(n):
            assert abs(o["probs"][t] - oracle.orc_prob_of_outcome(wd, n, t, 1, density)) < ptol
        if o["amp"] is not None:
            i = spec.get("amp_index", 3)
            if spec.get("reorder"):
                assert abs(complex(*o["amp"]) - want[i]) <= TOL
            else:
                assert o["amp"] == (want[i].real, want[i].imag)
    if spec.get("measure"):
        seq = [o["outcomes"] for o in outs.values()]
        assert all(s == seq[0] for s in seq), seq  # the same draw on every rank
        st = oracle.orc_seed(spec["measure"])
        amps = want
        exp = []
        for t in spec["measure_qubits"]:
            o_, _, amps, st = oracle.orc_measure(amps, n, t, st, density)
            exp.append(o_)
        assert seq[0] == exp
        after = np.concatenate([np.frombuffer(outs[r]["after"], dtype=np.complex128) for r in range(nranks)])
        assert np.max(np.abs(after - amps)) < TOL
    return outs


@pytest.mark.parametrize("swaps", [False, True])
@pytest.mark.parametrize("nranks", [2, 4])
def test_peer_state_vector(nranks, swaps):
    check({"n": 12, "gates": 160, "seed": 11 + nranks, "density": False, "swaps": swaps,
           "amp_index": (1 << 12) - 5, "measure": [7, 8], "measure_qubits": [11, 0, 10]}, nranks)


@pytest.mark.parametrize("swaps", [False, True])
@pytest.mark.parametrize("nranks", [2, 4])
def test_peer_density_matrix_with_channels(nranks, swaps):
    """Depolarising on a qubit whose bra copy is a rank bit runs the peer
    corner-pair kernel (swaps off) or swaps it local (swaps on)."""
    check({"n": 5, "gates": 140, "seed": 70 + nranks, "density": True, "swaps": swaps}, nranks)


@pytest.mark.parametrize("nranks", [2, 4])
def test_peer_reordered_tile_passes(nranks):
    """The library's default schedule on a multi-process register with
    tile-sized shards (16 qubits, 14-15 local): commutation-aware passes,
    same-qubit merging and unit coefficients on every rank, qubit swaps
    moving global targets local — amplitudes, probabilities and measurement
    within 1e-12 of the oracle, the same outcomes on every rank."""
    check({"n": 16, "layered": 8, "seed": 12345, "density": False, "swaps": True, "reorder": True,
           "amp_index": (1 << 16) - 7, "measure": [3, 4], "measure_qubits": [15, 2]}, nranks)


def test_peer_layered_circuit_single_precision():
    check({"n": 14, "layered": 6, "seed": 12345, "density": False, "swaps": True, "precision": "single"}, 2)


def test_peer_exchange_traffic_and_accounting():
    """Per-gate exchanges (swaps off): one fused combine per rank per
    communicated gate, 16 B x 2^(n-k) per direction; swaps move half that,
    once per displaced qubit."""
    spec = {"n": 12, "layered": 4, "seed": 5, "density": False, "swaps": False}
    o_off = check(spec, 2)
    o_on = check(dict(spec, swaps=True), 2)
    c = circuit_of(spec)
    exch = sum(1 for op in c.ops if op.target == 11 and op.name not in ("RZ", "PHASE", "Z", "CZ", "T"))
    assert o_off[0]["msgs"][0] == exch
    assert o_off[0]["bytes"][0] == exch * 16 * (1 << 11)
    assert 0 < o_on[0]["bytes"][0] < o_off[0]["bytes"][0]


def test_peer_rank_exit_fails_partner_fast():
    """A rank that exits after joining makes its partner's next collective
    fail with a CommError naming it (no hang)."""
    t0 = time.time()
    outs, codes = launch({"n": 12, "gates": 40, "seed": 3, "density": False, "swaps": True,
                          "die_after_env": True}, 2, limit=120)
    assert codes[1] == 7
    assert "error" in outs[0] and "CommError" in outs[0]["error"] and "rank 1" in outs[0]["error"], outs.get(0)
    assert time.time() - t0 < 100
