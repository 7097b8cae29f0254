"""Worker of the multi-process peer-transport tests (tests/test_peer_gpu.py):
one process per rank, spawned; every rank runs the same seeded program
(SPMD) through the C-ABI on its own partition and reports what it sees.
Test infrastructure only."""
from __future__ import annotations

import os
import traceback


def run(spec: dict, uid: bytes, rank: int, nranks: int, q) -> None:
    os.environ.setdefault("QGPU_PEER_TIMEOUT_S", "120")
    try:
        import numpy as np

        from paper_1802_08032_b200 import circuits as C
        from paper_1802_08032_b200 import quest
        from tests.harness import random_gate_circuit

        env = quest.Env.peer(rank, nranks, spec.get("device", 0), uid)
        out: dict = {"rank": rank}
        try:
            env.set_qubit_swaps(spec["swaps"])
            env.set_ordering(spec.get("reorder", False))
            if spec.get("chunk"):
                env.set_exchange_chunk(spec["chunk"])
            n, density = spec["n"], spec["density"]
            if spec.get("die_after_env") and rank == nranks - 1:
                os._exit(7)
            if spec.get("layered"):
                c = C.layered_random_circuit(n, spec["layered"], spec["seed"])
            else:
                c = random_gate_circuit(n, spec["gates"], seed=spec["seed"], max_controls=2, channels=density)
            qr = quest.QuregHandle(env, n, density, precision=spec.get("precision", "double"))
            C.apply_circuit(qr, c)
            flat = qr.flat_qubits
            local = 1 << (flat - (nranks.bit_length() - 1))
            # probabilities first (permuted layout when swaps moved qubits)
            out["total"] = qr.calcTotalProb()
            out["probs"] = [qr.calcProbOfOutcome(t, 1) for t in range(n)]
            a = qr.getAmp(spec.get("amp_index", 3)) if not density else None
            out["amp"] = None if a is None else (a.real, a.imag)
            out["shard"] = qr.state(rank * local, local).tobytes()
            if spec.get("measure"):
                env.seed(*spec["measure"])
                out["outcomes"] = [int(qr.measure(t)) for t in spec["measure_qubits"]]
                out["after"] = qr.state(rank * local, local).tobytes()
            out["msgs"], out["bytes"] = [int(x) for x in qr.comm_stats(nranks)[0]], \
                [int(x) for x in qr.comm_stats(nranks)[1]]
            out["launches"] = quest.kernel_launches()
            qr.destroy()
            env.sync()
        finally:
            env.destroy()
        q.put(out)
    except BaseException as e:  # reported to the parent, which fails the test
        q.put({"rank": rank, "error": f"{type(e).__name__}: {e}", "trace": traceback.format_exc()})
