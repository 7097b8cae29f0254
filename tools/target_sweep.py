"""Per-target gate sweep at 30 qubits: one gate per pass
(H, Rx, CNOT with the control above / below the target, CPhase) on every
target t = 0..n-1, device-timed per launch (CUDA events on the library's
stream, median of `--reps`). Reports ms per gate, the effective rate by the
north star's per-gate byte count (2 x 16 x 2^n), and that as a fraction of
the measured HBM peak. Controlled and diagonal gates move less than that
count when every tile they cannot change is skipped (TileParams.skip_ones),
so their effective rate can exceed the peak.

python tools/target_sweep.py [--qubits 30] [--reps 5] [--out profiles/x.json]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--qubits", type=int, default=30)
p.add_argument("--reps", type=int, default=5)
p.add_argument("--precision", default="double")
p.add_argument("--out", default=None)
a = p.parse_args()
n = a.qubits
amp = 8 if a.precision == "single" else 16
B = 2.0 * amp * 2.0 ** n
try:
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
except Exception:
    peak = 6650.0


def gate(kind, t):
    if kind == "H":
        return C.GateOp("H", t)
    if kind == "RX":
        return C.GateOp("RX", t, angle=0.3)
    if kind == "CNOT_above":
        return C.GateOp("X", t, controls=((t + 1) % n,))
    if kind == "CNOT_below":
        return C.GateOp("X", t, controls=((t - 1) % n,))
    if kind == "CPHASE":
        return C.GateOp("PHASE", t, controls=((t + n // 2) % n,), angle=0.7)
    raise ValueError(kind)


KINDS = ["H", "RX", "CNOT_above", "CNOT_below", "CPHASE"]
env = quest.Env()
q = quest.QuregHandle(env, n, precision=a.precision)
circs = {(k, t): C.Circuit(n, 1, [gate(k, t)]) for k in KINDS for t in range(n)}
for c in circs.values():  # first sight of every pass shape: queue its compile
    C.apply_circuit(q, c)
    q.flush()
env.sync()
quest.jit_wait()
rows = []
for (k, t), c in circs.items():
    C.apply_circuit(q, c)  # load the compiled kernel
    q.flush()
    env.sync()
    env.profile_start()
    for _ in range(a.reps):
        C.apply_circuit(q, c)
        q.flush()
    env.sync()
    ms, kinds = env.profile_stop()
    ms = np.asarray(ms)[np.asarray(kinds) == 0]
    med = float(statistics.median(ms)) if ms.size else float("nan")
    gbs = B / (med / 1e3) / 1e9
    rows.append({"gate": k, "target": t, "ms": round(med, 4), "effective_GBps": round(gbs, 1),
                 "frac_of_peak": round(gbs / peak, 4)})
norm = q.calcTotalProb()
q.destroy()
env.destroy()

print(f"# per-target sweep, {n} qubits ({a.precision}), one gate per pass, median of {a.reps}; "
      f"B = 2 x {amp} x 2^{n} B; peak {peak} GB/s; norm after sweep {norm:.15f}")
print("| t | " + " | ".join(KINDS) + " |")
print("|---|" + "---|" * len(KINDS))
by = {(r["gate"], r["target"]): r for r in rows}
for t in range(n):
    print(f"| {t} | " + " | ".join(f"{by[(k, t)]['ms']:.3f} ms ({by[(k, t)]['frac_of_peak']:.2f})" for k in KINDS) + " |")
for k in KINDS:
    v = [by[(k, t)]["ms"] for t in range(n)]
    print(f"{k}: mean {statistics.mean(v):.3f} ms, min {min(v):.3f}, max {max(v):.3f}")
if a.out:
    Path(a.out).write_text(json.dumps({"qubits": n, "precision": a.precision, "peak_GBps": peak,
                                       "bytes_per_gate": B, "rows": rows, "norm_after": norm}, indent=1))
