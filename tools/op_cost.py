"""Synthetic single-pass cost probes of the tile pass (default ordering).

python tools/op_cost.py [--qubits 30]
Each probe is one pass of 63 uncontrolled rotations (kinds cycling per
qubit so that no two neighbours on a qubit merge): on register qubits only
(one phase), on 8 qubits (two phases), on lane qubits 0-2 (shuffle ops;
QGPU_LANE_CAP=0 so they stay in one pass), and a 16-op pass. Prints the
event-timed pass time, the modelled FP64 instructions per amplitude and the
pass's FP64 efficiency (the FP64 time at the pipe's peak / the pass time).
"""
import argparse
import os
import sys
from pathlib import Path

os.environ.setdefault("QGPU_LANE_CAP", "0")
os.environ.setdefault("QGPU_JIT", "sync")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--qubits", type=int, default=30)
p.add_argument("--reps", type=int, default=3)
a = p.parse_args()

KINDS = ("RX", "RY", "RZ")


def probe(targets, n_ops, kinds=KINDS):
    ops = []
    for k in range(n_ops):
        q = targets[k % len(targets)]
        kind = kinds[(k // len(targets)) % len(kinds)]
        ops.append(C.GateOp(kind, q, angle=0.3 + 0.01 * k))
    return C.Circuit(a.qubits, 0, ops)


PROBES = {
    "reg4_63": probe([5, 6, 7, 8], 63),
    "reg4_63_rxry": probe([5, 6, 7, 8], 63, ("RX", "RY")),
    "reg4_16": probe([5, 6, 7, 8], 16),
    "reg8_63": probe([5, 6, 7, 8, 9, 10, 11, 12], 63),
    "lane3_63": probe([0, 1, 2], 63, ("RX", "RY")),
    "lane3_24": probe([0, 1, 2], 24, ("RX", "RY")),
    "h_reg4_63": C.Circuit(a.qubits, 0, [C.GateOp("H", 5 + k % 4) for k in range(63)]),
}

env = quest.Env()
q = quest.QuregHandle(env, a.qubits)
peak = 148 * 64 * 1.965e9
hbm = 2 * 16 * 2.0 ** a.qubits / 6544e9 * 1e3
print(f"HBM time per pass at the copy peak: {hbm:.3f} ms")
for name, c in PROBES.items():
    for _ in range(2):
        C.apply_circuit(q, c)
        q.flush()
        env.sync()
    best = None
    for _ in range(a.reps):
        env.profile_start()
        C.apply_circuit(q, c)
        q.flush()
        env.sync()
        ms, kinds = env.profile_stop()
        info = env.last_info[kinds == 0]
        t = ms[kinds == 0]
        if best is None or t.sum() < best[0].sum():
            best = (t, info)
    t, info = best
    fp = (info >> 16) / 4.0
    fp_ms = fp * 2.0 ** a.qubits / peak * 1e3
    for ti, ii, fi, fm in zip(t, info, fp, fp_ms):
        print(f"{name:14s} ops {int(ii) & 0xFF:3d} phases {(int(ii) >> 8) & 0xFF} {ti:8.3f} ms  "
              f"fp64/amp {fi:6.1f}  fp64 time {fm:6.3f} ms  fp64 eff {fm / ti:5.2f}  hbm eff {hbm / ti:5.2f}")
q.destroy()
env.destroy()
