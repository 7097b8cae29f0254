"""Per-op cost of the tile pass by op type: passes of N identical-kind ops
on 28 qubits; the slope of pass time vs N is the cost of one op.

python tools/op_costs.py [--qubits 28]
"""
import argparse
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--qubits", type=int, default=28)
a = p.parse_args()
n = a.qubits
env = quest.Env()
q = quest.QuregHandle(env, n)

REG = [5, 6, 7, 8]
KINDS = {
    "H on reg qubits (REAL)": lambda k: C.GateOp("H", REG[k % 4]),
    "Rx on reg qubits (RX)": lambda k: C.GateOp("RX", REG[k % 4], angle=0.1 * k),
    "U on reg qubits (GENERIC)": lambda k: C.GateOp("RY", REG[k % 4], angle=0.1 * k) if False else C.GateOp("U", REG[k % 4], matrix=tuple(C.rotation_matrix((0.6, 0.0, 0.8), 0.3 + k))),
    "X on reg qubits (SWAP)": lambda k: C.GateOp("X", REG[k % 4]),
    "CNOT reg->reg (SWAP, ctrl)": lambda k: C.GateOp("X", REG[k % 4], (REG[(k + 1) % 4],)),
    "H on lane qubits (REAL)": lambda k: C.GateOp("H", k % 5),
    "Rx on lane qubits (GENERIC)": lambda k: C.GateOp("RX", k % 5, angle=0.1 * k),
    "Rz on reg qubits (DIAG)": lambda k: C.GateOp("RZ", REG[k % 4], angle=0.1 * k),
    "CPhase reg (DIAG, a=1, ctrl)": lambda k: C.GateOp("PHASE", REG[k % 4], (REG[(k + 1) % 4],), angle=0.1 * k),
    "Rz on lane qubits (DIAG fixed)": lambda k: C.GateOp("RZ", k % 5, angle=0.1 * k),
    "Rz on outer qubits (DIAG fixed)": lambda k: C.GateOp("RZ", 20 + k % 4, angle=0.1 * k),
}
print(f"{n} qubits: pass time (ms) for N ops of one kind; slope = ms per op")
for name, mk in KINDS.items():
    times = {}
    for N in (1, 16, 40):
        c = C.Circuit(n, 0, [mk(k) for k in range(N)])
        for _ in range(2):
            C.apply_circuit(q, c)
            q.flush()
        env.profile_start()
        for _ in range(3):
            C.apply_circuit(q, c)
            q.flush()
        ms, kinds = env.profile_stop()
        passes = ms[kinds == 0]
        times[N] = float(passes.mean()) if passes.size else float("nan")
    slope = (times[40] - times[16]) / 24
    print(f"  {name:34s} N=1 {times[1]:7.3f}  N=16 {times[16]:7.3f}  N=40 {times[40]:7.3f}   {slope:.4f} ms/op")
