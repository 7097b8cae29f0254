"""Pass-time sweep: one tile pass of N identical ops, per-launch CUDA events.

python tools/sweep.py --qubits 30 --kinds RY,RZ,H,X --counts 1,2,4,8,16
Prints ms per pass per (kind, count); targets cycle over --targets.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--qubits", type=int, default=30)
p.add_argument("--kinds", default="RZ,RY,RX,H,X")
p.add_argument("--counts", default="1,4,8,16,32")
p.add_argument("--targets", default="5,6,7,8,9,10,11")
p.add_argument("--controls", default="")
p.add_argument("--reps", type=int, default=3)
a = p.parse_args()
tg = [int(x) for x in a.targets.split(",")]
ct = tuple(int(x) for x in a.controls.split(",")) if a.controls else ()
env = quest.Env()
q = quest.QuregHandle(env, a.qubits)
ab = 2 * 16 * 2.0 ** a.qubits
for kind in a.kinds.split(","):
    row = []
    for n in [int(x) for x in a.counts.split(",")]:
        ops = [C.GateOp(kind, tg[k % len(tg)], controls=ct, angle=0.1 + 0.01 * k) if kind in C.HAS_ANGLE
               else C.GateOp(kind, tg[k % len(tg)], controls=ct) for k in range(n)]
        c = C.Circuit(a.qubits, 0, ops)
        C.apply_circuit(q, c)
        q.flush()
        env.sync()
        quest.jit_wait()  # per-pass JIT: compile this shape before timing
        C.apply_circuit(q, c)
        q.flush()
        env.sync()
        env.profile_start()
        for _ in range(a.reps):
            C.apply_circuit(q, c)
            q.flush()
        env.sync()
        ms, kinds = env.profile_stop()
        m = float(ms.mean())
        row.append(f"{n}:{m:.2f}ms({ab / m / 1e6:.0f}GB/s,{len(ms) // a.reps}p)")
    print(kind, " ".join(row), flush=True)
