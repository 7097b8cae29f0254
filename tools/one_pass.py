"""One tile pass of N identical ops (for ncu source-level profiles).

python tools/one_pass.py --kind RY --targets 5,6,7 --n 32 --qubits 26 [--controls 9]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--kind", default="H")
p.add_argument("--targets", default="5,6,7,8")
p.add_argument("--controls", default="")
p.add_argument("--n", type=int, default=40)
p.add_argument("--qubits", type=int, default=26)
p.add_argument("--reps", type=int, default=2)
a = p.parse_args()
tg = [int(x) for x in a.targets.split(",")]
ct = tuple(int(x) for x in a.controls.split(",")) if a.controls else ()
env = quest.Env()
q = quest.QuregHandle(env, a.qubits)
ops = [C.GateOp(a.kind, tg[k % len(tg)], controls=ct, angle=0.1 * k) if a.kind in C.HAS_ANGLE
       else C.GateOp(a.kind, tg[k % len(tg)], controls=ct) for k in range(a.n)]
c = C.Circuit(a.qubits, 0, ops)
for _ in range(a.reps):
    C.apply_circuit(q, c)
    q.flush()
env.sync()
print("ok")
