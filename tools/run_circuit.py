"""Runs the layered random circuit through the C-ABI (for ncu / quick timing).

python tools/run_circuit.py --qubits 26 --depth 20 --reps 2 --reg-qubits 4 --fusion 0
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--qubits", type=int, default=26)
p.add_argument("--depth", type=int, default=20)
p.add_argument("--reps", type=int, default=2)
p.add_argument("--fusion", type=int, default=0)
p.add_argument("--reg-qubits", type=int, default=0)
p.add_argument("--max-ops", type=int, default=0)
a = p.parse_args()
env = quest.Env()
env.set_fusion(a.fusion, a.max_ops, a.reg_qubits)
c = C.layered_random_circuit(a.qubits, a.depth, 12345)
q = quest.QuregHandle(env, a.qubits)
for r in range(a.reps):
    env.profile_start()
    t0 = time.perf_counter()
    C.apply_circuit(q, c)
    q.flush()
    env.sync()
    t1 = time.perf_counter()
    ms, kinds = env.profile_stop()
    print(f"rep {r}: {len(c.ops)} gates, {len(ms)} launches, kernel sum {ms.sum():.2f} ms, "
          f"wall {1e3 * (t1 - t0):.2f} ms, mean launch {ms.mean():.3f} ms")
print("norm", q.calcTotalProb())
