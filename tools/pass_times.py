"""Per-pass device times of the bench circuit (A/B helper).

python tools/pass_times.py [--qubits 30] [--precision single] [--depth 20]
Prints one line per pass of the last (JIT-warm) step: index, ms, and the
pass statistics line when QGPU_PASS_STATS=1.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--qubits", type=int, default=30)
p.add_argument("--depth", type=int, default=20)
p.add_argument("--precision", default="double")
p.add_argument("--top", type=int, default=12)
a = p.parse_args()
env = quest.Env()
q = quest.QuregHandle(env, a.qubits, precision=a.precision)
c = C.layered_random_circuit(a.qubits, a.depth, 12345)
for _ in range(2):
    C.apply_circuit(q, c)
    q.flush()
    env.sync()
    quest.jit_wait()
C.apply_circuit(q, c)
q.flush()
env.sync()
env.profile_start()
C.apply_circuit(q, c)
q.flush()
env.sync()
ms, kinds = env.profile_stop()
ms = np.asarray(ms)
print(f"passes {ms.size} total {ms.sum():.2f} ms mean {ms.mean():.3f} min {ms.min():.3f} max {ms.max():.3f}")
print("per pass:", " ".join(f"{x:.2f}" for x in ms))
