"""Per-pass anatomy of the bench circuit (30 qubits, depth 20, seed 12345).

python tools/heavy_passes.py [--qubits 30] [--steps 1] [--out FILE]
Runs the circuit with every pass shape JIT-compiled before its first launch
(QGPU_JIT=sync), so the k-th k_tile_jit launch of the process is pass k of
step 0 (each step ends its last pass). Prints / writes, for the last step,
every pass's event-timed duration, op count, phase count and handler codes
(QGPU_PASS_STATS), sorted by duration: the input for
`ncu -k regex:k_tile_jit --launch-skip K --launch-count 1`.
"""
import argparse
import json
import os
import sys
from pathlib import Path

os.environ.setdefault("QGPU_JIT", "sync")
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--qubits", type=int, default=30)
p.add_argument("--depth", type=int, default=20)
p.add_argument("--steps", type=int, default=3)
p.add_argument("--out", default="")
a = p.parse_args()

env = quest.Env()
q = quest.QuregHandle(env, a.qubits)
c = C.layered_random_circuit(a.qubits, a.depth, 12345)
bytes_per_pass = 2.0 * 16 * 2.0 ** a.qubits
for s in range(a.steps):
    last = s == a.steps - 1
    if last:
        env.profile_start()
    C.apply_circuit(q, c)
    q.flush()
    env.sync()
    if last:
        ms, kinds = env.profile_stop()
        info = env.last_info
ms, info = ms[kinds == 0], info[kinds == 0]
rows = [{"pass": i, "ms": round(float(t), 4), "ops": int(x & 0xFF), "phases": int((x >> 8) & 0xFF),
         "fp64_per_amp": (int(x) >> 16) / 4.0,
         "frac": round(bytes_per_pass / (t / 1e3) / 1e9 / 6544.3, 4)} for i, (t, x) in enumerate(zip(ms, info))]
rows.sort(key=lambda r: -r["ms"])
print(f"passes/step {ms.size}, total {ms.sum():.2f} ms, mean {ms.mean():.3f} ms")
for r in rows[:12]:
    print(r)
if a.out:
    Path(a.out).write_text(json.dumps({"passes_per_step": int(ms.size), "rows": rows}, indent=1))
q.destroy()
env.destroy()
