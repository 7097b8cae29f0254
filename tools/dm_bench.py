"""Noisy density-matrix circuit timing (BASELINE configs[3]: 14 qubits =
28-qubit flat vector, dephasing + depolarising on every qubit per layer)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

N, depth = 14, int(sys.argv[1]) if len(sys.argv) > 1 else 10
c = C.layered_random_circuit(N, depth, 7, noise_pmax=0.1)
env = quest.Env()
q = quest.QuregHandle(env, N, density=True)
for _ in range(2):
    C.apply_circuit(q, c)
    q.flush()
    env.sync()
    quest.jit_wait()
q.initZeroState()
env.sync()
p0 = q.pass_count()
t0 = time.perf_counter()
C.apply_circuit(q, c)
q.flush()
env.sync()
dt = time.perf_counter() - t0
chan = sum(1 for o in c.ops if o.name in ("DEPHASE", "DEPOL"))
print(f"DM{N} depth {depth}: {len(c.ops)} ops ({chan} channels), {q.pass_count() - p0} passes, "
      f"{dt * 1e3:.1f} ms, {dt * 1e3 / len(c.ops):.3f} ms/op, trace {q.calcTotalProb():.15f}, "
      f"purity {q.calcPurity():.6f}")
