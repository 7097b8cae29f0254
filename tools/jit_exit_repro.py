"""Repro for teardown with JIT kernels loaded: run a layered circuit with the
per-pass JIT (background compiles + wait), then exit normally."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

env = quest.Env()
q = quest.QuregHandle(env, 20)
c = C.layered_random_circuit(20, 4, 1)
C.apply_circuit(q, c)
q.flush()
quest.jit_wait()
C.apply_circuit(q, c)
print("prob", q.calcTotalProb(), quest.jit_stats(), flush=True)
if "--destroy" in sys.argv:
    q.destroy()
    env.destroy()
print("exiting", flush=True)
