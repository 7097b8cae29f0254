"""Times the C5 measurement tail call by call (32-qubit QFT state):
calcProbOfOutcome on every qubit, 4 collapses, calcTotalProb."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_08032_b200 import circuits as C
from paper_1802_08032_b200 import quest
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
env = quest.Env()
q = quest.QuregHandle(env, n)
c = C.qft_circuit(n, mcpf_every=3)
for rep in range(2):
    q.initClassicalState(0x5A5A5A5A)
    C.apply_circuit(q, c)
    q.flush()
    env.sync()
    quest.jit_wait()
    t0 = time.perf_counter()
    ts = []
    for t in range(n):
        a = time.perf_counter()
        q.calcProbOfOutcome(t, 0)
        ts.append((f"p{t}", time.perf_counter() - a))
    for t, o in [(0, 1), (9, 0), (21, 1), (n - 1, 0)]:
        a = time.perf_counter()
        q.collapseToOutcome(t, o)
        ts.append((f"c{t}", time.perf_counter() - a))
    a = time.perf_counter()
    q.calcTotalProb()
    ts.append(("total", time.perf_counter() - a))
    print(f"rep {rep}: tail {1e3 * (time.perf_counter() - t0):.2f} ms;",
          " ".join(f"{k}={1e3 * v:.2f}" for k, v in ts if v > 2e-4))
