"""Times the C5 measurement tail call by call (32-qubit QFT state, the bench
circuit): calcProbOfOutcome on every qubit, 4 collapses, calcTotalProb, and
the pass / launch counts of each stage.

python tools/c5_tail.py [--qubits 32]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--qubits", type=int, default=32)
a = p.parse_args()
n = a.qubits
env = quest.Env()
q = quest.QuregHandle(env, n)
c = C.qft_circuit(n, mcpf_every=3)
for rep in range(2):
    q.initClassicalState(0x5A5A5A5A)
    C.apply_circuit(q, c)
    q.flush()
    env.sync()
    quest.jit_wait()
    stages = []

    def stage(name, fn):
        p0, l0, t0 = q.pass_count(), quest.kernel_launches(), time.perf_counter()
        fn()  # (each call returns a value: it completes its own work)
        stages.append((name, (time.perf_counter() - t0) * 1e3, q.pass_count() - p0, quest.kernel_launches() - l0))

    stage("prob q0", lambda: q.calcProbOfOutcome(0, 0))
    stage("prob q1..", lambda: [q.calcProbOfOutcome(t, 0) for t in range(1, n)])
    for t, o in [(0, 1), (9, 0), (21, 1), (n - 1, 0)]:
        stage(f"collapse {t}", lambda t=t, o=o: q.collapseToOutcome(t, o))
    stage("total", lambda: q.calcTotalProb())
    t0 = time.perf_counter()
    env.sync()  # the deferred collapses, applied
    stages.append(("sync", (time.perf_counter() - t0) * 1e3, 0, 0))
    if rep == 1:
        tot = sum(s[1] for s in stages)
        print(f"tail {tot:.2f} ms")
        for s in stages:
            print(f"  {s[0]:12s} {s[1]:8.2f} ms  passes {s[2]}  launches {s[3]}")
