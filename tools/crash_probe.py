"""Runs a layered circuit at --qubits and compares with the oracle when small
enough (variant debugging)."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_1802_08032_b200 import circuits as C
from paper_1802_08032_b200 import quest
from tests.harness import oracle_run
p = argparse.ArgumentParser(); p.add_argument("--qubits", type=int, default=24); p.add_argument("--depth", type=int, default=3)
a = p.parse_args()
env = quest.Env()
c = C.layered_random_circuit(a.qubits, a.depth, 12345)
q = quest.QuregHandle(env, a.qubits)
C.apply_circuit(q, c)
print("norm", q.calcTotalProb(), flush=True)
if a.qubits <= 24:
    print("bit-identical", np.array_equal(q.state(), oracle_run(c)))
