"""Workload for compute-sanitizer (racecheck / synccheck / memcheck) on the
tile pass: small registers, every pass shape of the layered circuit and of
a random circuit with controls on outer qubits (tiles that skip phases),
three-phase passes, a noisy density matrix (fused depolarising), on the JIT
kernels (QGPU_JIT=sync) and on the interpreter (QGPU_JIT=off), checked
against the oracle so a race that corrupts data also fails here.

compute-sanitizer --tool racecheck python tools/sanitize_run.py [--qubits 16]
(at >= 21 qubits a CTA walks more tiles than its 3 stages, so the per-warp
refill of a stage after the last phase is exercised too)
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402
from tests.harness import oracle_run, random_gate_circuit  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--qubits", type=int, default=16)
p.add_argument("--depth", type=int, default=4)
p.add_argument("--ops", type=int, default=120)
p.add_argument("--reorder", action="store_true",
               help="the default ordering (tolerance handlers, unit coefficients, merging): within 1e-12")
a = p.parse_args()
n = a.qubits
env = quest.Env()
env.set_ordering(a.reorder)
bad = 0
for name, c, dens in [
    ("layered", C.layered_random_circuit(n, a.depth, 12345), False),
    ("random+outer controls", random_gate_circuit(n, a.ops, seed=7, max_controls=3), False),
    ("noisy density", C.layered_random_circuit(n // 2, 3, 5, noise_pmax=0.1), True),
]:
    q = quest.QuregHandle(env, c.num_qubits, density=dens)
    C.apply_circuit(q, c)
    got = q.state()
    want = oracle_run(c, density=dens)
    ok = float(np.max(np.abs(got - want))) <= 1e-12 if a.reorder else np.array_equal(got, want)
    bad += not ok
    print(f"{name}: {('within 1e-12' if a.reorder else 'bit-identical') if ok else 'MISMATCH'}", flush=True)
    q.destroy()
env.destroy()
print("launches", quest.kernel_launches())
sys.exit(1 if bad else 0)
