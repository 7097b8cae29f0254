"""Launch kinds and device time of config C4 (14-qubit noisy density matrix)
in both precisions (env.profile kinds: 0 tile pass, 3 standalone
depolarise, ...). python tools/c4_kinds.py"""
import sys, collections
sys.path.insert(0, ".")
import numpy as np
from paper_1802_08032_b200 import circuits as C, quest
env = quest.Env()
for prec in ("double", "single"):
    q = quest.QuregHandle(env, 14, True, precision=prec)
    c = C.layered_random_circuit(14, 6, 99, noise_pmax=0.1)
    for _ in range(3):
        C.run_circuit(q, c); q.flush(); env.sync(); quest.jit_wait()
    env.profile_start(); C.run_circuit(q, c); q.flush(); env.sync()
    ms, kinds = env.profile_stop()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for m, k in zip(ms, kinds):
        agg[int(k)][0] += 1; agg[int(k)][1] += float(m)
    print(prec, {k: (v[0], round(v[1], 2)) for k, v in sorted(agg.items())}, "total", round(float(np.sum(ms)), 2))
    q.destroy()
env.destroy()
