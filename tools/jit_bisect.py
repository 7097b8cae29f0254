"""Smallest op prefix of a layered circuit where the JIT and the interpreter
differ (dumps that prefix's JIT programs to gpurun_out/jd_bisect)."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

n, depth = int(sys.argv[1]), int(sys.argv[2])
full = C.layered_random_circuit(n, depth, 12345)
env = quest.Env()


def differs(k):
    c = C.Circuit(n, depth, full.ops[:k])
    out = {}
    for mode in (0, 2):
        quest.set_jit(mode)
        q = quest.QuregHandle(env, n)
        C.apply_circuit(q, c)
        out[mode] = q.state()
        q.destroy()
    return not np.array_equal(out[0], out[2])


lo, hi = 0, len(full.ops)
assert differs(hi)
while hi - lo > 1:
    mid = (lo + hi) // 2
    if differs(mid):
        hi = mid
    else:
        lo = mid
print("first differing prefix", hi, "ops; op", hi - 1, full.ops[hi - 1], flush=True)
for o in full.ops[max(0, hi - 20):hi]:
    print("  ", o.name, o.target, o.controls)
