"""JIT vs interpreter, bit for bit, on layered circuits of growing size."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

env = quest.Env()
for n in [int(x) for x in sys.argv[1].split(",")]:
    c = C.layered_random_circuit(n, int(sys.argv[2]) if len(sys.argv) > 2 else 3, 12345)
    out = {}
    for mode in (0, 2):
        quest.set_jit(mode)
        q = quest.QuregHandle(env, n)
        C.apply_circuit(q, c)
        out[mode] = q.state()
        q.destroy()
    d = np.abs(out[0] - out[2])
    bad = np.nonzero(d > 0)[0]
    print(n, "max diff", d.max(), "n bad", bad.size, "first bad", bad[:8], flush=True)
