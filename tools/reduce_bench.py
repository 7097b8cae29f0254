"""Time calcTotalProb / calcProbOfOutcome at 30 qubits (per-launch events)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_08032_b200 import quest  # noqa: E402

env = quest.Env()
q = quest.QuregHandle(env, 30)
q.initPlusState()
for name, fn in [("total", lambda: q.calcTotalProb()), ("prob t=3", lambda: q.calcProbOfOutcome(3, 1)),
                 ("prob t=29", lambda: q.calcProbOfOutcome(29, 0))]:
    fn()
    env.profile_start()
    vals = [fn() for _ in range(5)]
    ms, kinds = env.profile_stop()
    print(name, vals[0], "ms per call %.3f" % (ms.sum() / 5), "GB/s (bytes read) %.0f" % (
        (16 * 2**30 / (2 if name != "total" else 1)) / (ms.sum() / 5 / 1e3) / 1e9))
