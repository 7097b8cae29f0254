"""Run the first K ops of a layered circuit with the JIT in sync mode (set
QGPU_JIT_DUMP to keep the generated programs)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

n, depth, k = (int(x) for x in sys.argv[1:4])
c = C.Circuit(n, depth, C.layered_random_circuit(n, depth, 12345).ops[:k])
env = quest.Env()
quest.set_jit(2)
q = quest.QuregHandle(env, n)
C.apply_circuit(q, c)
print(q.calcTotalProb())
