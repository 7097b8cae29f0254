"""Offline SASS of the bench circuit's tile passes (no GPU needed).

python tools/jit_offline.py [--qubits 30] [--out /tmp/jit_offline] [--passes 0,1,2]
Runs the runtime's own scheduler as a host dry run (qgpuPlanPasses with
QGPU_PLAN_JIT_DUMP), writes every pass's generated JIT program, compiles the
chosen ones with nvcc for sm_100a the way the JIT does (NVRTC options:
--fmad=false, the tile geometry macros) and prints registers / spills and
the static SASS opcode mix. The runtime uses the constant-bank variant
unless it spills, then the shared-memory one.
"""
import argparse
import collections
import os
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

p = argparse.ArgumentParser()
p.add_argument("--qubits", type=int, default=30)
p.add_argument("--out", default="/tmp/jit_offline")
p.add_argument("--passes", default="")
p.add_argument("--defines", default="-DQGPU_PHASE_REG_BITS=4 -DQGPU_TILE_WARP_BITS=3 -DQGPU_TILE_GROUP_BITS=1")
a = p.parse_args()
out = Path(a.out)
out.mkdir(parents=True, exist_ok=True)
os.environ["QGPU_PLAN_JIT_DUMP"] = str(out)

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402
from tests.test_reorder_plan import flat_ops  # noqa: E402

ops = flat_ops(C.layered_random_circuit(a.qubits, 20, 12345))
_, passes, _ = quest.plan_passes(a.qubits, ops, reorder=True)
n = int(passes.max()) + 1
chosen = [int(x) for x in a.passes.split(",")] if a.passes else list(range(n))
nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
for k in chosen:
    for variant in ("", "_smem"):
        src = out / f"pass_{k}{variant}.cu"
        cub = out / f"pass_{k}{variant}.cubin"
        r = subprocess.run([nvcc, "-cubin", "-arch=sm_100a", "-std=c++17", "--fmad=false", "-Xptxas", "-v",
                            f"-I{ROOT / 'paper_1802_08032_b200' / 'csrc'}", *a.defines.split(), "-o", str(cub),
                            str(src)], capture_output=True, text=True)
        info = " ".join(re.findall(r"Used \d+ registers|\d+ bytes spill stores", r.stderr))
        if r.returncode != 0:
            print(f"pass {k}{variant}: compile failed\n{r.stderr[-2000:]}")
            continue
        sass = subprocess.run(["cuobjdump", "-sass", str(cub)], capture_output=True, text=True).stdout
        opc = collections.Counter()
        for line in sass.splitlines():
            m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\d+\s+)?([A-Z][A-Z0-9]*)", line)
            if m:
                opc[m.group(2)] += 1
        tot = sum(opc.values())
        mix = ", ".join(f"{o} {100 * c / tot:.0f}%" for o, c in opc.most_common(8))
        print(f"pass {k:2d}{variant:5s} {info:45s} {tot:6d} instrs: {mix}")
