"""Every BASELINE / SURVEY.md §8(d) single-GPU config in one run: device ms per
gate (CUDA events on the library's stream, 3 warm-ups, median of 5 steps,
one step = the whole circuit, flushed), effective rate by the north star's
count, and the compiled reference on this host's cores for the configs whose
state fits host memory (C1, C2, C4; a bounded sample of each circuit's first
ops, allocation excluded).

  C1  20q state vector, layered circuit depth 20, seed 12345
  C2  30q state vector, same generator (the bench.py workload)
  C3a 33q state vector (128 GiB), depth 10
  C4  14q density matrix (28 flat qubits, 4 GiB), noisy layered: dephasing and
      depolarising p in [0, 0.1] on every qubit per layer, depth 6
  C5  32q QFT of a basis state with multi-controlled phase flips, then
      calcProbOfOutcome on every qubit and collapseToOutcome on four

python tools/config_table.py [--only C1,C4] [--no-cpu] [--out profiles/x.json]
"""
import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1802_08032_b200 import circuits as C  # noqa: E402
from paper_1802_08032_b200 import quest  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--only", default="C1,C2,C3a,C4,C5")
p.add_argument("--no-cpu", action="store_true")
p.add_argument("--cpu-ops", type=int, default=24)
p.add_argument("--precision", choices=["double", "single"], default="double")
p.add_argument("--out", default=None)
a = p.parse_args()

CONFIGS = {
    "C1": dict(n=20, density=False, circuit=lambda: C.layered_random_circuit(20, 20, 12345)),
    "C2": dict(n=30, density=False, circuit=lambda: C.layered_random_circuit(30, 20, 12345)),
    "C3a": dict(n=33, density=False, circuit=lambda: C.layered_random_circuit(33, 10, 12345)),
    "C4": dict(n=14, density=True, circuit=lambda: C.layered_random_circuit(14, 6, 99, noise_pmax=0.1)),
    "C5": dict(n=32, density=False, circuit=lambda: C.qft_circuit(32, mcpf_every=3)),
}


def gpu_time(cfg, c, batch=False):
    env = quest.Env()
    q = quest.QuregHandle(env, cfg["n"], cfg["density"], precision=a.precision)
    stream = torch.cuda.ExternalStream(env.stream)
    extra = None

    def step():
        if cfg is CONFIGS.get("C5"):
            q.initClassicalState(0x5A5A5A5A)
        (C.run_circuit if batch else C.apply_circuit)(q, c)
        q.flush()

    try:
        for _ in range(3):
            step()
            env.sync()
            quest.jit_wait()
        ts = []
        for _ in range(5):
            env.sync()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step()
            s1.record(stream)
            env.sync()
            torch.cuda.synchronize()
            ts.append(s0.elapsed_time(s1))
        if cfg is CONFIGS.get("C5"):
            # the measurement tail: P on every qubit, then four collapses
            env.sync()
            t0 = time.perf_counter()
            probs = [q.calcProbOfOutcome(t, 0) for t in range(cfg["n"])]
            for t, o in [(0, 1), (9, 0), (21, 1), (31, 0)]:
                q.collapseToOutcome(t, o)
            tot = q.calcTotalProb()
            extra = {"measure_tail_ms": round((time.perf_counter() - t0) * 1e3, 2),
                     "max_abs_P_minus_half": max(abs(x - 0.5) for x in probs), "norm_after_collapse": tot}
        norm = q.calcTotalProb()
        return statistics.median(ts), norm, extra
    finally:
        q.destroy()
        env.destroy()


def cpu_time(cfg, c):
    import oracle
    from tests.harness import to_oracle_ops

    if not oracle.ref_available():
        return None, None
    ops = to_oracle_ops(C.Circuit(c.num_qubits, c.depth, c.ops[: a.cpu_ops]))
    workers = os.cpu_count() or 1
    secs = oracle.ref_time_ops(cfg["n"], ops, workers, 3, density=cfg["density"], single=a.precision == "single")
    return statistics.median(secs[1:]) / len(ops) * 1e3, workers


rows = []
for name in a.only.split(","):
    cfg = CONFIGS[name]
    c = cfg["circuit"]()
    flat = 2 * cfg["n"] if cfg["density"] else cfg["n"]
    gates = sum(1 for op in c.ops if op.name not in ("DEPHASE", "DEPOL"))
    ms, norm, extra = gpu_time(cfg, c)
    B = 2.0 * (8 if a.precision == "single" else 16) * 2.0 ** flat
    row = {"config": name, "precision": a.precision, "qubits": cfg["n"], "density": cfg["density"],
           "flat_qubits": flat, "ops": len(c.ops),
           "gates": gates, "ms_per_step": round(ms, 3), "ms_per_op": round(ms / len(c.ops), 4),
           "effective_TBps": round(B * len(c.ops) / (ms / 1e3) / 1e12, 2), "norm_after": norm}
    if extra:
        row.update(extra)
    if name == "C1":  # host-bound: also through qgpuRunCircuit (one C-ABI call per step)
        msb, _, _ = gpu_time(cfg, c, batch=True)
        row.update({"ms_per_step_run_circuit": round(msb, 3), "ms_per_op_run_circuit": round(msb / len(c.ops), 4)})
    if not a.no_cpu and name in ("C1", "C2", "C4"):
        cms, workers = cpu_time(cfg, c)
        if cms is not None:
            row.update({"cpu_ref_ms_per_op": round(cms, 3), "cpu_workers": workers,
                        "cpu_sample": f"first {min(a.cpu_ops, len(c.ops))} ops",
                        "speedup_vs_cpu": round(cms / (ms / len(c.ops)), 1)})
    rows.append(row)
    print(json.dumps(row), flush=True)

print("\n| config | state | ops | ms/step | ms/op | effective | CPU ref ms/op | x |")
print("|---|---|---|---|---|---|---|---|")
for r in rows:
    amp = 8 if r["precision"] == "single" else 16
    st = f"{'DM ' if r['density'] else ''}{r['qubits']}q ({2 ** r['flat_qubits'] * amp / 2 ** 30:g} GiB)"
    print(f"| {r['config']} | {st} | {r['ops']} | {r['ms_per_step']} | {r['ms_per_op']} | {r['effective_TBps']} TB/s | "
          f"{r.get('cpu_ref_ms_per_op', '—')} | {r.get('speedup_vs_cpu', '—')} |")
if a.out:
    Path(a.out).write_text(json.dumps(rows, indent=1))
