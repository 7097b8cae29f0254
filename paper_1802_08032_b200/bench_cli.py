"""The reference spec's bench CLI (SPEC.md [MODULE] bench-cli, lines 492-548)
over the B200 C-ABI: BenchRecords for random circuits and rotation sweeps,
and the memory report — the benchmarking harness the reference specifies but
does not ship.

    python -m paper_1802_08032_b200.bench_cli --qubits 24 --depth 10 --reps 5
    python -m paper_1802_08032_b200.bench_cli --mode sweep --qubits 12 --ranks-log2 2
    python -m paper_1802_08032_b200.bench_cli --mode memory --node-bytes 68719476736

Timing protocol (PAPER §III.B.2): the register is allocated
once and reused; per repetition: initZeroState, barrier (syncQuESTEnv),
start a monotonic clock, run the circuit, barrier, stop. Allocation, init
and teardown are outside the clock; 3 untimed warm-ups precede the timed
repetitions (they also let the per-pass JIT compile the circuit's shapes).

Ranks (--ranks-log2 K): 2^K virtual ranks on this GPU (the loopback
transport: the reference's InProcessTransport on device), or the NCCL
transport when launched under torchrun. Strategies: full_clone /
half_exchange / per_amplitude run the reference's exchange per
global-target gate (one message per sub-chunk) and report the reference's
modeled bytes for that strategy; `swap` runs this runtime's global<->local
qubit swaps. Exit code 0 on success, 2 on an infeasible size, 1 otherwise.
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time

from . import circuits as C
from . import quest

FIELDS = ["num_qubits", "depth", "seed", "workers", "ranks_log2", "strategy", "wall_time_seconds",
          "time_per_gate_seconds", "peak_modeled_bytes", "measured_process_bytes", "comm_bytes",
          "comm_messages"]
SWEEP_FIELDS = FIELDS + ["target", "communicated"]
STRATEGIES = ["full_clone", "half_exchange", "per_amplitude", "swap"]


def _env(ranks_log2: int, strategy: str) -> quest.Env:
    env = quest.Env.loopback(1 << ranks_log2) if ranks_log2 else quest.Env()
    if ranks_log2:
        env.set_qubit_swaps(strategy == "swap")
    return env


def _modeled(flat: int, k: int, strategy: str, precision: str, chunk: int) -> int:
    if strategy == "swap":
        return quest.device_bytes_per_rank(flat, k, chunk, precision == "single")
    block = min(chunk, 1 << (flat - k)) if strategy == "per_amplitude" else 1
    return quest.modeled_bytes_per_rank(flat, k, strategy, precision == "single", block)


def _device_bytes_used():
    try:
        import torch

        free, total = torch.cuda.mem_get_info()
        return int(total - free)
    except Exception:
        return None


def _comm(q, ranks: int):
    msgs, byts = q.comm_stats(ranks)
    return int(byts.sum()), int(msgs.sum())


def _timed_run(env, q, circuit) -> float:
    q.initZeroState()
    env.sync()
    t0 = time.perf_counter()
    C.apply_circuit(q, circuit)
    q.flush()
    env.sync()
    return time.perf_counter() - t0


def bench_random_circuit(n: int, depth: int, seed: int, ranks_log2: int = 0, strategy: str = "swap",
                         reps: int = 5, warmup: int = 3, kind: str = "statevector",
                         precision: str = "double", circuit: C.Circuit | None = None) -> list[dict]:
    """one BenchRecord per timed repetition."""
    density = kind == "density"
    c = circuit if circuit is not None else C.reference_random_circuit(n, depth, seed)
    env = _env(ranks_log2, strategy)
    ranks = 1 << ranks_log2
    try:
        q = quest.QuregHandle(env, n, density, precision=precision)
        try:
            gates = max(1, len(c.ops))
            flat = 2 * n if density else n
            modeled = _modeled(flat, ranks_log2, strategy, precision, 1 << 24)
            for _ in range(warmup):
                _timed_run(env, q, c)
            quest.jit_wait()
            if warmup:
                _timed_run(env, q, c)  # loads the compiled pass kernels
            out = []
            for _ in range(reps):
                b0, m0 = _comm(q, ranks)
                t = _timed_run(env, q, c)
                b1, m1 = _comm(q, ranks)
                out.append({"num_qubits": n, "depth": c.depth, "seed": seed, "workers": 1,
                            "ranks_log2": ranks_log2, "strategy": strategy, "wall_time_seconds": t,
                            "time_per_gate_seconds": t / gates, "peak_modeled_bytes": modeled,
                            "measured_process_bytes": _device_bytes_used(), "comm_bytes": b1 - b0,
                            "comm_messages": m1 - m0})
            return out
        finally:
            q.destroy()
    finally:
        env.destroy()


def bench_rotation_sweep(n: int, ranks_log2: int = 0, axis=(1.0, 0.0, 0.0), angle: float = 0.3,
                         targets=None, strategy: str = "per_amplitude", reps: int = 5,
                         precision: str = "double") -> list[dict]:
    """one record per target (median of `reps` timings of a
    single rotation), flagged communicated when the target is a rank bit."""
    targets = list(range(n)) if targets is None else list(targets)
    env = _env(ranks_log2, strategy)
    ranks = 1 << ranks_log2
    local = n - ranks_log2
    try:
        q = quest.QuregHandle(env, n, precision=precision)
        try:
            modeled = _modeled(n, ranks_log2, strategy, precision, 1 << 24)
            out = []
            for t in targets:
                # apply_single_qubit_rotation (kernels.cpp:124-132): R_n(angle)
                op = C.Circuit(n, 1, [C.GateOp("U", t, matrix=tuple(C.rotation_matrix(axis, angle)))])
                _timed_run(env, q, op)
                b0, m0 = _comm(q, ranks)
                times = [_timed_run(env, q, op) for _ in range(reps)]
                b1, m1 = _comm(q, ranks)
                tm = statistics.median(times)
                out.append({"num_qubits": n, "depth": 1, "seed": 0, "workers": 1, "ranks_log2": ranks_log2,
                            "strategy": strategy, "wall_time_seconds": tm, "time_per_gate_seconds": tm,
                            "peak_modeled_bytes": modeled, "measured_process_bytes": _device_bytes_used(),
                            "comm_bytes": (b1 - b0) // reps, "comm_messages": (m1 - m0) // reps,
                            "target": t, "communicated": t >= local})
            return out
        finally:
            q.destroy()
    finally:
        env.destroy()


def slowdown_ratio(records: list[dict]) -> float | None:
    """mean communicated time / mean local time."""
    com = [r["wall_time_seconds"] for r in records if r["communicated"]]
    loc = [r["wall_time_seconds"] for r in records if not r["communicated"]]
    return statistics.mean(com) / statistics.mean(loc) if com and loc else None


def report_memory(n: int, kind: str = "statevector", precision: str = "double", strategy: str = "full_clone",
                  node_bytes: int = 64 << 30, overhead: int = 50 << 20) -> list[dict]:
    """state-only bytes, modeled total, ratio and max_qubits
    for k in [0, 16] under the reference's node model."""
    flat = 2 * n if kind == "density" else n
    amp = 8 if precision == "single" else 16
    state = amp << flat
    rows = []
    for k in range(0, 17):
        if k > flat:
            break
        model = quest.modeled_bytes_per_rank(flat, k, strategy, precision == "single")
        local = amp << (flat - k)
        rows.append({"num_qubits": n, "kind": kind, "precision": precision, "strategy": strategy,
                     "ranks_log2": k, "state_bytes": state, "state_bytes_per_rank": local,
                     "modeled_bytes_per_rank": model, "ratio": model / local,
                     "max_qubits": quest.max_qubits(node_bytes, k, strategy, precision == "single", overhead)})
    return rows


def emit(rows: list[dict], fields: list[str], fmt: str, out) -> None:
    """Schema-stable records: every field in fixed order, missing values as
    an explicit null / empty CSV cell."""
    if fmt == "json":
        for r in rows:
            out.write(json.dumps({f: r.get(f) for f in fields}) + "\n")
    else:
        out.write(",".join(fields) + "\n")
        for r in rows:
            out.write(",".join("" if r.get(f) is None else str(r.get(f)) for f in fields) + "\n")


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="bench_cli", description=__doc__.split("\n\n")[0])
    p.add_argument("--mode", choices=["circuit", "sweep", "memory"], default="circuit")
    p.add_argument("--qubits", type=int, default=20)
    p.add_argument("--depth", type=int, default=10)
    p.add_argument("--seed", type=int, default=12345)
    p.add_argument("--workers", type=int, default=1, help="(host threads: the GPU does the work)")
    p.add_argument("--ranks-log2", type=int, default=0)
    p.add_argument("--strategy", choices=STRATEGIES, default="swap")
    p.add_argument("--kind", choices=["statevector", "density"], default="statevector")
    p.add_argument("--precision", choices=["single", "double"], default="double")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--format", choices=["csv", "json"], default="csv")
    p.add_argument("--out", default="-")
    p.add_argument("--circuit", default=None, help="circuit text file (overrides the generator)")
    p.add_argument("--node-bytes", type=int, default=64 << 30)
    p.add_argument("--targets", default=None, help="sweep targets, comma separated")
    a = p.parse_args(argv)
    out = sys.stdout if a.out == "-" else open(a.out, "w")
    try:
        if a.mode == "memory":
            rows = report_memory(a.qubits, a.kind, a.precision,
                                 "full_clone" if a.strategy == "swap" else a.strategy, a.node_bytes)
            emit(rows, list(rows[0].keys()), a.format, out)
        elif a.mode == "sweep":
            tg = [int(x) for x in a.targets.split(",")] if a.targets else None
            strategy = "per_amplitude" if a.strategy == "swap" and a.ranks_log2 == 0 else a.strategy
            rows = bench_rotation_sweep(a.qubits, a.ranks_log2, targets=tg, strategy=strategy, reps=a.reps,
                                        precision=a.precision)
            emit(rows, SWEEP_FIELDS, a.format, out)
            r = slowdown_ratio(rows)
            if r is not None:
                sys.stderr.write(f"slowdown ratio (communicated / local): {r:.3f}\n")
        else:
            circ = None
            if a.circuit:
                with open(a.circuit) as f:
                    circ = C.parse(f.read())
                a.qubits = circ.num_qubits
            rows = bench_random_circuit(a.qubits, a.depth, a.seed, a.ranks_log2, a.strategy, a.reps,
                                        a.warmup, a.kind, a.precision, circ)
            emit(rows, FIELDS, a.format, out)
        return 0
    except quest.ResourceError as e:
        sys.stderr.write(f"infeasible size: {e}\n")
        return 2
    except Exception as e:  # noqa: BLE001 -- CLI boundary
        sys.stderr.write(f"error: {e}\n")
        return 1
    finally:
        if out is not sys.stdout:
            out.close()


if __name__ == "__main__":
    sys.exit(main())
