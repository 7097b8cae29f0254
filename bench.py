#!/usr/bin/env python
"""Benchmark: ms/gate and effective HBM GB/s of a seeded random circuit.

Workload (BASELINE.json configs[1]): the layered random
circuit (H layer; brickwork CNOT / CPhase(theta); Rx/Ry/Rz(theta) on every
qubit; SplitMix64 seed 12345) of depth 20 on 30 qubits per GPU, complex
double, state in HBM (16 GiB per GPU, far larger than the 126 MB L2, so no L2
flush is needed between steps). One step = one application of the whole
circuit. N GPUs (torchrun) = weak scaling: 30 + log2(N) qubits, 2^30 amplitudes
per GPU, gates on the top log2(N) qubits exchange over NCCL.

  value  effective HBM GB/s = gates * 2 * 16 * 2^n / device time (the north
         star's per-gate byte count), whole job, CUDA events on the library's
         stream, max over ranks. ms_per_gate beside it.
  e2e    the same metric end to end through the C-ABI from the host: per step
         initZeroState + one QuEST call per gate + calcTotalProb (which
         synchronises and reads the result back), wall clock.
  roofline  the fused-pass kernel: algorithmic bytes per launch
         (2 * 16 * 2^(local qubits): one read + one write of the state) / its
         average launch time (CUDA event pair per launch, same stream),
         against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline  the unmodified reference (oracle/_ref, compiled from
         /root/reference) on this host's cores, on the first G gates of the
         same circuit.

  single_precision  side measurement (not the headline): the same circuit
         on a Precision::Single register (2 x 8 B per amplitude per gate),
         device-timed the same way (`--no-single` skips it; `--precision
         single` makes it the measured arm).

Each timed step is one whole circuit ending in a flush (an asynchronous
launch of its last pass), so every step runs the pass shapes the warm-up
compiled.

--impl reference: the reference's own CPU implementation on the same
config/metric, each step a bounded sample (first G gates).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "effective HBM GB/s (gates x 2x16x2^n B / time), layered random circuit, 30 qubits per GPU"
# --precision single: 8-byte amplitudes, the same
# per-gate accounting with 8 B
METRIC_SINGLE = ("effective HBM GB/s (gates x 2x8x2^n B / time), layered random circuit, "
                 "30 qubits per GPU, single precision")
UNIT = "GB/s"
AMP = 16  # bytes per amplitude (set from --precision)


def metric_name():
    return METRIC_SINGLE if AMP == 8 else METRIC


def dtype_name():
    return "c64 (f32 pairs)" if AMP == 8 else "c128 (f64 pairs)"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--local-qubits", type=int, default=30)
    p.add_argument("--depth", type=int, default=20)
    p.add_argument("--seed", type=int, default=12345)
    p.add_argument("--cpu-gates", type=int, default=12, help="gates in the CPU baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--fusion", type=int, default=0, help="0 fused, 1 pass per op, 2 simple kernels")
    p.add_argument("--reg-qubits", type=int, default=0)
    p.add_argument("--precision", choices=["double", "single"], default="double",
                   help="register precision (the headline is double)")
    p.add_argument("--no-single", action="store_true",
                   help="skip the single-precision side measurement of the double run")
    p.add_argument("--jit", type=int, default=None,
                   help="per-pass JIT: 0 off, 1 on (default; env QGPU_JIT=off|sync also applies)")
    return p.parse_args()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def circuit_for(n: int, depth: int, seed: int):
    from paper_1802_08032_b200 import circuits as C

    return C.layered_random_circuit(n, depth, seed)


def _traffic(key: str, local_qubits: int):
    """ncu DRAM bytes of one tile-pass launch (profiles/traffic.json)."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text())[key]
        return t["bytes"] if t["local_qubits"] == local_qubits else None
    except Exception:
        return None


def effective_bytes(n: int, gates: int) -> float:
    return gates * 2.0 * AMP * (2.0 ** n)


# ------------------------------------------------------------ CPU reference

def cpu_reference(n: int, circuit, gates: int, reps: int, workers: int, seed: int = 12345):
    """Times the unmodified reference (oracle/_ref) on the first `gates` gates:
    returns (GB/s per rep, kind, sample description)."""
    import oracle
    from tests.harness import to_oracle_ops  # test infrastructure, checker side

    sub = type(circuit)(circuit.num_qubits, circuit.depth, circuit.ops[:gates])
    ops = to_oracle_ops(sub)
    single = AMP == 8
    if oracle.ref_available():
        secs = oracle.ref_time_ops(n, ops, workers, reps, single=single)
        kind = "reference"
    else:  # restatement (single-threaded C)
        amps = oracle.zero_state_f(n) if single else oracle.zero_state(n)
        run = oracle.restated().orc_run_ops_f if single else oracle.restated().orc_run_ops
        secs = []
        for _ in range(reps):
            t0 = time.perf_counter()
            run(n, 0, len(ops), ops.ctypes.data, amps.ctypes.data)
            secs.append(time.perf_counter() - t0)
        kind, workers = "port", 1
    vals = [effective_bytes(n, gates) / s / 1e9 for s in secs]
    sample = (f"first {gates} gates of the {n}-qubit depth-{circuit.depth} layered circuit "
              f"(seed {seed}), qsim::Register({'Single' if single else 'Double'}) + apply_controlled_gate, "
              f"workers={workers}, allocation/init excluded")
    return vals, kind, workers, sample


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.local_qubits + int(math.log2(args.gpus))
    n = min(n, args.local_qubits)  # the CPU reference holds one host copy
    c = circuit_for(n, args.depth, args.seed)
    workers = os.cpu_count() or 1
    vals, kind, workers, sample = cpu_reference(n, c, args.cpu_gates, args.warmup + args.steps, workers)
    timed = vals[args.warmup:]
    v = statistics.median(timed)
    ms_gate = effective_bytes(n, 1) / (v * 1e9) * 1e3
    line = {
        "impl": "reference", "metric": metric_name(), "value": round(v, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_gate * args.cpu_gates, 3), "ms_per_gate": round(ms_gate, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_name(),
        "data": "synthetic seeded circuit",
        "config": {"workload": f"layered random circuit, {n} qubits, depth {args.depth}, seed {args.seed}",
                   "qubits": n, "sample_gates": args.cpu_gates, "precision": args.precision,
                   "l2": f"state {AMP << n >> 30} GiB >> L2"},
        "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": workers, "kind": kind, "sample": sample},
        "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours

def run_ours(args):
    import numpy as np
    import torch

    from paper_1802_08032_b200 import circuits as C
    from paper_1802_08032_b200 import quest

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        uid = [quest.Env.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        env = quest.Env.nccl(rank, world, local_rank, uid[0])
    else:
        env = quest.Env()
    if args.fusion or args.reg_qubits:
        env.set_fusion(args.fusion, 0, args.reg_qubits)
    if args.jit is not None:
        quest.set_jit(args.jit)
    jit_wait_s = 0.0
    k = int(math.log2(world))
    n = args.local_qubits + k
    circuit = circuit_for(n, args.depth, args.seed)
    gates = len(circuit.ops)
    q = quest.QuregHandle(env, n, precision=args.precision)
    stream = torch.cuda.ExternalStream(env.stream)

    def barrier():
        env.sync()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    # warm-up: each step queues its new pass shapes for the per-pass JIT
    # (NVRTC on background threads; the interpreter runs meanwhile) and waits
    # for those compiles; later steps load and run the compiled kernels
    for i in range(args.warmup):
        C.apply_circuit(q, circuit)
        q.flush()
        env.sync()
        t_jit = time.perf_counter()
        quest.jit_wait()  # (step junctions cut a few more shapes than step 1)
        jit_wait_s += time.perf_counter() - t_jit
    barrier()

    launches0 = quest.kernel_launches()
    passes0 = q.pass_count()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    env.profile_start()
    with ClockSampler(local_rank) as clocks:
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            C.apply_circuit(q, circuit)
            # a step ends its last pass (an async launch, no sync), so every
            # step runs the pass shapes the warm-up compiled; without it the
            # pass boundaries drift across step junctions
            q.flush()
        stop.record(stream)
        barrier()
    ms_launch, kinds = env.profile_stop()
    launches = quest.kernel_launches() - launches0
    passes = q.pass_count() - passes0
    elapsed = start.elapsed_time(stop)  # ms
    if dist:
        t = torch.tensor([elapsed], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    value = effective_bytes(n, gates * args.steps) / (elapsed / 1e3) / 1e9
    ms_gate = elapsed / (gates * args.steps)

    # roofline of the dominant kernel (the fused pass)
    pk, src = peaks()
    traffic = None
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text())[
            "k_tile_pass_single" if AMP == 8 else "k_tile_pass"]
        if t["local_qubits"] == args.local_qubits and t.get("amp_bytes", 16) == AMP:
            traffic = t["bytes"]
    except Exception:
        pass
    pass_ms = ms_launch[kinds == 0]
    exch_ms = ms_launch[kinds == 2]  # per-gate exchanges (swaps off)
    swap_ms = ms_launch[kinds == 5]  # global<->local qubit swaps
    per_launch_bytes = 2.0 * AMP * (2.0 ** args.local_qubits)
    achieved = per_launch_bytes / (float(pass_ms.mean()) / 1e3) / 1e9 if pass_ms.size else None
    share = float(pass_ms.sum()) / float(ms_launch.sum()) if ms_launch.size else None

    # sanity: the timed steps kept the state normalised
    norm_error = abs(q.calcTotalProb() - 1.0)

    # the same tile kernel run one gate per pass (fusion mode 1): the
    # streaming roofline of a single-gate pass, the north star's "gate pass"
    # (BASELINE.json), on the first 24 gates of the circuit
    single = None
    if args.fusion == 0:
        sub = C.Circuit(n, circuit.depth, circuit.ops[:24])
        env.set_fusion(1, 0, 0)
        C.apply_circuit(q, sub)
        q.flush()
        quest.jit_wait()
        C.apply_circuit(q, sub)
        q.flush()
        env.sync()
        env.profile_start()
        C.apply_circuit(q, sub)
        q.flush()
        env.sync()
        ms1, k1 = env.profile_stop()
        env.set_fusion(0, 0, 0)
        p1 = ms1[k1 == 0]
        if p1.size:
            gbs = 2.0 * AMP * (2.0 ** args.local_qubits) / (float(p1.mean()) / 1e3) / 1e9
            single = {"gates": int(p1.size), "avg_pass_ms": round(float(p1.mean()), 4),
                      "achieved_GBps": round(gbs, 1), "frac": round(gbs / peaks()[0]["hbm_gbs"], 4),
                      "what": "one gate per tile pass (fusion mode 1), same kernel, same bytes per pass"}

    # side measurement: the same circuit on a single-precision register
    # (Precision::Single, 2 x 8 B per amplitude per gate), device-timed the
    # same way; not the headline
    sp = None
    if args.precision == "double" and not args.no_single and world == 1:
        qs = quest.QuregHandle(env, n, precision="single")
        for _ in range(max(2, args.warmup)):
            C.apply_circuit(qs, circuit)
            qs.flush()
            env.sync()
            quest.jit_wait()
        barrier()
        env.profile_start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            C.apply_circuit(qs, circuit)
            qs.flush()
        e1.record(stream)
        barrier()
        ms_s, k_s = env.profile_stop()
        t_sp = e0.elapsed_time(e1)
        p_s = ms_s[k_s == 0]
        b_sp = 2.0 * 8 * 2.0 ** n
        sp = {"metric": METRIC_SINGLE, "value": round(gates * args.steps * b_sp / (t_sp / 1e3) / 1e9, 1),
              "unit": UNIT, "ms_per_gate": round(t_sp / (gates * args.steps), 4), "dtype": "c64 (f32 pairs)",
              "roofline_frac": round(b_sp / (float(p_s.mean()) / 1e3) / 1e9 / pk["hbm_gbs"], 4) if p_s.size else None,
              "avg_launch_ms": round(float(p_s.mean()), 4) if p_s.size else None,
              "traffic": _traffic("k_tile_pass_single", args.local_qubits),
              "norm_error": abs(qs.calcTotalProb() - 1.0)}
        qs.destroy()

    # e2e through the C-ABI from the host: init + gates + readback, wall clock
    e2e_vals = []
    for _ in range(max(1, min(args.steps, 3))):
        barrier()
        t0 = time.perf_counter()
        q.initZeroState()
        C.apply_circuit(q, circuit)
        q.calcTotalProb()
        t1 = time.perf_counter()
        e2e_vals.append(t1 - t0)
    e2e_t = max(e2e_vals) if not dist else e2e_vals[-1]
    if dist:
        t = torch.tensor([statistics.median(e2e_vals)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    else:
        e2e_t = statistics.median(e2e_vals)
    e2e = effective_bytes(n, gates) / e2e_t / 1e9
    # host->device bytes per step: each fused pass carries its op list as
    # kernel parameters (sizeof(PassParams) = 4528 B + the state pointer), and
    # initZeroState writes amplitude 0 (16 B, or 8 B single).
    h2d = int(passes / args.steps * 4536) + AMP
    d2h = 16 * max(1, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            vals, kind, workers, sample = cpu_reference(n, circuit, args.cpu_gates, 2, os.cpu_count() or 1)
            cpu = {"value": round(statistics.median(vals), 3), "unit": UNIT, "cores": workers,
                   "kind": kind, "sample": sample}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": metric_name(), "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(elapsed / args.steps, 3),
            "ms_per_gate": round(ms_gate, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dtype_name(), "data": "synthetic seeded circuit",
            "config": {"workload": f"layered random circuit, {n} qubits, depth {args.depth}, seed {args.seed}",
                       "qubits": n, "local_qubits": args.local_qubits, "gates": gates,
                       "parallelism": f"amplitude partition over {world} GPU(s)",
                       "precision": args.precision,
                       "l2": f"state {AMP << args.local_qubits >> 30} GiB per GPU >> 126 MB L2 (no flush needed)",
                       "passes_per_step": passes / args.steps, "fusion": args.fusion,
                       "jit": {"mode": quest.lib().qgpuGetJit(), "kernels": quest.jit_stats()[0],
                               "failed": quest.jit_stats()[1],
                               "compile_wait_s": round(jit_wait_s, 2) if args.warmup else None}},
            "gpu_launches": int(launches),
            "e2e": {"value": round(e2e, 1), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "what": "initZeroState + one C-ABI call per gate + calcTotalProb readback, wall clock"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
                         "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": round(achieved / pk["hbm_gbs"], 4) if achieved else None,
                         "traffic": traffic, "kernel": "k_tile_pass", "peak_source": src,
                         "bytes_per_launch": per_launch_bytes,
                         "avg_launch_ms": round(float(pass_ms.mean()), 4) if pass_ms.size else None,
                         "launches": int(pass_ms.size), "share_of_step": round(share, 4) if share else None},
            "clocks": clocks.summary(),
            "check": {"norm_error_after_timed_steps": norm_error},
            "single_gate_pass": single,
            "single_precision": sp,
            "cpu_baseline": cpu,
        }
        if exch_ms.size or swap_ms.size:
            # bytes each way per rank: a whole partition per exchange gate,
            # half a partition per qubit swap
            part = AMP * (2.0 ** args.local_qubits)
            moved = part * exch_ms.size + 0.5 * part * swap_ms.size
            t_s = (float(exch_ms.sum()) + float(swap_ms.sum())) / 1e3
            nv = moved / t_s / 1e9
            line["nvlink"] = {"exchange_gates": int(exch_ms.size) // args.steps,
                              "qubit_swaps": int(swap_ms.size) // args.steps,
                              "bytes_per_direction_per_step": int(moved / args.steps),
                              "avg_ms": round(t_s * 1e3 / max(1, exch_ms.size + swap_ms.size), 3),
                              "GBps_per_direction": round(nv, 1), "frac_of_900": round(nv / 900.0, 4)}
        print(json.dumps(line), flush=True)
    q.destroy()
    env.destroy()
    if dist:
        dist.destroy_process_group()


def main():
    global AMP
    args = parse_args()
    AMP = 8 if args.precision == "single" else 16
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
