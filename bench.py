#!/usr/bin/env python
"""Benchmark: ms/gate and effective HBM GB/s of a seeded random circuit.

Workload (BASELINE.json configs[1] at N = 1, configs[2] at N > 1; SURVEY.md
§8(d)): the layered random circuit (H layer; brickwork CNOT / CPhase(theta);
Rx/Ry/Rz(theta) on every qubit; SplitMix64 seed 12345), depth 20, complex
double, state in HBM (far larger than the 126 MB L2, so no flush is needed
between steps). One step = one application of the whole circuit.

  N = 1   30 qubits (16 GiB), C2.
  N > 1   one process per GPU (self-launched with torch.distributed.run when
          WORLD_SIZE is unset), 33 local qubits per GPU = 34 / 35 / 36 qubits
          at 2 / 4 / 8 GPUs (C3b: 36 qubits over 8 B200s), weak scaling; the
          peer-memory transport (qgpuCreatePeerEnv: partitions mapped over
          NVLink, exchanges and qubit swaps as one kernel per rank) or NCCL
          (--transport nccl). --local-qubits overrides.

  value  effective HBM GB/s = gates * 2 * 16 * 2^n / device time (the north
         star's per-gate byte count), whole job, CUDA events on the library's
         stream, max over ranks. ms_per_gate beside it.
  e2e    the same metric end to end through the C-ABI from the host: per step
         initZeroState + one QuEST call per gate + calcTotalProb (which
         synchronises and reads the result back), wall clock; h2d/d2h bytes
         are the library's own transfer counters over those steps (op tables
         riding in the pass launches + explicit copies). `e2e_cold` is the
         first circuit of the process (JIT compiling in the background, the
         interpreter running meanwhile).
  roofline  the fused-pass kernel: algorithmic bytes per launch
         (2 * 16 * 2^(local qubits): one read + one write of the state) / its
         average launch time (CUDA event pair per launch, same stream),
         against MEASURED_PEAKS.json hbm_gbs; `passes` splits the launches
         by op count with each class's own achieved bandwidth.
  nvlink (N > 1)  exchange gates / qubit swaps per step, bytes per direction
         and GB/s against 900 GB/s, from the event pairs around them.
  c5     side measurement (C5, BASELINE.json configs[4]): QFT with
         multi-controlled phase flips on 32 qubits at every N, then
         calcProbOfOutcome on every qubit and collapseToOutcome on 4 (ms per
         gate, the measurement tail's wall time).
  cpu_baseline  the unmodified reference (oracle/_ref, compiled from
         /root/reference) on this host's cores, on a systematic sample of the
         same circuit (every k-th gate: all gate kinds and targets).

--impl reference: the reference's own CPU implementation on the same
config/metric: N = 1 qsim::Register + apply_controlled_gate on all host
cores; N > 1 its run_gate_ops over InProcessTransport with 2^k rank threads
(the distributed CPU path, capped at 30 qubits by host RAM). Each step is
the bounded systematic sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "effective HBM GB/s (gates x 2x16x2^n B / time), layered random circuit"
# --precision single: 8-byte amplitudes, the same
# per-gate accounting with 8 B
METRIC_SINGLE = "effective HBM GB/s (gates x 2x8x2^n B / time), layered random circuit, single precision"
UNIT = "GB/s"
AMP = 16  # bytes per amplitude (set from --precision)
NVLINK_GBS = 900.0


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
    p.add_argument("--local-qubits", type=int, default=None,
                   help="qubits per GPU (default 30 at N = 1, 33 at N > 1)")
    p.add_argument("--depth", type=int, default=20)
    p.add_argument("--seed", type=int, default=12345)
    p.add_argument("--cpu-gates", type=int, default=30, help="gates in the CPU sample (systematic)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--fusion", type=int, default=0, help="0 fused, 1 pass per op, 2 simple kernels")
    p.add_argument("--reg-qubits", type=int, default=0)
    p.add_argument("--precision", choices=["double", "single"], default="double",
                   help="register precision (the headline is double)")
    p.add_argument("--no-single", action="store_true",
                   help="skip the single-precision side measurement of the double run")
    p.add_argument("--no-c5", action="store_true", help="skip the C5 QFT + measurement side measurement")
    p.add_argument("--jit", type=int, default=None,
                   help="per-pass JIT: 0 off, 1 on (default; env QGPU_JIT=off|sync also applies)")
    p.add_argument("--order", choices=["reorder", "exact"], default="reorder",
                   help="op order in the passes: reorder (library default: commuting ops scheduled into fewer "
                        "passes, within 1e-12 of the reference) or exact (circuit order, bit-identical)")
    p.add_argument("--no-exact-side", action="store_true",
                   help="skip the circuit-order side measurement of a reorder run")
    p.add_argument("--transport", choices=["peer", "nccl"], default="peer", help="N > 1 data plane")
    p.add_argument("--swaps", type=int, default=1, help="N > 1: global<->local qubit swaps (0: exchange per gate)")
    a = p.parse_args()
    if a.local_qubits is None:
        a.local_qubits = 30 if a.gpus == 1 else 33
    return a


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
        self.lines = []

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


def workload_name(n: int, depth: int, seed: int) -> str:
    return f"layered random circuit, {n} qubits, depth {depth}, seed {seed}"


def _traffic(key: str, local_qubits: int):
    """ncu DRAM bytes of one tile-pass launch (profiles/traffic.json, from a
    committed `ncu --set full` capture)."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text())[key]
        if t["local_qubits"] == local_qubits and t.get("amp_bytes", 16) == AMP:
            return t["bytes"]
    except Exception:
        pass
    return None


def effective_bytes(n: int, gates: int) -> float:
    return gates * 2.0 * AMP * (2.0 ** n)


def systematic_sample(circuit, g: int):
    """Every k-th gate of the circuit (k = len / g): the circuit's own mix of
    gate kinds, targets and controls, in circuit order."""
    ops = circuit.ops
    g = max(1, min(g, len(ops)))
    idx = [int(i * len(ops) / g) for i in range(g)]
    return type(circuit)(circuit.num_qubits, circuit.depth, [ops[i] for i in idx])


def sample_desc(n, circuit, g, extra=""):
    return (f"systematic sample: every {len(circuit.ops) / g:.1f}th gate of the {n}-qubit depth-{circuit.depth} "
            f"layered circuit ({g} of {len(circuit.ops)} gates: H/Rx/Ry/Rz/CNOT/CPhase on targets across "
            f"0..{n - 1}){extra}, allocation/init excluded")


# ------------------------------------------------------------ CPU reference

def cpu_reference(n: int, circuit, gates: int, reps: int, workers: int, k: int = 0):
    """Times the unmodified reference (oracle/_ref) on the systematic sample:
    returns (GB/s per rep, kind, workers, sample description)."""
    import oracle
    from tests.harness import to_oracle_ops  # test infrastructure, checker side

    sub = systematic_sample(circuit, gates)
    ops = to_oracle_ops(sub)
    single = AMP == 8
    if oracle.ref_available() and k > 0:
        secs, _ = oracle.ref_time_distributed(n, ops, k, workers, reps)
        kind = "reference"
        extra = f", qsim::run_gate_ops over InProcessTransport, 2^{k} ranks (FullClone), {workers} worker threads"
    elif oracle.ref_available():
        secs = oracle.ref_time_ops(n, ops, workers, reps, single=single)
        kind = "reference"
        extra = (f", qsim::Register({'Single' if single else 'Double'}) + apply_controlled_gate, "
                 f"workers={workers}")
    else:  # restatement (single-threaded C)
        amps = oracle.zero_state_f(n) if single else oracle.zero_state(n)
        run = oracle.restated().orc_run_ops_f if single else oracle.restated().orc_run_ops
        secs = []
        for _ in range(reps):
            t0 = time.perf_counter()
            run(n, 0, len(ops), ops.ctypes.data, amps.ctypes.data)
            secs.append(time.perf_counter() - t0)
        kind, workers, extra = "port", 1, ", oracle restatement (1 thread)"
    g = len(sub.ops)
    vals = [effective_bytes(n, g) / s / 1e9 for s in secs]
    return vals, kind, workers, sample_desc(n, circuit, g, extra), g


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    k = int(math.log2(args.gpus))
    n_ours = args.local_qubits + k
    # the CPU reference holds the state in host RAM (196 GB on the GPU box):
    # at N > 1 its distributed path runs FullClone (2x) up to 30 qubits
    n = min(n_ours, 30)
    c = circuit_for(n, args.depth, args.seed)
    workers = os.cpu_count() or 1
    vals, kind, workers, sample, g = cpu_reference(n, c, args.cpu_gates, args.warmup + args.steps, workers, k)
    timed = vals[args.warmup:]
    v = statistics.median(timed)
    ms_gate = effective_bytes(n, 1) / (v * 1e9) * 1e3
    line = {
        "impl": "reference", "metric": metric_name(), "value": round(v, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_gate * g, 3), "ms_per_gate": round(ms_gate, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dtype_name(),
        "data": "synthetic seeded circuit",
        "config": {"workload": workload_name(n, args.depth, args.seed), "qubits": n,
                   "ranks": 1 << k, "sample_gates": g, "precision": args.precision,
                   "l2": f"state {AMP << n >> 30} GiB >> L2",
                   **({"note": f"ours runs {n_ours} qubits at N={args.gpus}; the reference's distributed CPU path "
                               f"is capped at 30 qubits by host RAM (the metric is per byte moved)"}
                      if n != n_ours else {})},
        "cpu_baseline": {"value": round(v, 3), "unit": UNIT, "cores": workers, "kind": kind, "sample": sample},
        "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ ours

def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int:
    """`python bench.py --gpus N` without torchrun: launch N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


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
    ndev = torch.cuda.device_count()
    device = local_rank % max(1, ndev)
    shared_gpu = world > ndev  # a dry run of the N > 1 protocol on fewer GPUs
    torch.cuda.set_device(device)
    dist = None
    if world > 1:
        import torch.distributed as dist

        # control plane only (group id broadcast, max-over-ranks timing); the
        # data plane is the library's peer memory or its own NCCL communicator
        dist.init_process_group("gloo")
        if args.transport == "peer":
            uid = [quest.Env.peer_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            env = quest.Env.peer(rank, world, device, uid[0])
        else:
            uid = [quest.Env.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            env = quest.Env.nccl(rank, world, device, uid[0])
        env.set_qubit_swaps(bool(args.swaps))
    else:
        env = quest.Env()
    env.set_ordering(args.order == "reorder")
    if args.fusion or args.reg_qubits:
        env.set_fusion(args.fusion, 0, args.reg_qubits)
    if args.jit is not None:
        quest.set_jit(args.jit)

    def allmax(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

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

    # cold end-to-end: the first circuit of this process through the C-ABI
    # (pass shapes compile on background threads; the interpreter runs them
    # until their kernels load)
    barrier()
    t0 = time.perf_counter()
    q.initZeroState()
    C.apply_circuit(q, circuit)
    q.calcTotalProb()
    cold_s = allmax(time.perf_counter() - t0)

    # warm-up: each step queues its new pass shapes for the per-pass JIT and
    # waits for those compiles; later steps run the compiled kernels
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
    with ClockSampler(device) as clocks:
        barrier()
        start.record(stream)
        for _ in range(args.steps):
            C.apply_circuit(q, circuit)
            # a step ends its last pass (an async launch, no sync), so every
            # step runs the pass shapes the warm-up compiled
            q.flush()
        stop.record(stream)
        barrier()
    ms_launch, kinds = env.profile_stop()
    info = env.last_info
    launches = quest.kernel_launches() - launches0
    passes = q.pass_count() - passes0
    elapsed = allmax(start.elapsed_time(stop))  # ms
    value = effective_bytes(n, gates * args.steps) / (elapsed / 1e3) / 1e9
    ms_gate = elapsed / (gates * args.steps)

    # roofline of the dominant kernel (the fused pass)
    pk, src = peaks()
    pass_ms = ms_launch[kinds == 0]
    exch_ms = ms_launch[kinds == 2]  # per-gate exchanges (swaps off)
    swap_ms = ms_launch[kinds == 5]  # global<->local qubit swaps
    per_launch_bytes = 2.0 * AMP * (2.0 ** args.local_qubits)
    achieved = per_launch_bytes / (float(pass_ms.mean()) / 1e3) / 1e9 if pass_ms.size else None
    share = float(pass_ms.sum()) / float(ms_launch.sum()) if ms_launch.size else None

    # sanity: the timed steps kept the state normalised
    norm_error = abs(q.calcTotalProb() - 1.0)

    # the same tile kernel run one gate per pass (fusion mode 1): the
    # streaming roofline of a single-gate pass on the first 24 gates
    single = None
    if args.fusion == 0 and world == 1:
        sub = C.Circuit(n, circuit.depth, circuit.ops[:24])
        env.set_fusion(1, 0, 0)
        for _ in range(2):
            C.apply_circuit(q, sub)
            q.flush()
            quest.jit_wait()
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
                      "achieved_GBps": round(gbs, 1), "frac": round(gbs / pk["hbm_gbs"], 4),
                      "what": "one gate per tile pass (fusion mode 1), same kernel, same bytes per pass"}

    # side measurement: the same circuit in circuit order (bit-identical to
    # the reference), same register, same timing
    exact = None
    if args.order == "reorder" and not args.no_exact_side and args.fusion == 0:
        env.set_ordering(False)
        for _ in range(max(2, args.warmup)):
            C.apply_circuit(q, circuit)
            q.flush()
            env.sync()
            quest.jit_wait()
        barrier()
        p0x = q.pass_count()
        env.profile_start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            C.apply_circuit(q, circuit)
            q.flush()
        e1.record(stream)
        barrier()
        ms_x, k_x = env.profile_stop()
        t_x = allmax(e0.elapsed_time(e1))
        p_x = ms_x[k_x == 0]
        exact = {"order": "circuit order (bit-identical to the reference)",
                 "value": round(effective_bytes(n, gates * args.steps) / (t_x / 1e3) / 1e9, 1), "unit": UNIT,
                 "ms_per_step": round(t_x / args.steps, 3), "ms_per_gate": round(t_x / (gates * args.steps), 4),
                 "passes_per_step": (q.pass_count() - p0x) / args.steps,
                 "avg_pass_ms": round(float(p_x.mean()), 4) if p_x.size else None,
                 "pass_roofline_frac": round(per_launch_bytes / (float(p_x.mean()) / 1e3) / 1e9 / pk["hbm_gbs"], 4)
                 if p_x.size else None}
        env.set_ordering(True)

    # side measurement: the same circuit on a single-precision register
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
              "traffic": _traffic("k_tile_pass_single", args.local_qubits) if AMP == 16 else None,
              "norm_error": abs(qs.calcTotalProb() - 1.0)}
        qs.destroy()

    # e2e through the C-ABI from the host: init + gates + readback, wall clock
    e2e_vals = []
    h0, d0 = quest.transfer_bytes()
    reps = max(1, min(args.steps, 3))
    for _ in range(reps):
        barrier()
        t0 = time.perf_counter()
        q.initZeroState()
        C.apply_circuit(q, circuit)
        q.calcTotalProb()
        e2e_vals.append(time.perf_counter() - t0)
    h1, d1 = quest.transfer_bytes()
    e2e_t = allmax(statistics.median(e2e_vals))
    e2e = effective_bytes(n, gates) / e2e_t / 1e9
    h2d = (h1 - h0) // reps
    d2h = (d1 - d0) // reps

    # C5 side measurement: QFT + multi-controlled phase flips, then the
    # measurement tail (probabilities of every qubit, 4 collapses)
    c5 = None
    if not args.no_c5 and args.precision == "double":
        q.destroy()
        q = None
        c5 = run_c5(env, world, args, barrier, allmax, stream)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            vals, kind, workers, sample, _ = cpu_reference(n, circuit, args.cpu_gates, 2, os.cpu_count() or 1)
            cpu = {"value": round(statistics.median(vals), 3), "unit": UNIT, "cores": workers,
                   "kind": kind, "sample": sample}
        except Exception as e:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    # per-pass bound: max(HBM time of the pass's bytes at the measured copy
    # peak, FP64 time of its modelled instructions at the FP64 pipe's peak:
    # 148 SMs x 64 DFMA/clk x the max SM clock); the timed passes against
    # the sum of their bounds
    bound = None
    if pass_ms.size:
        pinfo = info[kinds == 0]
        fp64_per_amp = (pinfo >> 16) / 4.0
        fp64_rate = 148 * 64 * 1.965e9  # instructions / s
        t_hbm = per_launch_bytes / (pk["hbm_gbs"] * 1e9) * 1e3  # ms
        t_fp = fp64_per_amp * (2.0 ** args.local_qubits) / fp64_rate * 1e3
        t_bound = np.maximum(t_hbm, t_fp)
        bound = {"hbm_ms": round(t_hbm, 4), "fp64_ms_mean": round(float(t_fp.mean()), 4),
                 "fp64_bound_passes": int((t_fp > t_hbm).sum()),
                 "bound_ms_mean": round(float(t_bound.mean()), 4),
                 "frac_of_bound": round(float(t_bound.sum() / pass_ms.sum()), 4),
                 "fp64_model": "per handler class: 8 (generic 2x2), 4 (real / Rx-class / diagonal), 0 (swap) "
                               "FP64 instructions per amplitude, halved per control outside the tile; "
                               "peak 148 x 64 DFMA/clk x 1.965 GHz"}

    # per-pass-class split: passes by op count, each class's bandwidth
    classes = None
    if pass_ms.size:
        ops_per_pass = info[kinds == 0] & 0xFF
        if ops_per_pass.size == pass_ms.size:
            classes = []
            for lo, hi in ((1, 8), (9, 16), (17, 24), (25, 1 << 30)):
                m = (ops_per_pass >= lo) & (ops_per_pass <= hi)
                if m.any():
                    t = float(pass_ms[m].mean())
                    classes.append({"ops": f"{lo}-{hi}" if hi < (1 << 30) else f">={lo}", "launches": int(m.sum()),
                                    "avg_ms": round(t, 4),
                                    "frac": round(per_launch_bytes / (t / 1e3) / 1e9 / pk["hbm_gbs"], 4),
                                    "share_of_pass_time": round(float(pass_ms[m].sum() / pass_ms.sum()), 4)})

    if rank == 0:
        line = {
            "metric": metric_name(), "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(elapsed / args.steps, 3),
            "ms_per_gate": round(ms_gate, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dtype_name(), "data": "synthetic seeded circuit",
            "config": {"workload": workload_name(n, args.depth, args.seed),
                       "qubits": n, "local_qubits": args.local_qubits, "gates": gates,
                       "parallelism": f"amplitude partition over {world} GPU(s)"
                                      + (f", {args.transport} transport, qubit swaps {'on' if args.swaps else 'off'}"
                                         if world > 1 else ""),
                       "precision": args.precision,
                       "order": ("reorder: commuting ops scheduled into fewer passes (amplitudes within 1e-12 "
                                 "of the reference, tests/test_gpu_reorder.py)" if args.order == "reorder"
                                 else "exact: circuit order (bit-identical to the reference)"),
                       "l2": f"state {AMP << args.local_qubits >> 30} GiB per GPU >> 126 MB L2 (no flush needed)",
                       "passes_per_step": passes / args.steps, "fusion": args.fusion,
                       "jit": {"mode": quest.lib().qgpuGetJit(), "kernels": quest.jit_stats()[0],
                               "failed": quest.jit_stats()[1],
                               "compile_wait_s": round(jit_wait_s, 2) if args.warmup else None},
                       **({"shared_gpu": f"{world} ranks on {ndev} GPU(s): protocol dry run, not a scaling number"}
                          if shared_gpu else {})},
            "gpu_launches": int(launches),
            "e2e": {"value": round(e2e, 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "what": "initZeroState + one C-ABI call per gate + calcTotalProb readback, wall clock, "
                            "warm (pass kernels compiled); bytes from the library's transfer counters"},
            "e2e_cold": {"value": round(effective_bytes(n, gates) / cold_s / 1e9, 1), "unit": UNIT,
                         "seconds": round(cold_s, 3),
                         "what": "first circuit of a fresh process: pass shapes compile on background threads "
                                 "while the interpreter runs them"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1) if achieved else None,
                         "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": round(achieved / pk["hbm_gbs"], 4) if achieved else None,
                         "traffic": _traffic("k_tile_pass", args.local_qubits),
                         "kernel": "k_tile_jit" if quest.lib().qgpuGetJit() else "k_tile_pass",
                         "peak_source": src, "bytes_per_launch": per_launch_bytes,
                         "avg_launch_ms": round(float(pass_ms.mean()), 4) if pass_ms.size else None,
                         "launches": int(pass_ms.size), "share_of_step": round(share, 4) if share else None,
                         "per_pass_bound": bound, "passes_by_op_count": classes},
            "clocks": clocks.summary(),
            "check": {"norm_error_after_timed_steps": norm_error},
            "circuit_order": exact,
            "single_gate_pass": single,
            "single_precision": sp,
            "c5": c5,
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
                              "GBps_per_direction": round(nv, 1), "frac_of_900": round(nv / NVLINK_GBS, 4),
                              "share_of_step": round(t_s * 1e3 / elapsed, 4),
                              "what": "event pairs around each exchange / swap kernel (incl. its fences), "
                                      "rank 0's stream"}
        print(json.dumps(line), flush=True)
    if q is not None:
        q.destroy()
    env.destroy()
    if dist:
        dist.destroy_process_group()


def run_c5(env, world, args, barrier, allmax, stream):
    """C5 (BASELINE.json configs[4]): QFT of a basis state with a
    multiControlledPhaseFlip every 3 stages on 32 qubits (more if the
    partition allows), then calcProbOfOutcome on every qubit and
    collapseToOutcome on 4 qubits; ms per gate (device) and the tail's wall
    time."""
    import torch

    from paper_1802_08032_b200 import circuits as C
    from paper_1802_08032_b200 import quest

    n = 32
    c = C.qft_circuit(n, mcpf_every=3)
    q = quest.QuregHandle(env, n)
    try:
        q.initClassicalState(0x5A5A5A5A)
        C.apply_circuit(q, c)  # warm-up (JIT)
        q.flush()
        quest.jit_wait()
        q.initClassicalState(0x5A5A5A5A)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        C.apply_circuit(q, c)
        q.flush()
        e1.record(stream)
        barrier()
        gate_ms = allmax(e0.elapsed_time(e1))
        t0 = time.perf_counter()
        probs = [q.calcProbOfOutcome(t, 0) for t in range(n)]
        for t, o in [(0, 1), (9, 0), (21, 1), (n - 1, 0)]:
            q.collapseToOutcome(t, o)
        total = q.calcTotalProb()
        tail_ms = allmax((time.perf_counter() - t0) * 1e3)
        return {"workload": f"QFT of |0x5A5A5A5A> on {n} qubits, multiControlledPhaseFlip every 3 stages",
                "qubits": n, "gates": len(c.ops), "ms_per_gate": round(gate_ms / len(c.ops), 4),
                "effective_GBps": round(effective_bytes(n, len(c.ops)) / (gate_ms / 1e3) / 1e9, 1),
                "measurement_tail_ms": round(tail_ms, 3),
                "what_tail": f"calcProbOfOutcome on all {n} qubits + 4 collapseToOutcome + calcTotalProb",
                "check": {"max_abs_p_minus_half": max(abs(p - 0.5) for p in probs),
                          "norm_error": abs(total - 1.0)}}
    finally:
        q.destroy()


def main():
    global AMP
    args = parse_args()
    AMP = 8 if args.precision == "single" else 16
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(args))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
