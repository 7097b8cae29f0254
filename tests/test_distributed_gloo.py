"""N>1 path on CPU: world_size-2 (and 4) gloo process groups run the product's
host-side exchange plan (qgpuPlanGate / qgpuPlanChunks from libqgpu.so —
pure host code, no GPU) over real torch.distributed send/recv, with the
oracle's restated kernels (apply_gate_span / combine) standing in for the
device kernels. The gathered state must equal the single-rank result and the
reference's own distributed engine bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1802_08032_b200 import quest
from tests.harness import random_gate_circuit, to_oracle_ops


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, seed, chunk, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k = world.bit_length() - 1
    L = 1 << (n - k)
    ops = to_oracle_ops(random_gate_circuit(n, 60, seed, max_controls=2))
    full = oracle.zero_state(n)
    mine = full[rank * L:(rank + 1) * L].copy()
    nchunks, clen = quest.plan_chunks(L, chunk)
    msgs = 0
    for op in ops:
        t, mask = int(op["target"]), int(op["ctrl_mask"])
        kind, peer, own_lo, low = quest.plan_gate(n, k, rank, t, mask)
        if kind == "skip":
            continue
        if kind == "local":
            oracle.restated().orc_apply_gate(mine.ctypes.data, n - k, t, low, op["m"].ctypes.data)
            continue
        # sub-chunked pairwise exchange; chunk j is sent before it is combined
        for j in range(nchunks):
            sl = slice(j * clen, (j + 1) * clen)
            send = torch.from_numpy(mine[sl].view(np.float64).copy())
            recv = torch.empty_like(send)
            reqs = [dist.isend(send, peer), dist.irecv(recv, peer)]
            for r in reqs:
                r.wait()
            theirs = recv.numpy().view(np.complex128)
            lowmask_chunk = low
            # combine on local indices j*clen + i (controls on local bits)
            idx = np.arange(j * clen, (j + 1) * clen, dtype=np.uint64)
            part = oracle.orc_combine(mine[sl], theirs, 0, own_lo, op["m"])
            sel = (idx & np.uint64(lowmask_chunk)) == np.uint64(lowmask_chunk)
            mine[sl] = np.where(sel, part, mine[sl])
            msgs += 1
    gathered = [torch.empty(2 * L, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(mine.view(np.float64).copy()))
    if rank == 0:
        state = np.concatenate([g.numpy().view(np.complex128) for g in gathered])
        np.save(out_path, state)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,chunk", [(2, 9, 32), (2, 7, 1 << 20), (4, 8, 16)])
def test_gloo_exchange_protocol_matches_single_rank(tmp_path, world, n, chunk):
    seed = 1000 + world * 10 + n
    out = tmp_path / "state.npy"
    mp.spawn(_worker, args=(world, _free_port(), n, seed, chunk, str(out)), nprocs=world, join=True)
    got = np.load(out)
    ops = to_oracle_ops(random_gate_circuit(n, 60, seed, max_controls=2))
    want = oracle.orc_run(n, ops)
    assert np.array_equal(got, want)
    if oracle.ref_available():
        k = world.bit_length() - 1
        ref_out, *_ = oracle.ref_run_distributed(n, ops, k, "per_amplitude", block_amps=chunk)
        assert np.array_equal(got, ref_out)


def _swap_worker(rank, world, port, n, seed, chunk, out_path):
    """Global<->local qubit swaps (qgpuPlanSwaps decisions) over gloo: the
    half-partition trade of QuregImpl::run_swap, then every gate is local."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    k = world.bit_length() - 1
    m = n - k
    L = 1 << m
    ops = to_oracle_ops(random_gate_circuit(n, 80, seed, max_controls=2))
    plan = quest.plan_swaps(n, k, [(int(o["target"]), True) for o in ops], chunk)
    swaps_at = {}
    for i, g, v in plan:
        swaps_at.setdefault(i, []).append((g, v))
    l2p, p2l = list(range(n)), list(range(n))
    mine = oracle.zero_state(n)[rank * L:(rank + 1) * L].copy()
    for i, op in enumerate(ops):
        for g, v in swaps_at.get(i, []):
            j, a = g - m, (rank >> (g - m)) & 1
            peer = rank ^ (1 << j)
            block = 1 << v
            unit = min(chunk, block, L // 2)
            for u in range((L // 2) // unit):
                e = u * unit
                off = ((e >> v) << (v + 1)) | ((a ^ 1) << v) | (e & (block - 1))
                send = torch.from_numpy(mine[off:off + unit].view(np.float64).copy())
                recv = torch.empty_like(send)
                for r in [dist.isend(send, peer), dist.irecv(recv, peer)]:
                    r.wait()
                mine[off:off + unit] = recv.numpy().view(np.complex128)
            lg, lv = p2l[g], p2l[v]
            p2l[g], p2l[v], l2p[lg], l2p[lv] = lv, lg, v, g
        t = l2p[int(op["target"])]
        assert t < m, "a planned swap left the target global"
        pmask = 0
        for q in range(n):
            if (int(op["ctrl_mask"]) >> q) & 1:
                pmask |= 1 << l2p[q]
        rank_mask = pmask >> m
        if (rank & rank_mask) != rank_mask:
            continue  # a control on a global position fails on this rank
        oracle.restated().orc_apply_gate(mine.ctypes.data, m, t, pmask & (L - 1), op["m"].ctypes.data)
    gathered = [torch.empty(2 * L, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(mine.view(np.float64).copy()))
    if rank == 0:
        phys = np.concatenate([g.numpy().view(np.complex128) for g in gathered])
        # physical bit p holds logical qubit p2l[p]: back to the logical order
        idx = np.arange(1 << n, dtype=np.int64)
        src = np.zeros_like(idx)
        for p in range(n):
            src |= ((idx >> p2l[p]) & 1) << p
        np.save(out_path, phys[src])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,chunk", [(2, 9, 32), (4, 8, 16), (4, 10, 1 << 20)])
def test_gloo_qubit_swaps_match_single_rank(tmp_path, world, n, chunk):
    seed = 2000 + world * 10 + n
    out = tmp_path / "state.npy"
    mp.spawn(_swap_worker, args=(world, _free_port(), n, seed, chunk, str(out)), nprocs=world, join=True)
    ops = to_oracle_ops(random_gate_circuit(n, 80, seed, max_controls=2))
    assert np.array_equal(np.load(out), oracle.orc_run(n, ops))


def test_swap_plan_traffic_on_layered_circuits():
    """Belady eviction over the buffered window: a 36-qubit / 8-rank layered
    circuit needs well under half the reference's exchange traffic (a swap
    moves half a partition, an exchange gate a whole one)."""
    from paper_1802_08032_b200 import circuits as C

    for n, k in [(36, 3), (33, 3), (12, 2)]:
        c = C.layered_random_circuit(n, 20, 12345)
        ops = []
        for o in c.ops:
            mm = o.m8()
            ops.append((o.target, not (mm[2] == 0 and mm[3] == 0 and mm[4] == 0 and mm[5] == 0)))
        plan = quest.plan_swaps(n, k, ops)
        exch = sum(1 for t, p in ops if p and t >= n - k)
        assert 0.5 * len(plan) < 0.45 * exch, (n, k, len(plan), exch)
        # every swap trades a global position for a local one
        assert all(g >= n - k > v for _, g, v in plan)


def test_lightcone_drain_swaps_on_layered_circuits():
    """The default ordering's light-cone drain (qgpuPlanDistributed, host
    dry run of the runtime's own queue): a layered circuit touches every
    qubit per layer, so circuit order swaps the global qubits in and out
    every few layers; releasing every op that can run with the local qubits
    first needs a handful of swaps per step — and far fewer tile passes,
    since each swap drains the pass window. 36 qubits on 8 ranks (BASELINE
    C3b): 6 swaps and 25 passes per step against 27 and 96."""
    from paper_1802_08032_b200 import circuits as C
    from tests.test_reorder_plan import flat_ops

    for n, k, max_swaps in [(36, 3, 8), (35, 2, 6), (34, 1, 3), (27, 1, 3)]:
        ops = flat_ops(C.layered_random_circuit(n, 20, 12345))
        p_lc, sw_lc = quest.plan_distributed(n, k, ops, reorder=True)
        p_ex, sw_ex = quest.plan_distributed(n, k, ops, reorder=False)
        assert len(sw_lc) <= max_swaps, (n, k, len(sw_lc))
        assert 2 * len(sw_lc) < len(sw_ex) and 2 * p_lc < p_ex, (n, k, p_lc, p_ex, len(sw_lc), len(sw_ex))
        # every swap trades a global position for a local one off the lane qubits
        assert all(g >= n - k and 5 <= v < n - k for g, v in sw_lc)
