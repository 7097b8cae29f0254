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
