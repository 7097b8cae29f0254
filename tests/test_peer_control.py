"""The peer transport's host control plane (peer.h) on CPU: a shared-memory
group of processes runs checked all-gathers and barriers (the mailboxes that
carry IPC handles, reduction partials, single amplitudes and the RNG seed),
and a rank that dies mid-protocol makes the survivors fail with
QGPU_COMM_ERROR naming it instead of hanging (the failure the reference's
InProcessTransport barrier cannot report)."""
import ctypes
import multiprocessing as mp
import os
import time

import pytest

from paper_1802_08032_b200 import quest


def _probe(uid, rank, n, rounds, exit_after, q):
    os.environ["QGPU_PEER_TIMEOUT_S"] = "60"
    rc = quest.lib().qgpuPeerProbe(uid, rank, n, rounds, exit_after)
    buf = ctypes.create_string_buffer(512)
    quest.lib().qgpuGetLastError(buf, 512)
    q.put((rank, rc, buf.value.decode()))


def _run(n, rounds, exit_rank=-1, exit_after=-1, limit=60.0):
    uid = quest.Env.peer_unique_id()
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    procs = [ctx.Process(target=_probe, args=(uid, r, n, rounds, exit_after if r == exit_rank else -1, q))
             for r in range(n)]
    for p in procs:
        p.start()
    t0 = time.time()
    try:
        while any(p.is_alive() for p in procs):  # is_alive() reaps exited children
            if time.time() - t0 > limit:
                raise AssertionError("peer probe hung")
            time.sleep(0.01)
    finally:
        for p in procs:
            if p.is_alive():
                p.kill()
            p.join()
    out = {}
    while not q.empty():
        r, rc, msg = q.get()
        out[r] = (rc, msg)
    return out, time.time() - t0, [p.exitcode for p in procs]


@pytest.mark.parametrize("n", [2, 4, 8])
def test_peer_group_allgather_and_barrier(n):
    out, _, codes = _run(n, 300)
    assert codes == [0] * n
    assert sorted(out) == list(range(n))
    assert all(rc == 0 for rc, _ in out.values()), out


def test_dead_rank_fails_partners_fast():
    out, dt, codes = _run(3, 400, exit_rank=2, exit_after=50)
    assert codes[2] == 3
    assert set(out) == {0, 1}
    for rc, msg in out.values():
        assert rc == 3 and "rank 2" in msg and "exited" in msg, msg
    assert dt < 30


def test_group_needs_a_valid_id():
    rc = quest.lib().qgpuPeerProbe(b"/qgpu-peer-does-not-exist", 0, 2, 1, -1)
    assert rc == 3
