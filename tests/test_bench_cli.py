"""The spec's bench CLI (SPEC.md [MODULE] bench-cli): memory report known
answers on CPU; BenchRecords from real runs on the GPU."""
import io
import json

import pytest

from paper_1802_08032_b200 import bench_cli

GiB = 1 << 30


def test_memory_report_kats():
    rows = bench_cli.report_memory(30, strategy="full_clone", node_bytes=64 * GiB)
    # 16 GiB state-only row; max_qubits 30 + k; ratio 2.0
    assert rows[0]["state_bytes"] == 16 * GiB
    assert [r["max_qubits"] for r in rows[:9]] == [30 + k for k in range(9)]
    assert all(r["ratio"] == 2.0 for r in rows)
    assert len(rows) == 17  # k in [0, 16]
    half = bench_cli.report_memory(30, strategy="half_exchange")
    assert half[1]["ratio"] == 1.5


def test_records_are_schema_stable():
    buf = io.StringIO()
    bench_cli.emit([{"num_qubits": 5, "comm_bytes": 0}], bench_cli.FIELDS, "json", buf)
    rec = json.loads(buf.getvalue())
    assert list(rec) == bench_cli.FIELDS and rec["measured_process_bytes"] is None
    buf = io.StringIO()
    bench_cli.emit([{"num_qubits": 5}], bench_cli.FIELDS, "csv", buf)
    header, row = buf.getvalue().splitlines()
    assert header.split(",") == bench_cli.FIELDS and len(row.split(",")) == len(bench_cli.FIELDS)


def test_cli_memory_mode_exit_code(capsys):
    assert bench_cli.main(["--mode", "memory", "--qubits", "20", "--format", "json"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert len(lines) == 17


@pytest.mark.gpu
def test_random_circuit_records():
    # (n=5, depth=10, 1 worker, k=0) -> time_per_gate > 0, no comm
    recs = bench_cli.bench_random_circuit(5, 10, 1, reps=5, warmup=1)
    assert len(recs) == 5 and all(r["time_per_gate_seconds"] > 0 and r["comm_bytes"] == 0 for r in recs)
    # (n=10, depth=10, k=2, full_clone): each rank sends one
    # message per communicated gate; repetitions carry identical counters
    from paper_1802_08032_b200 import circuits as C

    c = C.reference_random_circuit(10, 10, 3)
    comm_gates = sum(1 for op in c.ops
                     if op.target >= 8 and not (op.name in ("Z", "CZ", "RZ", "PHASE", "T", "S")))
    recs = bench_cli.bench_random_circuit(10, 10, 3, ranks_log2=2, strategy="full_clone", reps=3, warmup=1)
    assert len({r["comm_messages"] for r in recs}) == 1
    # exact count: one message per rank per communicated gate, minus the
    # ranks whose rank-bit controls fail (they skip the gate without traffic,
    # distributed.cpp:141-145); diagonal gates (T, CZ) never exchange here
    local = 8

    def passing_ranks(op):
        return sum(1 for r in range(4)
                   if all((r >> (cq - local)) & 1 for cq in op.controls if cq >= local))

    exact = sum(passing_ranks(op) for op in c.ops if op.target >= local and op.name not in ("T", "CZ", "Z"))
    assert recs[0]["comm_messages"] == exact
    assert recs[0]["comm_bytes"] == exact * 16 * (1 << local)
    import oracle

    if oracle.ref_available():  # the reference's own count (every global target exchanges)
        from tests.harness import to_oracle_ops

        _, msgs, byts, _ = oracle.ref_run_distributed(10, to_oracle_ops(c), 2, "full_clone")
        assert int(msgs.sum()) == sum(passing_ranks(op) for op in c.ops if op.target >= local)
        assert int(byts.sum()) == int(msgs.sum()) * 16 * (1 << local)
    swap = bench_cli.bench_random_circuit(10, 10, 3, ranks_log2=2, strategy="swap", reps=2, warmup=1)
    assert swap[0]["comm_bytes"] < recs[0]["comm_bytes"]


@pytest.mark.gpu
def test_rotation_sweep_threshold():
    # (n=12, k=2): targets 0..9 local, 10, 11 move 16 * 2^10 B per rank
    recs = bench_cli.bench_rotation_sweep(12, 2, reps=2)
    assert [r["communicated"] for r in recs] == [t >= 10 for t in range(12)]
    assert all(r["comm_bytes"] == 0 for r in recs[:10])
    assert all(r["comm_bytes"] == 4 * 16 * (1 << 10) for r in recs[10:])
    assert bench_cli.slowdown_ratio(recs) > 0
