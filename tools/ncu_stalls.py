"""Stall attribution of one ncu --set full capture by SASS opcode.

  python tools/ncu_stalls.py <report.ncu-rep> [top]
Sums the sampled warp stalls (all samples / not-issued samples) and the
executed instructions per opcode from the source page, and lists the
instructions with the most stall samples.
"""
import collections
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ia, isrc = h.index("Instructions Executed"), h.index("Source")
iall, inot = h.index("Warp Stall Sampling (All Samples)"), h.index("Warp Stall Sampling (Not-issued Samples)")
by_op = collections.defaultdict(lambda: [0, 0, 0])
lines = []
for r in rows[2:]:
    try:
        n, a, ni = int(r[ia] or 0), int(r[iall] or 0), int(r[inot] or 0)
    except (ValueError, IndexError):
        continue
    t = r[isrc].split()
    if not t:
        continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    by_op[op][0] += n
    by_op[op][1] += a
    by_op[op][2] += ni
    lines.append((a, r[0], r[isrc][:70]))
ta = sum(v[1] for v in by_op.values()) or 1
tn = sum(v[0] for v in by_op.values()) or 1
print("| opcode | executed | share | stall samples (all) | share |")
print("|---|---|---|---|---|")
for op, (n, a, ni) in sorted(by_op.items(), key=lambda x: -x[1][1])[:top]:
    print(f"| {op} | {n} | {100 * n / tn:.1f}% | {a} | {100 * a / ta:.1f}% |")
print()
for a, addr, s in sorted(lines, reverse=True)[:top]:
    print(f"{a:8d} {addr} {s}")
