"""Per-instruction hot spots of an ncu capture (run here, no GPU needed).

  python tools/ncu_hotspots.py REPORT.ncu-rep [top]

Exports the source page (SASS) and prints: the stall-sample total per
reason, the samples per opcode, and the `top` instructions by samples with
their dominant stall reasons. Needs the kernel compiled with -lineinfo.
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
col = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


tot = collections.Counter()
by_op = collections.Counter()
for r in data:
    for h in reasons:
        tot[h] += num(r[col[h]])
    op = r[col["Source"]].split()[0] if r[col["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[col["Source"]].split()[1]
    by_op[op.split(".")[0]] += num(r[col["Warp Stall Sampling (All Samples)"]])
S = sum(tot.values()) or 1
print("stall samples by reason:", ", ".join(f"{k[6:]} {100 * v / S:.1f}%" for k, v in tot.most_common(10)))
print("samples by opcode:", ", ".join(f"{k} {100 * v / S:.1f}%" for k, v in by_op.most_common(14)))
data.sort(key=lambda r: -num(r[col["Warp Stall Sampling (All Samples)"]]))
for r in data[:top]:
    s = num(r[col["Warp Stall Sampling (All Samples)"]])
    rs = sorted(((num(r[col[h]]), h[6:]) for h in reasons), reverse=True)[:3]
    print(f"{100 * s / S:5.2f}%  {r[col['Source']].strip()[:60]:60s} " + " ".join(f"{n}:{int(v)}" for v, n in rs if v))
