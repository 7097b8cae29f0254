"""Summarise ncu outputs for profiles/ (run here, no GPU needed).

  python tools/summarize_ncu.py launches <launches.csv>   # per-kernel share of a launch list
  python tools/summarize_ncu.py full <report.ncu-rep>     # key metrics of one --set full capture
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = ""
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        unit = r["Metric Unit"]
        v = float(r["Metric Value"].replace(",", ""))
        agg[name][0] += 1
        agg[name][1] += v
    total = sum(v for _, v in agg.values())
    print(f"| kernel | launches | total ({unit}) | share | mean ({unit}) |")
    print("|---|---|---|---|---|")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {v:.1f} | {100 * v / total:.1f}% | {v / n:.1f} |")


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__block_size", "launch__grid_size",
    "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print(f"kernel: `{d.get('Kernel Name', '?')[:120]}`\n")
    print("| metric | value |")
    print("|---|---|")
    for k in KEYS:
        if k in d:
            print(f"| {k} | {d[k]} {u.get(k, '')} |")
    st = {k: float(d[k].replace(",", "")) for k in d if "pcsamp_warps_issue_stalled" in k
          and "not_issued" not in k and d[k] not in ("", "n/a")}
    tot = sum(st.values()) or 1
    print("\nwarp stall reasons (sampled): " + ", ".join(
        f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%"
        for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2:
        h = srows[1]
        ia, isrc = h.index("Instructions Executed"), h.index("Source")
        op = collections.Counter()
        for r in srows[2:]:
            try:
                n = int(r[ia])
            except (ValueError, IndexError):
                continue
            t = r[isrc].split()
            if t:
                op[(t[1] if t[0].startswith("@") else t[0]).split(".")[0]] += n
        tot = sum(op.values()) or 1
        print("\nSASS opcode mix (executed): " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in op.most_common(12)))
        print("\ntcgen05 / TMA evidence: UBLKCP executed = %d" % op.get("UBLKCP", 0))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
