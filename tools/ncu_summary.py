"""Summarise one ncu report: key metrics + instruction/stall hot spots (SASS).

    python tools/ncu_summary.py rep.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_bytes.sum"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, top=30):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    print(vals[hdr.index("Kernel Name")][:80])
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            print(f"  {k:70s} {vals[i]:>16s} {units[i]}")
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            try:
                if float(vals[i]) > 0.3:
                    print(f"  {h[34:]:70s} {vals[i]:>16s}")
            except ValueError:
                pass
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hdr, data = rows[1], rows[2:]
    ia, isamp, src = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    tot = sum(int(r[ia] or 0) for r in data) or 1
    ts = sum(int(r[isamp] or 0) for r in data) or 1
    print(f"  SASS instructions executed {tot}, stall samples {ts}")
    ops, ops_s = collections.Counter(), collections.Counter()
    for r in data:
        t = r[src].strip().split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
        ops[op] += int(r[ia] or 0)
        ops_s[op] += int(r[isamp] or 0)
    print("  opcode mix (inst %, stall-sample %):")
    for op, n in ops.most_common(18):
        print(f"    {op:10s} {100 * n / tot:5.1f}%  {100 * ops_s[op] / ts:5.1f}%")
    print("  top stall instructions:")
    for k in sorted(range(len(data)), key=lambda k: -int(data[k][isamp] or 0))[:top]:
        r = data[k]
        print(f"    {k:5d} {100 * int(r[isamp] or 0) / ts:5.1f}%  n={r[ia]:>9s}  {r[src].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
