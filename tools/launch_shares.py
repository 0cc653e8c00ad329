"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_shares.py launches.csv [batches] > shares.txt
"""
import collections
import csv
import sys


def main(path, batches=10):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0]
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
        tot[name] += us
        cnt[name] += 1
    s = sum(tot.values())
    print(f"sum of launch times per batch: {s / batches:.1f} us")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:24s} launches={cnt[k]:4d} {v / cnt[k]:9.2f} us/launch {100 * v / s:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 10)
