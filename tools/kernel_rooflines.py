"""Per-kernel DRAM throughput from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --csv:
mean per launch, achieved GB/s (measured DRAM bytes / duration) and the
fraction of the measured HBM peak (MEASURED_PEAKS.json). Cold, serialised
launches (ncu): shares and rates, not bench numbers.

    python tools/kernel_rooflines.py launches.csv
"""
import collections
import csv
import json
import os
import sys

UNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1}


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, ii = h.index("Kernel Name"), h.index("ID")
    mi, ui, vi = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").split("<")[0]
    peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"]
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    tmax = collections.defaultdict(float)
    for i, m in per.items():
        tmax[names[i]] = max(tmax[names[i]], m.get("gpu__time_duration.sum", 0))
    for i, m in per.items():
        # empty launches (e.g. the rebuild block's recompute with no rows) are skipped
        if m.get("gpu__time_duration.sum", 0) < max(2e-6, 0.05 * tmax[names[i]]):
            continue
        k = names[i]
        cnt[k] += 1
        for key, v in m.items():
            agg[k][key] += v
    print(f"{'kernel':22s} {'launches':>8s} {'us/launch':>10s} {'DRAM MB':>9s} {'GB/s':>8s} "
          f"{'% HBM':>6s} {'tensor %':>8s}")
    for k in sorted(agg, key=lambda k: -agg[k]["gpu__time_duration.sum"]):
        n = cnt[k]
        t = agg[k]["gpu__time_duration.sum"] / n
        b = (agg[k]["dram__bytes_read.sum"] + agg[k]["dram__bytes_write.sum"]) / n
        tp = agg[k].get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0) / n
        gbs = b / t / 1e9
        print(f"{k:22s} {n:8d} {t * 1e6:10.2f} {b / 1e6:9.2f} {gbs:8.1f} {100 * gbs / hbm:6.1f} "
              f"{tp:8.2f}")
    print(f"(HBM peak {hbm} GB/s, MEASURED_PEAKS.json; launches under 2 us or under 5% of the "
          f"kernel's longest are skipped)")


if __name__ == "__main__":
    main(sys.argv[1])
