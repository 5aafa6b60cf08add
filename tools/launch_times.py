"""Per-kernel average durations from an ncu --csv launch list (profiling aid).

    python tools/launch_times.py gpurun_out/launches.csv
"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            agg[r[ki][:70]].append(float(r[vi].replace(",", "")))
    unit = "ns"
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{sum(v) / len(v) / 1e3:9.2f} us x{len(v):4d}  {sum(v) / tot * 100:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
