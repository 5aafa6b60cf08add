"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of
the spread / gather kernels from an `ncu --set full` report, merged into
profiles/ncu_traffic.json under "<workload>:<kernel>_d<d>" (read by bench.py
for roofline.traffic).

    python tools/ncu_traffic.py <report.ncu-rep> <workload name>
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "ncu_traffic.json")


def kernel_key(name):
    if "spread_cells_kernel" in name:
        return "spread_d3"
    if "lat_spread_kernel" in name:
        return "spread_d2"
    if "lat_gather_kernel" in name:
        return "gather_d2"
    for kern in ("spread_kernel<", "gather_kernel<"):
        if kern in name:
            d = name.split(kern)[1].split(",")[0].replace("(int)", "").strip()
            return f"{kern[:-8]}_d{d}"
    return None


def main(rep, workload):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    col = {k: i for i, k in enumerate(h)}
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for r in rows[2:]:
        key = kernel_key(r[col["Kernel Name"]])
        if key is None:
            continue
        b = sum(float(r[col[m]].replace(",", "")) * scale.get(units[col[m]], 1)
                for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        per.setdefault(key, []).append(b)
    try:
        with open(OUT) as fh:
            data = json.load(fh)
    except (OSError, ValueError):
        data = {}
    for key, vals in per.items():
        data[f"{workload}:{key}"] = {"bytes": sum(vals) / len(vals), "launches": len(vals),
                                    "source": os.path.basename(rep)}
    with open(OUT, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
    print(json.dumps({k: v for k, v in data.items() if k.startswith(workload)}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
