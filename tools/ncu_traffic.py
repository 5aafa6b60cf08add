"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
of the spread / gather kernels from an ncu --set full report into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic)."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, out=os.path.join(ROOT, "profiles", "ncu_traffic.json")):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    col = {k: i for i, k in enumerate(h)}
    units = rows[1]
    res = {}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        for kern in ("spread", "gather", "spread_cells"):
            if name.startswith(f"void mlb::{kern}_kernel") or f"{kern}_kernel<" in name:
                if kern == "spread_cells":  # the d = 3 spread
                    key = "spread_d3"
                else:
                    d = name.split("<")[1].split(",")[0].replace("(int)", "").strip()
                    key = f"{kern}_d{d}"

                def val(metric):
                    i = col[metric]
                    v = float(r[i].replace(",", ""))
                    u = units[i]
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                    return v * scale
                res[key] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    with open(out, "w") as fh:
        json.dump({"source": os.path.basename(rep), "bytes_per_launch": res, **res}, fh, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main(*sys.argv[1:])
