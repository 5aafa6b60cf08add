"""Stall reasons per SASS region of one kernel in an ncu report (profiling aid).

    python tools/ncu_regions.py REPORT PATTERN [BIN]
"""
import csv
import subprocess
import sys


def main(path, pattern, binsz=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name" and pattern in r[1]]
    if not starts:
        print("no kernel matches", pattern)
        return
    s0 = starts[0]
    h = rows[s0 + 1]
    data = []
    for r in rows[s0 + 2:]:
        if r and r[0] == "Kernel Name":
            break
        data.append(r)
    stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    si = {c: h.index(c) for c in stalls}
    ex = h.index("Instructions Executed")

    def I(x):
        try:
            return int(x)
        except ValueError:
            return 0
    tot = sum(I(r[si[c]]) for r in data for c in stalls) or 1
    print(f"{rows[s0][1][:80]}  instructions={len(data)}")
    for b in range(0, len(data), binsz):
        seg = data[b:b + binsz]
        per = {c: sum(I(r[si[c]]) for r in seg) for c in stalls}
        s = sum(per.values())
        if s / tot < 0.01:
            continue
        top = sorted(per.items(), key=lambda x: -x[1])[:5]
        exe = max(I(r[ex]) for r in seg)
        print(f"{b:5d} {s / tot * 100:5.1f}% maxexec {exe:8d} " +
              " ".join(f"{k[6:]}={v / tot * 100:.1f}" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
