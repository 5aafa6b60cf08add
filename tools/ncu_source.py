"""Per-instruction stall hot spots of one kernel in an ncu report (needs -lineinfo)."""
import collections
import csv
import subprocess
import sys


def main(path, pattern, top=20):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1], None, []]
            blocks.append(cur)
        elif cur is not None and r and r[0] == "Address":
            cur[1] = r
        elif cur is not None and cur[1] is not None and len(r) > 5:
            cur[2].append(r)
    for name, h, data in blocks:
        if pattern not in name:
            continue
        si = h.index("Warp Stall Sampling (All Samples)")

        def I(x):
            try:
                return int(x)
            except ValueError:
                return 0
        tot = sum(I(r[si]) for r in data) or 1
        print(f"== {name[:90]}  instructions={len(data)} samples={tot}")
        byop = collections.Counter()
        for r in data:
            t = r[1].split()
            if t:
                op = t[1] if t[0].startswith("@") else t[0]
                byop[op.split(".")[0]] += I(r[si])
        print("   " + ", ".join(f"{op} {v / tot * 100:.1f}%" for op, v in byop.most_common(10)))
        idx = sorted(range(len(data)), key=lambda i: -I(data[i][si]))[:top]
        for i in sorted(idx):
            print(f"   {i:5d} {I(data[i][si]) / tot * 100:5.1f}%  {data[i][1].strip()[:90]}")
        break


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 20)
