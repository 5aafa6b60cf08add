"""Summarise an ncu report: per kernel duration, occupancy, throughput, top stalls."""
import csv
import subprocess
import sys


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    col = {k: i for i, k in enumerate(h)}
    keys = [("gpu__time_duration.sum", "dur"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
            ("launch__registers_per_thread", "regs"), ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
            ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
            ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64pipe%"),
            ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64cyc%"),
            ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
            ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
            ("launch__grid_size", "grid"), ("launch__block_size", "block")]
    for r in rows[2:]:
        name = r[col["Kernel Name"]][:60]
        out = []
        for k, lab in keys:
            if k in col:
                out.append(f"{lab}={r[col[k]]}")
        stalls = []
        for k, i in col.items():
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), k.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print(name)
        print("   " + " ".join(out))
        print("   stalls: " + ", ".join(f"{n}={v:.2f}" for v, n in stalls[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
