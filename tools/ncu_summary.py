"""Key per-kernel metrics from an ncu report (--page details --csv)."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Theoretical Occupancy", "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "Warp Cycles Per Issued Instruction", "No Eligible", "Eligible Warps Per Scheduler",
        "Dynamic Shared Memory Per Block"]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    lines, cur = [], None
    for r in rows[1:]:
        if r[mi] in WANT:
            k = (r[ii], r[ki][:40])
            if k != cur:
                lines.append(f"--- {k[0]} {k[1]}")
                cur = k
            lines.append(f"    {r[mi]}: {r[vi]} {r[ui]}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summary(sys.argv[1]))
