"""Per-launch DRAM bytes / duration / fp64-pipe use from an ncu report (raw page)."""
import csv
import subprocess
import sys


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2:]


if __name__ == "__main__":
    h, u, data = rows(sys.argv[1])
    col = lambda n: h.index(n) if n in h else None
    f64 = col("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active")
    for r in data:
        scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}
        tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
        rd = float(r[col("dram__bytes_read.sum")]) * scale[u[col("dram__bytes_read.sum")]]
        wr = float(r[col("dram__bytes_write.sum")]) * scale[u[col("dram__bytes_write.sum")]]
        print(r[col("ID")], r[col("Kernel Name")].split("(")[0], f"dram read {rd:.6f} GB write {wr:.6f} GB",
              f"duration {float(r[col('gpu__time_duration.sum')]) * tscale[u[col('gpu__time_duration.sum')]]:.3f} us",
              f"fp64 pipe {r[f64]} %" if f64 is not None else "")
