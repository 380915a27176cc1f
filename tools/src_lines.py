"""Per-CUDA-source-line instruction counts from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur_file = None
out = []
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or not r[0]:
        continue
    ie = hdr.index("Instructions Executed")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        out.append((int(r[ie]), int(r[ws]), cur_file, r[0], r[1][:90]))
    except ValueError:
        pass
tot = sum(o[0] for o in out)
tws = sum(o[1] for o in out)
out.sort(reverse=True)
for n, w, f, ln, src in out[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100 * n / tot:5.1f}% {100 * w / max(tws, 1):5.1f}%  {f}:{ln}  {src.strip()}")
