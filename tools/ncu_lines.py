"""Per-CUDA-line stall samples / executed instructions of an ncu report
(--print-source cuda,sass; needs -lineinfo).  usage: ncu_lines.py <rep> [top]"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(io.StringIO(raw)))
f = "?"
hdr = None
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        try:
            s = int(r[4])
            e = int(r[7])
        except ValueError:
            continue
        agg.append((s, e, f, r[0], r[1].strip()[:80]))
tot = sum(a[0] for a in agg) or 1
tote = sum(a[1] for a in agg) or 1
print(f"total samples {tot}, warp instructions {tote}")
for s, e, f, ln, src in sorted(agg, reverse=True)[:top]:
    print(f"{s / tot:6.3f} {e / tote:6.3f}  {f}:{ln}  {src}")
