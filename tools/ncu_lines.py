"""Aggregate an `ncu --page source --print-source cuda,sass --csv` dump to per-source-line stall
samples and executed instructions (used to read profiles/ captures)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = None
hdr = None
agg = []
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Function Name":
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) >= 8 and r[2] == "-":  # source-line summary rows
        try:
            agg.append((float(r[4] or 0), float(r[7] or 0), cur, r[0], r[1]))
        except ValueError:
            pass
tot = sum(a[0] for a in agg) or 1
tinst = sum(a[1] for a in agg) or 1
agg.sort(key=lambda a: -a[0])
print(f"total stall samples {tot:.0f}, warp instructions {tinst:.3e}")
for s, i, f, ln, src in agg[:top]:
    print(f"{100*s/tot:5.1f}%  inst {100*i/tinst:5.1f}%  {f}:{ln}  {src.strip()[:100]}")
