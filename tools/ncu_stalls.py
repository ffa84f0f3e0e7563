"""Sum the per-instruction warp-stall columns of an `ncu --page source --csv --print-source sass` dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Address")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = {hdr[i]: 0.0 for i in cols}
for r in rows:
    if r and r[0].startswith("0x") and len(r) == len(hdr):
        for i in cols:
            tot[hdr[i]] += float(r[i] or 0)
s = sum(tot.values()) or 1
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    if v:
        print(f"{k:28s} {100 * v / s:5.1f}%")
