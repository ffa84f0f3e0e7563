"""Hot-code footprint of a kernel from `ncu --page source --csv --print-source sass`: how many bytes
of SASS carry a given share of the executed instructions (instruction-cache working set).
python tools/ncu_hot_footprint.py dump.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "Address")
ie = hdr.index("Instructions Executed")
ins = []
for r in rows:
    if r and r[0].startswith("0x") and len(r) == len(hdr):
        ins.append((int(r[0], 16), float(r[ie] or 0), r[1]))
tot = sum(x[1] for x in ins)
print(f"SASS instructions {len(ins)} ({16 * len(ins) / 1024:.0f} KB), executed {tot:.3e}")
srt = sorted(ins, key=lambda x: -x[1])
acc = 0.0
marks = [0.5, 0.8, 0.9, 0.95, 0.99, 0.999]
mi = 0
for k, x in enumerate(srt):
    acc += x[1]
    while mi < len(marks) and acc >= marks[mi] * tot:
        print(f"  {100 * marks[mi]:5.1f}% of executed instructions in the hottest {k + 1} SASS lines = {16 * (k + 1) / 1024:.1f} KB")
        mi += 1
lines = {}
for a, e, _ in ins:
    lines[a // 128] = lines.get(a // 128, 0) + e
hot = [v for v in lines.values() if v > 0]
print(f"  128-B code lines touched: {len(hot)} ({len(hot) * 128 / 1024:.0f} KB); "
      f"lines with >= 1e-4 of executions: {sum(1 for v in hot if v >= 1e-4 * tot)}, >= 1e-5: {sum(1 for v in hot if v >= 1e-5 * tot)}")
