"""Aggregate an ncu source page (cuda,sass) by CUDA source line: share of
executed instructions and of stall samples.
    ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [n]"""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg, cur, h = {}, None, None
for row in r:
    if not row:
        continue
    if row[0] in ("File Path", "File Name"):
        cur = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        h = row
        continue
    if h is None or len(row) < 8 or not row[0]:
        continue
    try:
        inst, st = float(row[7] or 0), float(row[4] or 0)
    except ValueError:
        continue
    a = agg.setdefault((cur, row[0], row[1].strip()[:80]), [0.0, 0.0])
    a[0] += inst
    a[1] += st
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"instructions {ti:.0f}, stall samples {ts:.0f}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{100 * v[0] / ti:5.1f}% inst {100 * v[1] / ts:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")
