"""Executed warp instructions per SASS instruction inside an address range of
an `ncu --page source --csv --print-source sass` export.
Usage: sass_seg.py SASS_CSV FRAME_ITERS LO HI [MIN_PER_FI]"""
import csv
import sys

rows = []
for r in csv.reader(open(sys.argv[1])):
    if len(r) > 8 and r[0].startswith("0x"):
        rows.append((int(r[0], 16), r[1].strip(), int(r[5]) if r[5].isdigit() else 0, int(r[6]) if r[6].isdigit() else 0))
rows.sort()
base = rows[0][0]
fi = float(sys.argv[2])
lo, hi = int(sys.argv[3], 16), int(sys.argv[4], 16)
thr = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
seg = [(a - base, s, i, t) for a, s, i, t in rows if lo <= a - base < hi]
print("segment total per frame-iteration", round(sum(x[2] for x in seg) / fi, 1))
for a, s, i, t in seg:
    if i / fi >= thr:
        print(f"{a:#07x} {i / fi:7.1f} {t / max(i, 1):5.1f}  {s[:90]}")
