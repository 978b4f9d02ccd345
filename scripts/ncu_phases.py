"""Executed warp instructions per barrier-delimited SASS segment of the decode
kernel (ncu --page source --csv --print-source sass): a phase breakdown that
does not depend on source-line attribution.  Usage: ncu_phases.py SASS_CSV FRAME_ITERS"""
import csv
import sys

rows = []
for r in csv.reader(open(sys.argv[1])):
    if len(r) > 8 and r[0].startswith("0x"):
        rows.append((int(r[0], 16), r[1].strip(), int(r[5]) if r[5].isdigit() else 0))
rows.sort()
base = rows[0][0]
fi = float(sys.argv[2])
segs, cur, start, cnt = [], 0, 0, 0
for a, src, i in rows:
    cur += i
    cnt += 1
    if "BAR.SYNC" in src or "BAR.RED" in src:
        segs.append((start, a - base, cur, cnt))
        cur, start, cnt = 0, a - base, 0
segs.append((start, rows[-1][0] - base, cur, cnt))
tot = sum(s[2] for s in segs)
print(f"total {tot:.3e} warp instructions = {tot / fi:.0f} per frame-iteration")
for s in segs:
    if s[2] / tot > 0.005:
        print(f"  {s[0]:#07x}-{s[1]:#07x}  {100 * s[2] / tot:5.1f}%  {s[2] / fi:6.0f}/frame-iter  ({s[3]} SASS instructions)")
