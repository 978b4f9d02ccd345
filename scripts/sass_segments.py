"""Per barrier-delimited SASS segment: stall samples, instructions and shared
wavefronts per unit (frame or frame-iteration), from an
`ncu --page source --csv --print-source sass` export.
Usage: sass_segments.py SASS_CSV UNITS"""
import csv
import sys

rows, hdr = [], None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) > 8 and r[0].startswith("0x"):
        rows.append(r)
base = min(int(r[0], 16) for r in rows)
iS = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
iw = hdr.index("L1 Wavefronts Shared")
rows.sort(key=lambda r: int(r[0], 16))
tot = sum(int(r[iS] or 0) for r in rows)
u = float(sys.argv[2])
cur, start = [0, 0, 0], 0
print(f"total: {sum(int(r[ie] or 0) for r in rows) / u:.0f} instructions, {sum(int(r[iw] or 0) for r in rows) / u:.0f} shared wavefronts per unit")
for r in rows + [None]:
    if r is not None:
        a = int(r[0], 16) - base
        cur[0] += int(r[iS] or 0)
        cur[1] += int(r[ie] or 0)
        cur[2] += int(r[iw] or 0)
    if r is None or "BAR.SYNC" in r[1]:
        if cur[0] / tot > 0.01:
            print(f"  {start:#07x}-{(a if r is not None else 0):#07x}  samples {100 * cur[0] / tot:5.1f}%  inst {cur[1] / u:6.0f}  wavefronts {cur[2] / u:6.0f}")
        cur, start = [0, 0, 0], (a if r is not None else 0)
