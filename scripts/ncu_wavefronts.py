"""Per-source-line shared-memory wavefronts (and % of ideal) from
`ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

hdr = None
rows = []
fname = "?"
for r in csv.reader(open(sys.argv[1])):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    if len(r) > 2 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 8 and r[0].isdigit():
        k, ki = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
        w = int(r[k]) if r[k].isdigit() else 0
        wi = int(r[ki]) if r[ki].isdigit() else 0
        rows.append((w, wi, fname, int(r[0]), r[1].strip()[:80]))
tot = sum(x[0] for x in rows)
print("total wavefronts", tot, "ideal", sum(x[1] for x in rows))
for w, wi, f, ln, s in sorted(rows, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100 * w / tot:5.1f}% ideal {100 * wi / max(w, 1):4.0f}% {f}:{ln} {s}")
