"""Per-source-line warp samples / instructions from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = []
fname = "?"
tot_s = tot_i = 0
with open(sys.argv[1]) as fh:
    for r in csv.reader(fh):
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
        if len(r) > 8 and r[0] not in ("", "Line No") and r[0].isdigit():
            s, i = (int(r[4]) if r[4].isdigit() else 0), (int(r[7]) if r[7].isdigit() else 0)
            tot_s += s
            tot_i += i
            rows.append((s, i, fname, int(r[0]), r[1].strip()[:90]))
rows.sort(reverse=True)
print(f"total samples {tot_s} inst {tot_i}")
for s, i, f, ln, src in rows[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*s/tot_s:5.1f}% {100*i/tot_i:5.1f}%i {f}:{ln} {src}")
