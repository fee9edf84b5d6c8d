"""DEVELOPMENT: per-source-line warp-stall samples and executed instructions
from `ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = []
fname = None
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] and r[0] not in ("Line No", "Function Name") and len(r) > 7 and r[4] != "-":
        try:
            rows.append((fname, int(r[0]), int(r[4]), int(r[7]), r[1][:90]))
        except ValueError:
            pass
ts = sum(x[2] for x in rows)
ti = sum(x[3] for x in rows)
print(f"total samples {ts}  total warp instructions {ti}")
key = 2 if len(sys.argv) < 3 or sys.argv[2] == "samples" else 3
for f, ln, s, i, src in sorted(rows, key=lambda x: -x[key])[: int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{f:16s}{ln:5d} {100*s/ts:5.1f}% {100*i/ti:5.1f}%  {src}")

if len(sys.argv) > 4:  # ranges "file:a-b,..." summed
    for spec in sys.argv[4].split(","):
        f, ab = spec.split(":")
        a, b = map(int, ab.split("-"))
        sel = [x for x in rows if x[0] == f and a <= x[1] <= b]
        print(f"{spec:24s} samples {100*sum(x[2] for x in sel)/ts:5.1f}%  instr {100*sum(x[3] for x in sel)/ti:5.1f}%")
