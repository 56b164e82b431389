"""Per-SASS-instruction executed counts and stall samples of an ncu report (source page,
sass view), in address order; optionally only instructions executed >= min_count times.
  python tools/ncu_sass_hot.py report.ncu-rep [min_count] [groups]  (groups: divide counts)"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 0
div = float(sys.argv[3]) if len(sys.argv) > 3 else 1
out = subprocess.run(["ncu", "-i", rep, "--csv", "--page", "source", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
iS, iI = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
tot = 0
for r in rows[hi + 1:]:
    if len(r) <= iI:
        continue
    n = float(r[iI] or 0)
    tot += n
    if n >= mn:
        print(f"{r[0][-5:]} {n / div:8.2f} {r[iS]:>6} {r[1].strip()}")
print("total", tot / div)
