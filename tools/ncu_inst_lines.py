"""Executed warp instructions per CUDA source line (per token if given), from an ncu report.
  python tools/ncu_inst_lines.py report.ncu-rep [tokens] [n]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
tokens = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--csv", "--page", "source", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
iI = hdr.index("Instructions Executed")
fname, inst, text = "", collections.Counter(), {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) < len(hdr) or not r[0].strip().isdigit():
        continue
    k = (fname, int(r[0]))
    text[k] = r[1].strip()
    try:
        inst[k] += int(r[iI] or 0)
    except ValueError:
        pass
tot = sum(inst.values())
print(f"total {tot / tokens:.2f} per token")
for k, v in inst.most_common(n):
    print(f"{v / tokens:6.2f} {100 * v / tot:5.1f}% {k[0][:14]}:{k[1]:<5} {text[k][:95]}")
