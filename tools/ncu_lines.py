"""Aggregate an ncu report's per-SASS warp-stall samples and executed
instructions by CUDA source line (needs -lineinfo + --import-source on).
  python tools/ncu_lines.py report.ncu-rep [n]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--csv", "--page", "source", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iI = hdr.index("Instructions Executed")
stall, inst, text = collections.Counter(), collections.Counter(), {}
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) < len(hdr) or not r[0].strip().isdigit():
        continue
    key = (fname, int(r[0]))
    text[key] = r[1].strip()
    try:
        stall[key] += int(r[iS] or 0)
        inst[key] += int(r[iI] or 0)
    except ValueError:
        pass
tot_s, tot_i = sum(stall.values()) or 1, sum(inst.values()) or 1
print(f"total stall samples {tot_s}, instructions {tot_i}")
for key, v in stall.most_common(n):
    print(f"{v:7d} {100 * v / tot_s:5.1f}%  inst {100 * inst[key] / tot_i:5.1f}%  {key[0][:14]}:{key[1]:<5} {text.get(key, '')[:90]}")
