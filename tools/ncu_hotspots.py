"""Top SASS instructions by a stall reason from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep, col = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "Warp Stall Sampling (All Samples)"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--csv", "--page", "source", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS, iA, iC = hdr.index("Source"), hdr.index("Address"), hdr.index(col)
seq = []
for r in rows[2:]:
    try:
        seq.append((int(r[iC]), int(r[iA], 16), r[iS].strip()))
    except (ValueError, IndexError):
        pass
base = min(a for _, a, _ in seq)
tot = sum(w for w, _, _ in seq) or 1
print(f"{col}: total {tot}")
for w, a, s in sorted(seq, reverse=True)[:n]:
    print(f"{w:6d} {100 * w / tot:5.1f}% +{a - base:6d} {s[:90]}")
