"""SASS instruction histogram of a kernel's main loop (the loop with the most HMMA/UTCHMMA),
static, from cuobjdump of a built object: proves which tensor-core / TMA instructions the hot
path uses (HMMA vs UTCHMMA, UTMALDG, LDSM ...).

  python tools/sass_hist.py paper_2505_10938_b200/_lib/obj/ott_attend.o attend_mma_kernelILi8ELi32
"""
import collections
import re
import subprocess
import sys

obj, name = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
body = next(f for f in funcs if f.split("\n", 1)[0].strip().find(name) >= 0)
ins = []
for line in body.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
whole = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for _, t in ins)
loops = []
for a, t in ins:
    m = re.search(r"BRA(?:\.U)?(?:\.ANY)?\s+(0x[0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        s = int(m.group(1), 16)
        b = [x for (addr, x) in ins if s <= addr <= a]
        loops.append((sum("MMA" in x for x in b), len(b), s, a))
loops.sort(reverse=True)
print(f"kernel {name}: {len(ins)} SASS instructions")
print("whole kernel, selected opcodes:", {k: whole[k] for k in sorted(whole) if re.search(
    "MMA|UTMA|UBLKCP|LDSM|MOVM|STTM|LDTM|SYNCS", k)})
if loops:
    n, L, s, e = loops[0]
    b = [x for (addr, x) in ins if s <= addr <= e]
    c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in b)
    print(f"main loop [{s:#x}, {e:#x}]: {L} instructions")
    for k, v in c.most_common():
        print(f"  {v:5d} {k}")
