"""Summarise an ncu report: key throughput metrics, stall reasons and the SASS
instruction mix (per token if --tokens is given). Used to write profiles/*.md."""
import csv
import collections
import io
import subprocess
import sys


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, "--csv", *args], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    tokens = float(sys.argv[2]) if len(sys.argv) > 2 else None
    rows = ncu_csv(rep, "--page", "raw")
    d = dict(zip(rows[0], rows[2] if len(rows) > 2 else rows[1]))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__cycles_active.avg", "sm__cycles_elapsed.avg"]
    for k in keys:
        print(f"{k:60s} {d.get(k)}")
    print("stalls (warps per issue):")
    st = {k: float(v) for k, v in d.items() if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")
          and v not in ("", "n/a")}
    for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]:
        print(f"  {v:6.3f} {k.split('stalled_')[1].split('_per')[0]}")
    rows = ncu_csv(rep, "--page", "source", "--print-source", "sass")
    hdr = rows[1]
    iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
    ops = collections.Counter()
    tot = 0
    for r in rows[2:]:
        try:
            n = int(r[iE])
        except (ValueError, IndexError):
            continue
        t = r[iS].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] += n
        tot += n
    print(f"warp instructions {tot}" + (f" = {tot / tokens:.2f} per token" if tokens else ""))
    for op, n in ops.most_common(22):
        print(f"  {op:10s} {n / tokens if tokens else n:8.3f}  {100 * n / tot:5.1f}%")


if __name__ == "__main__":
    main()
