"""Summarise an ncu report: key SOL metrics, stall reasons, SASS opcode mix.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [launch_id]
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def ncu(*args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    lid = sys.argv[2] if len(sys.argv) > 2 else "0"
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    h = rows[0]
    ki, si, mi, vi, ui = (h.index(x) for x in ("ID", "Section Name", "Metric Name", "Metric Value", "Metric Unit"))
    keep = {"Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
            "Warp Cycles Per Issued Instruction", "Registers Per Thread", "Achieved Occupancy",
            "Executed Instructions", "L1/TEX Cache Throughput", "L2 Cache Throughput"}
    for r in rows[1:]:
        if r[ki] == lid and r[mi] in keep:
            print(f"{r[mi]:40s} {r[vi]} {r[ui]}")
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, row = raw[0], raw[2 + int(lid)]
    stalls = {}
    for i, name in enumerate(h):
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(row[i].replace(",", ""))
            except ValueError:
                pass
        if name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"):
            print(f"{name:40s} {row[i]} {raw[1][i]}")
    tot = sum(stalls.values()) or 1
    print("stalls:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:9]))
    sass = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hh = sass[1]
    si, st, ie = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
    c, cs = Counter(), Counter()
    ti = ts = 0
    for r in sass[2:]:
        try:
            i, s = int(r[ie] or 0), int(r[st] or 0)
        except (ValueError, IndexError):
            continue
        toks = r[si].split()
        if not toks:
            continue
        op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
        c[op] += i
        cs[op] += s
        ti += i
        ts += s
    print("opcodes:", ", ".join(f"{op} {v / ti * 100:.1f}%/{cs[op] / max(ts, 1) * 100:.1f}%" for op, v in c.most_common(14)))


if __name__ == "__main__":
    main()
