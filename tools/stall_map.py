"""Per-instruction stall sampling of an ncu report (source page, SASS):
samples by opcode, by reason, and a coarse timeline (instruction index
buckets) so the stalled phases of a pass kernel show up.

    python tools/stall_map.py report.ncu-rep [buckets]
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict


def main():
    rep = sys.argv[1]
    nb = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    idx = {c: i for i, c in enumerate(h)}
    reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    ins = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        src = r[idx["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        samp = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        rs = {c: int(r[idx[c]] or 0) for c in reasons}
        ins.append((op, samp, rs, src))
    tot = sum(s for _, s, _, _ in ins)
    by_op = Counter()
    by_reason = Counter()
    op_reason = defaultdict(Counter)
    for op, s, rs, _ in ins:
        by_op[op] += s
        for c, v in rs.items():
            by_reason[c] += v
            op_reason[op][c] += v
    print(f"{len(ins)} instructions, {tot} samples")
    print("by opcode (samples at the instruction = the warp is stalled BEFORE issuing it):")
    for op, s in by_op.most_common(14):
        top = ", ".join(f"{c[6:]} {100 * v / max(s, 1):.0f}%" for c, v in op_reason[op].most_common(3))
        print(f"  {op:8s} {100 * s / tot:5.1f}%   ({top})")
    print("by reason:", ", ".join(f"{c[6:]} {100 * v / tot:.1f}%" for c, v in by_reason.most_common(10)))
    print("timeline (instruction index buckets): share of samples / dominant opcode")
    step = max(1, len(ins) // nb)
    for b in range(0, len(ins), step):
        seg = ins[b:b + step]
        s = sum(x[1] for x in seg)
        ops = Counter()
        for x in seg:
            ops[x[0]] += 1
        rsn = Counter()
        for x in seg:
            rsn.update(x[2])
        print(f"  [{b:5d}-{b + len(seg) - 1:5d}] {100 * s / tot:5.1f}%  ops {dict(ops.most_common(3))}  "
              f"stall {', '.join(f'{c[6:]} {100 * v / max(s, 1):.0f}%' for c, v in rsn.most_common(2))}")


if __name__ == "__main__":
    main()
