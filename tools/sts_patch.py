"""Experiment: in every register group that stores to shared memory, move the
store-hazard barrier up to just after the group's loads and issue each
shared-memory store right after the last statement that writes its register,
so the store phase overlaps the group's remaining FP64 work.

    python tools/sts_patch.py pass.cu out.cu
"""
import re
import sys


def top_level(stmts_lines):
    stmts, cur, depth = [], [], 0
    for ln in stmts_lines:
        cur.append(ln)
        depth += ln.count("{") - ln.count("}")
        if depth == 0:
            stmts.append(cur)
            cur = []
    assert not cur
    return stmts


def patch(src):
    lines = src.split("\n")
    gstarts = [i for i, ln in enumerate(lines) if re.match(r"\{ // group \d+", ln)]
    out = lines[:gstarts[0]]
    for gi, s in enumerate(gstarts):
        e = gstarts[gi + 1] if gi + 1 < len(gstarts) else len(lines)
        blk = lines[s:e]
        b0i = next((i for i, ln in enumerate(blk) if ln.startswith("unsigned b0 =")), None)
        if b0i is None:
            out.extend(blk)
            continue
        g0 = next(i for i, ln in enumerate(blk) if ln.startswith("d2 ph = mk("))
        bar = None
        pre_start = b0i
        if blk[b0i - 1].startswith("__syncthreads();") or blk[b0i - 1].startswith("__syncwarp();"):
            bar = blk[b0i - 1]
            pre_start = b0i - 1
        st0 = next(i for i in range(b0i, len(blk)) if blk[i].startswith("*reinterpret_cast<d2 *>(sb +"))
        st1 = st0
        while blk[st1].startswith("*reinterpret_cast<d2 *>(sb +"):
            st1 += 1
        preamble = blk[b0i:st0]
        stores = {int(re.search(r"= v\[(\d+)\];", ln).group(1)): ln for ln in blk[st0:st1]}
        stmts = top_level(blk[g0:pre_start])
        last = {}
        for k, st in enumerate(stmts):
            for ln in st:
                for r in re.findall(r"v\[(\d+)\] =", ln):
                    last[int(r)] = k
        out.extend(blk[:g0])
        if bar:
            out.append(bar)
        out.extend(preamble)
        for r in sorted(stores):
            if r not in last:
                out.append(stores[r])
        for k, st in enumerate(stmts):
            out.extend(st)
            for r in sorted(stores):
                if last.get(r) == k:
                    out.append(stores[r])
        out.extend(blk[st1:])
    return "\n".join(out)


if __name__ == "__main__":
    open(sys.argv[2], "w").write(patch(open(sys.argv[1]).read()))
