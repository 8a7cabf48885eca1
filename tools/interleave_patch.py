"""Experiment: in the last register group of a mode-2 pass source, issue each
direct HBM store right after the last statement that writes its register
(instead of all 32 stores after all gates), so the store queue drains under
the remaining FP64 work.

    python tools/interleave_patch.py pass.cu out.cu
"""
import re
import sys


def patch(src):
    lines = src.split("\n")
    gstarts = [i for i, ln in enumerate(lines) if re.match(r"\{ // group \d+", ln)]
    s = gstarts[-1]
    g0 = next(i for i in range(s, len(lines)) if lines[i].startswith("d2 ph = mk("))
    pre = next(i for i in range(g0, len(lines)) if lines[i].startswith("unsigned s0 =") or lines[i].startswith("i64 s0 ="))
    st0 = next(i for i in range(pre, len(lines)) if lines[i].startswith("stcs("))
    st1 = st0
    while lines[st1].startswith("stcs("):
        st1 += 1
    preamble = lines[pre:st0]
    stores = {int(re.search(r"v\[(\d+)\]\);", ln).group(1)): ln for ln in lines[st0:st1]}
    gates = lines[g0:pre]
    # top-level statements of the gate section
    stmts = []
    depth = 0
    cur = []
    for ln in gates:
        cur.append(ln)
        depth += ln.count("{") - ln.count("}")
        if depth == 0:
            stmts.append(cur)
            cur = []
    assert not cur
    last = {}
    for k, st in enumerate(stmts):
        for ln in st:
            for r in re.findall(r"v\[(\d+)\] =", ln):
                last[int(r)] = k
    out = lines[:g0] + preamble
    pending = sorted(stores)
    for r in pending:
        if r not in last:
            out.append(stores[r])  # never written in this group: store at once
    for k, st in enumerate(stmts):
        out.extend(st)
        for r in pending:
            if last.get(r) == k:
                out.append(stores[r])
    out += lines[st1:]
    return "\n".join(out)


if __name__ == "__main__":
    open(sys.argv[2], "w").write(patch(open(sys.argv[1]).read()))


def spread_prefetch(src):
    """Also spread the next tile's 32 cp.async over the last group's gate
    statements (they are issued in one burst after the barrier otherwise)."""
    lines = src.split("\n")
    f0 = next(i for i, ln in enumerate(lines) if ln.startswith("auto fill = "))
    f1 = next(i for i in range(f0, len(lines)) if "cp.async.commit_group" in lines[i])
    body = lines[f0 + 1:f1]
    setup = [ln for ln in body if not ln.startswith("cpa(")]
    cpas = [ln for ln in body if ln.startswith("cpa(")]
    gstarts = [i for i, ln in enumerate(lines) if re.match(r"\{ // group \d+", ln)]
    s = gstarts[-1]
    call = next(i for i in range(s, len(lines)) if "fill(reinterpret_cast<unsigned char *>(dsm), a + tbase(nx))" in lines[i])
    g0 = next(i for i in range(call, len(lines)) if lines[i].startswith("d2 ph = mk("))
    out = lines[:call]
    out.append("const i64 nx = tix + gridDim.x; const bool pf = nx < ntiles;")
    out.append("unsigned char *const dstb = reinterpret_cast<unsigned char *>(dsm); const d2 *const p = a + tbase(pf ? nx : tix);")
    # the fill's per-thread parts (r, s, pr) in their own names
    ren = lambda ln: re.sub(r"\bpr\b", "fpr_", re.sub(r"\bs\b", "fs_", re.sub(r"(?<!\")\br\b(?!\")", "fr_", re.sub(r"\btg\b", "ftg_", ln))))
    out.extend(ren(ln) for ln in setup)
    cpas = [ren(ln) for ln in cpas]
    out.extend(lines[call + 1:g0])
    region = lines[g0:]
    # top-level statements until the group's closing brace
    stmts, cur, depth, k = [], [], 0, 0
    while True:
        ln = region[k]
        if depth == 0 and ln == "}":
            break
        cur.append(ln)
        depth += ln.count("{") - ln.count("}")
        if depth == 0:
            stmts.append(cur)
            cur = []
        k += 1
    n = len(stmts)
    per = max(1, n // (len(cpas) + 1))
    ci = 0
    for j, st in enumerate(stmts):
        out.extend(st)
        if ci < len(cpas) and j % per == per - 1 and not st[0].startswith("d2 ") :
            out.append("if (pf) " + cpas[ci])
            ci += 1
    while ci < len(cpas):
        out.append("if (pf) " + cpas[ci])
        ci += 1
    out.append('asm volatile("cp.async.commit_group;\\n" ::: "memory");')
    out.extend(region[k:])
    return "\n".join(out)


if __name__ == "__main__" and len(sys.argv) > 3 and sys.argv[3] == "spread":
    open(sys.argv[2], "w").write(spread_prefetch(patch(open(sys.argv[1]).read())))
