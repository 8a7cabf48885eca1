"""Experiment: global-memory addressing of a specialised pass with base +
constant offsets instead of a per-access XOR (thread bits and per-register
constants never share address bits, so x ^ c == x + c).

    python tools/addr_patch.py pass.cu out.cu
"""
import re
import sys


def bits_of_xor_updates(lines, var):
    m = 0
    for ln in lines:
        for c in re.findall(rf"\b{var} \^= (\d+)u;", ln):
            m |= int(c)
        mm = re.match(rf"unsigned {var} = (\d+)u", ln)
        if mm:
            m |= int(mm.group(1))
        if re.match(rf"unsigned {var} = tg & (\d+)", ln):
            m |= int(re.match(rf"unsigned {var} = tg & (\d+)", ln).group(1))
    return m


def patch(src):
    lines = src.split("\n")
    out = []
    i = 0
    # fill lambda: r built from tg bits
    fill_start = next(k for k, ln in enumerate(lines) if ln.startswith("auto fill = "))
    fill_end = next(k for k in range(fill_start, len(lines)) if "cp.async.commit_group" in lines[k] or lines[k].startswith("};"))
    rbits = bits_of_xor_updates(lines[fill_start:fill_end], "r") | 7
    cbits = 0
    for ln in lines[fill_start:fill_end]:
        for c in re.findall(r"p \+ \(r \^ (\d+)u\)", ln):
            cbits |= int(c)
    assert rbits & cbits == 0, (rbits, cbits)
    first_cpa = True
    for k, ln in enumerate(lines):
        if fill_start <= k < fill_end and "p + (r ^ " in ln:
            if first_cpa:
                out.append("const d2 *const pr = p + r;")
                first_cpa = False
            ln = re.sub(r"p \+ \(r \^ (\d+)u\)", r"pr + \1u", ln)
        out.append(ln)
    lines = out
    out = []
    # direct stores of the last group
    k = 0
    while k < len(lines):
        ln = lines[k]
        if ln.startswith("unsigned s0 ="):
            e = next(j for j in range(k, len(lines)) if lines[j].startswith("stcs("))
            e2 = e
            while e2 < len(lines) and lines[e2].startswith("stcs("):
                e2 += 1
            sbits = bits_of_xor_updates(lines[k:e], "s0")
            cb = 0
            for l2 in lines[e:e2]:
                cb |= int(re.search(r"s0 \^ (\d+)u", l2).group(1))
            if sbits & cb == 0:
                out.extend(lines[k:e])
                out.append("d2 *const ps = pa + s0;")
                for l2 in lines[e:e2]:
                    out.append(re.sub(r"pa \+ \(s0 \^ (\d+)u\)", r"ps + \1u", l2))
                k = e2
                continue
        out.append(ln)
        k += 1
    return "\n".join(out)


if __name__ == "__main__":
    open(sys.argv[2], "w").write(patch(open(sys.argv[1]).read()))


def patch_smem(src):
    """sb + (x0 ^ C) -> sb + ((x0 ^ (C & M)) + K): M = the bits the thread-varying
    terms of x0 can set; the other bits of the address are the constant
    K = (B ^ C) & ~M (B = x0's constant start), an immediate offset."""
    lines = src.split("\n")
    out = []
    k = 0
    while k < len(lines):
        m = re.match(r"unsigned ([ab]0) = (\d+)u;", lines[k])
        if not m:
            out.append(lines[k])
            k += 1
            continue
        var, B = m.group(1), int(m.group(2))
        # header: up to the first access
        acc = re.compile(r"sb \+ \(" + var + r" \^ (\d+)u\)")
        e = k + 1
        while not acc.search(lines[e]):
            e += 1
        e2 = e
        while e2 < len(lines) and acc.search(lines[e2]):
            e2 += 1
        M = 0
        for ln in lines[k + 1:e]:
            for c in re.findall(var + r" \^= (\d+)u;", ln):
                M |= int(c)
        out.append(f"unsigned {var} = {B & M}u;")
        out.extend(lines[k + 1:e])
        pats = {}
        body = []
        for ln in lines[k + 0:0]:
            pass
        for ln in lines[e:e2]:
            C = int(acc.search(ln).group(1))
            L, K = C & M, (B ^ C) & ~M
            if L not in pats:
                pats[L] = f"{var}_{len(pats)}"
            body.append(acc.sub(f"sb + ({pats[L]} + {K}u)", ln))
        for L, name in pats.items():
            out.append(f"const unsigned {name} = {var} ^ {L}u;")
        out.extend(body)
        k = e2
    return "\n".join(out)


if __name__ == "__main__" and len(sys.argv) > 3 and sys.argv[3] == "smem":
    open(sys.argv[2], "w").write(patch_smem(patch(open(sys.argv[1]).read())))
