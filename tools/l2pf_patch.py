"""Experiment: mode-0 pass source (first group loads its registers straight
from global memory, no tile fill through shared memory) + an L2 prefetch of
the CTA's next tile issued at the start of the current one (4
prefetch.global.L2 per thread: one per 128 B row).

    python tools/l2pf_patch.py mode0_pass.cu out.cu [ahead]
"""
import re
import sys


def patch(src, ahead=1):
    lines = src.split("\n")
    f0 = next(i for i, ln in enumerate(lines) if ln.startswith("auto fill = "))
    f1 = next(i for i in range(f0, len(lines)) if "cp.async.commit_group" in lines[i])
    body = lines[f0 + 1:f1]
    rterms = []  # (thread bit, offset) for thread bits >= 3
    for ln in body:
        m = re.match(r"if \(\(tg >> (\d+)\) & 1\) r \^= (\d+)u;", ln)
        if m:
            rterms.append((int(m.group(1)), int(m.group(2))))
    krow = [int(re.search(r"pr \+ (\d+)u\)", ln).group(1)) for ln in body if ln.startswith("cpa(")]
    assert len(krow) == 32
    basis = [krow[1], krow[2], krow[4], krow[8], krow[16]]
    for k in range(32):
        assert krow[k] == sum(basis[b] for b in range(5) if (k >> b) & 1), "k_row not additive"
    pf = ["{ const i64 nxp = tix + %d * (i64)gridDim.x; if (nxp < ntiles) {" % ahead,
          "unsigned tg = tid; asm volatile(\"\" : \"+r\"(tg));",
          "unsigned r = 0;"]
    for bit, off in rterms:
        pf.append(f"if ((tg >> {bit}) & 1) r += {off}u;")
    # k = 4 * (tg & 7) + j: bits 2..4 of k from tg's low three bits
    for b in range(3):
        pf.append(f"if ((tg >> {b}) & 1) r += {basis[2 + b]}u;")
    pf.append("const d2 *const q = a + tbase(nxp) + r;")
    for j in range(4):
        off = sum(basis[b] for b in range(2) if (j >> b) & 1)
        pf.append(f'asm volatile("prefetch.global.L2 [%0];" :: "l"(q + {off}u));')
    pf.append("} }")
    out = []
    for ln in lines:
        out.append(ln)
        if ln.startswith("d2 v[32];"):
            out.extend(pf)
    return "\n".join(out)


if __name__ == "__main__":
    ahead = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    open(sys.argv[2], "w").write(patch(open(sys.argv[1]).read(), ahead))
