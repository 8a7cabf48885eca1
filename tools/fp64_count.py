"""Static FP64 instruction count of the generated passes of a circuit
(per thread per tile, summed over passes) and the share spent applying
phases -- a CPU-only proxy for the specialised passes' FP64 work.

    python tools/fp64_count.py DUMP_DIR
"""
import glob
import os
import re
import sys


def count(path):
    src = open(path).read()
    body = src[src.index('extern "C"'):]
    tot = app = 0
    for line in body.split("\n"):
        n = line.count("__fma_rn") + line.count("__dmul_rn") + line.count("__dadd_rn") + line.count("__dsub_rn")
        n += 4 * len(re.findall(r"\bcm\(", line)) + 8 * len(re.findall(r"\brow\(", line))
        n += 4 * len(re.findall(r"\brrow\(", line)) + 4 * len(re.findall(r"\brirow\(", line))
        tot += n
        if "X = v[" in line:
            app += n
    return tot, app


d = sys.argv[1]
files = sorted(glob.glob(os.path.join(d, "pass*.cu")), key=lambda f: int(re.findall(r"\d+", os.path.basename(f))[0]))
T = A = 0
for f in files:
    t, a = count(f)
    T += t
    A += a
print(f"{len(files)} passes, FP64 per thread-tile summed {T}, phase applications {A} ({A / max(T, 1):.3f})")
