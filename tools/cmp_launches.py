"""Compare per-launch kernel times of two ncu launch lists (same kernels in
the same order): python tools/cmp_launches.py a.csv b.csv"""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ii, mi, vi = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
    out = {}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        out.setdefault(int(r[ii]), {})[r[mi]] = float(r[vi].replace(",", ""))
    return [out[k] for k in sorted(out)]


a, b = load(sys.argv[1]), load(sys.argv[2])
key = "gpu__time_duration.sum"
ta, tb = [x[key] for x in a], [x[key] for x in b]
print(f"launches {len(ta)} vs {len(tb)}; total {sum(ta) / 1e3:.2f} vs {sum(tb) / 1e3:.2f} us x1e3")
d = sorted(((y - x) / x, i, x, y) for i, (x, y) in enumerate(zip(ta, tb)))
print("most improved:", [(i, round(x / 1e3, 1), round(y / 1e3, 1)) for _, i, x, y in d[:8]])
print("most regressed:", [(i, round(x / 1e3, 1), round(y / 1e3, 1)) for _, i, x, y in d[-8:]])
for k in a[0]:
    if k != key:
        print(k, round(sum(x[k] for x in a) / len(a), 2), round(sum(x[k] for x in b) / len(b), 2))
