"""Fit per-pass kernel time against the pass's shape (tools/pass_fit.sh output).

    python tools/pass_fit.py gpurun_out/pass_fit.csv gpurun_out/plan_dbg.log
"""
import csv
import re
import sys
from collections import defaultdict

import numpy as np

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
by = defaultdict(dict)
for r in data:
    by[int(r[ix["ID"]])][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
ids = sorted(by)
# final passes as plan_passes prints them at SVB_PLAN_DEBUG=3
plan = [ln for ln in open(sys.argv[2]) if ln.startswith("pass:") and "| banks:" in ln]
X, Y = [], []
for i, ln in zip(ids, plan):
    g, gr, c0, c1 = map(int, re.match(r"pass: (\d+) gates, (\d+) groups, (?:\d+ targets, )?coalesced (\d) (\d)", ln).groups())
    conf = sum(int(w) - 1 for w in re.findall(r" (?:ld|st) (\d)", ln) if int(w) > 0)
    d = by[i]
    X.append((g, gr, 1 - c1 + conf))
    Y.append((d["gpu__time_duration.sum"] / 1e3, d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"],
              d["l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"] / 1e6))
X, Y = np.array(X, float), np.array(Y)
t = Y[:, 0]
coef = np.linalg.lstsq(np.c_[np.ones(len(X)), X], t, rcond=None)[0]
print(f"{len(t)} passes: mean {t.mean():.1f} us  min {t.min():.1f}  max {t.max():.1f}  sum {t.sum() / 1e3:.1f} ms")
print("fit t = %.1f + %.2f*gates + %.1f*groups + %.1f*(uncoalesced last store + bank-conflict phases) (us)" % tuple(coef))
print(f"fp64 pipe mean {Y[:, 1].mean():.1f}%  smem bank conflicts mean {Y[:, 2].mean():.2f} M/pass")
