"""Column-window statistics of the large AMG level operators: for slices of
32 consecutive rows, the number of distinct columns, the contiguous column
segments (gaps <= GAP merged) and the staged window size.
usage: python tools/window_stats.py C4 [n]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1904_05960_b200 import mgr, problems, sparse  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C4"
kw = {"n": int(sys.argv[2])} if len(sys.argv) > 2 else {}
pb = problems.make(cfgname, device=True, **kw)
h = mgr.mgr_setup(pb.A, sparse.FieldLayout(pb.field_of, pb.entity_of),
                  mgr.config_from_options(problems.solver_options(cfgname, pb)))
a = h.amg(0)
print("amg sizes", a.level_sizes())


def stats(name, ro, ci, rows_per=32, gap=8):
    n = len(ro) - 1
    ns = min((n + rows_per - 1) // rows_per, 4000)
    pick = np.linspace(0, (n + rows_per - 1) // rows_per - 1, ns).astype(np.int64)
    uni, seg, win, ent, dmax = [], [], [], [], []
    for s in pick:
        r0, r1 = s * rows_per, min(n, (s + 1) * rows_per)
        c = np.unique(ci[ro[r0]:ro[r1]])
        if len(c) == 0:
            continue
        d = np.diff(c)
        brk = d > gap
        seg.append(int(brk.sum()) + 1)
        uni.append(len(c))
        win.append(int(c[-1] - c[0] + 1 - (d[brk] - 1).sum()))
        ent.append(int(ro[r1] - ro[r0]))
        # largest in-row column delta
        m = 0
        for r in range(r0, r1):
            cc = ci[ro[r]:ro[r + 1]]
            if len(cc) > 1:
                m = max(m, int(np.diff(cc).max()))
        dmax.append(m)
    q = lambda x: (int(np.mean(x)), int(np.percentile(x, 50)), int(np.percentile(x, 99)), int(np.max(x)))
    print(f"{name}: rows {n} entries/slice {q(ent)} distinct cols {q(uni)} segments {q(seg)} window {q(win)} "
          f"max in-row delta {q(dmax)}   (mean, p50, p99, max)")


for l, lv in enumerate(a.levels[:4]):
    A = lv.A
    ro, ci = np.asarray(A.row_offsets), np.asarray(A.col_indices)
    if l >= 1:
        for gap in (0, 8, 32):
            stats(f"A_{l} gap{gap}", ro, ci, gap=gap)
    P = lv.P
    stats(f"P_{l}", np.asarray(P.row_offsets), np.asarray(P.col_indices))
L0 = h.levels[0]
for nm in ("P",):
    M = getattr(L0, nm)
    stats(f"mgr0.{nm}", np.asarray(M.row_offsets), np.asarray(M.col_indices))
