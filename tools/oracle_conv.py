"""Oracle convergence at a given size (diagnostics): the CPU restatement's
GMRES iteration count for a config, to set beside tools/conv_probe2.py's GPU
count (same seeded problem, same preconditioner options)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402
from paper_1904_05960_b200 import problems  # noqa: E402


def levels_for(pb, nmax=4, fs=1, gs="none"):
    nf = len(pb.cell_fields)
    if nf == 1:
        return (O.MgrLevelSpec(frozenset({0}), frozenset({2}), "amg", fs, None),)
    if nf == 3:
        return (O.MgrLevelSpec(frozenset({0}), frozenset({1, 3, 2}), "amg", fs, nmax),
                O.MgrLevelSpec(frozenset({3}), frozenset({1, 2}), "jacobi", 1, None, global_smoother=gs),
                O.MgrLevelSpec(frozenset({1}), frozenset({2}), "jacobi", 1, None))
    return (O.MgrLevelSpec(frozenset({0}), frozenset({1, 2}), "amg", fs, nmax),
            O.MgrLevelSpec(frozenset({1}), frozenset({2}), "jacobi", 1, None, global_smoother=gs))


def main():
    name, n = sys.argv[1], int(sys.argv[2])
    gsk = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    max_iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3000
    O.build()
    pb = problems.make(name, n=n)
    pf = 10 ** 9 if not gsk else max(1, pb.n_u // gsk)
    pt = 10 ** 9 if not gsk else max(1, (pb.n - pb.n_u) // len(pb.cell_fields) // gsk)
    cfg = O.MgrConfig(levels=levels_for(pb),
                      amg_f_relax=O.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=pf),
                      amg_terminal=O.AmgConfig(strength_threshold=0.25, npartitions=pt))
    A = O.Csr(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    t0 = time.perf_counter()
    h = O.mgr_setup(A, pb.field_of, pb.entity_of, cfg)
    t1 = time.perf_counter()
    x, its, hist, conv = O.gmres(lambda v: O.spmv(A, v), h.apply, pb.rhs, restart=100, max_iters=max_iters)
    t2 = time.perf_counter()
    marks = {int(k): float(hist[k] / hist[0]) for k in range(0, len(hist), 100)}
    print(json.dumps(dict(cfg=name, n=n, gs=gsk, dofs=pb.n, its=int(its), conv=bool(conv),
                          rel=float(hist[-1] / hist[0]), setup_s=round(t1 - t0, 2), solve_s=round(t2 - t1, 2),
                          levels=h.level_sizes(), hist=marks)), flush=True)


if __name__ == "__main__":
    main()
