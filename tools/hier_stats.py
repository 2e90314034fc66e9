"""Print the solve operators of a config's MGR hierarchy (rows, nnz, row
lengths) as setup finalises them: PMGR_HIER_STATS=1 python tools/hier_stats.py C4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PMGR_HIER_STATS"] = "1"
import bench  # noqa: E402
from paper_1904_05960_b200 import amg, mgr, sparse  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
pb, levels = bench.workload(cfgname, 0, device=cfgname not in ("C1", "C2"))
F = sparse.Field
specs = tuple(mgr.MgrLevelSpec({F(t) for t in f}, {F(t) for t in c}, f_relax=r, n_max=nm) for r, f, c, nm in levels)
cfg = mgr.MgrConfig(levels=specs,
                    amg_f_relax=amg.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=10 ** 9),
                    amg_terminal=amg.AmgConfig(strength_threshold=0.25, npartitions=10 ** 9))
A = pb.A if cfgname not in ("C1", "C2") else sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of), cfg)
print("levels", h.level_sizes(), file=sys.stderr)
for l in range(len(h.level_sizes()) - 1):
    a = h.amg(l)
    if a is not None:
        print("mgr level", l, "amg", a.level_sizes(), file=sys.stderr)
print("terminal", h.terminal_solver.level_sizes(), file=sys.stderr)
