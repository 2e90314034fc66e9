"""Print the solve operators of a config's MGR hierarchy (rows, nnz, row
lengths) as setup finalises them: python tools/hier_stats.py C4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PMGR_HIER_STATS"] = "1"
from paper_1904_05960_b200 import mgr, problems, sparse  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
dev = cfgname not in ("C1", "C2")
pb = problems.make(cfgname, device=dev)
A = pb.A if dev else sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of),
                  mgr.config_from_options(problems.solver_options(cfgname, pb)))
print("levels", h.level_sizes(), file=sys.stderr)
for l in range(len(h.level_sizes()) - 1):
    a = h.amg(l)
    if a is not None:
        print("mgr level", l, "amg", a.level_sizes(), file=sys.stderr)
print("terminal", h.terminal_solver.level_sizes(), file=sys.stderr)
print("apply bytes / kernels", h.apply_bytes(), file=sys.stderr)
