"""Time mgr_setup phase by phase (PMGR_SETUP_TRACE=1) on a BASELINE config
under its production solver configuration: python tools/setup_trace.py C4"""
import os
import sys
import time

os.environ.setdefault("PMGR_SETUP_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_05960_b200 import mgr, problems, sparse  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
dev = name not in ("C1", "C2")
pb = problems.make(name, device=dev)
A = pb.A if dev else sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
cfg = mgr.config_from_options(problems.solver_options(name, pb))
lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
for rep in range(int(os.environ.get("SETUP_REPS", "3"))):
    torch.cuda.synchronize()
    t = time.time()
    h = mgr.mgr_setup(A, lay, cfg)
    torch.cuda.synchronize()
    print(f"=== setup {rep}: {time.time() - t:.3f} s levels {h.level_sizes()}", file=sys.stderr, flush=True)
    del h
