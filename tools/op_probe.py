"""SpMV timing of single operators of a config's hierarchy (the F-relaxation
AMG's level operators, exported as their own matrices), one process per
kernel variant (PMGR_* environment):
    PMGR_SJ_D=2 python tools/op_probe.py C4"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_05960_b200 import _lib, mgr, problems, sparse  # noqa: E402
from paper_1904_05960_b200.amg import _export_dev  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
pb = problems.make(name, device=True)
h = mgr.mgr_setup(pb.A, sparse.FieldLayout(pb.field_of, pb.entity_of),
                  mgr.config_from_options(problems.solver_options(name, pb)))
a = h.amg(0)
L = _lib.lib()
out = {"env": {k: v for k, v in os.environ.items() if k.startswith("PMGR_")}}
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
for lvl, what, tag in ((1, 0, "A1"), (2, 0, "A2"), (3, 0, "A3"), (0, 1, "P0"), (1, 1, "P1")):
    M = _export_dev(a._h, lvl, what)
    x = torch.randn(M.ncols, dtype=torch.float64, device="cuda")
    y = torch.empty(M.nrows, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        _lib.check(L.pmgr_spmv(M.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(st)))
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.pmgr_spmv(M.handle, ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(st)))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    us = ts[len(ts) // 2]
    by = 12.0 * M.nnz + 8.0 * (M.nrows + 1) + 8.0 * M.ncols + 8.0 * M.nrows
    out[tag] = {"rows": M.nrows, "nnz": M.nnz, "us": round(us, 1), "csr_gbs": round(by / us / 1e3, 1)}
    del M
print(json.dumps(out), flush=True)
