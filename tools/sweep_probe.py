"""Level-0 sweep and MGR-apply timing of a config (diagnostics for kernel
A/B runs; variants through PMGR_* environment variables, one process each):
    PMGR_BSR_TPW=1 python tools/sweep_probe.py C4"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_05960_b200 import _lib, mgr, problems, sparse  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
pb = problems.make(name, device=True)
h = mgr.mgr_setup(pb.A, sparse.FieldLayout(pb.field_of, pb.entity_of),
                  mgr.config_from_options(problems.solver_options(name, pb)))
v = torch.randn(pb.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    h.apply(v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    h.apply(v)
e1.record()
torch.cuda.synchronize()
apply_ms = e0.elapsed_time(e1) / reps
L = _lib.lib()
L.pmgr_prof_enable(1)
for _ in range(reps):
    h.apply(v)
torch.cuda.synchronize()
out = {"apply_ms": apply_ms, "env": {k: v for k, v in os.environ.items() if k.startswith("PMGR_")}}
for kind, nm in ((1, "sweep0_residual"), (2, "post_sweep")):
    c, ms, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    L.pmgr_prof_query(kind, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(by))
    if c.value:
        out[nm + "_us"] = ms.value * 1e3 / c.value
        out[nm + "_gbs"] = by.value / (ms.value / 1e3) / 1e9
L.pmgr_prof_enable(0)
print(json.dumps(out), flush=True)
