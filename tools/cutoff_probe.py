"""C4 solve under the production configuration with a different
coarse_size_cutoff of the F-relaxation AMG (a reference AmgConfig option):
iterations, solve time, apply time, setup time.
    python tools/cutoff_probe.py C4 10000"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_05960_b200 import krylov, mgr, problems, sparse  # noqa: E402

name = sys.argv[1]
cut = int(sys.argv[2])
pb = problems.make(name, device=True)
opts = problems.solver_options(name, pb)
if cut > 0:
    opts["amg_f_relax"]["coarse_size_cutoff"] = cut
cfg = mgr.config_from_options(opts)
lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
for rep in range(2):
    torch.cuda.synchronize()
    t = time.time()
    h = mgr.mgr_setup(pb.A, lay, cfg)
    torch.cuda.synchronize()
    ts = time.time() - t
    if rep == 0:
        del h
print("cutoff", cut, "setup", round(ts, 3), "amg0", h.amg(0).level_sizes(), flush=True)
b = torch.from_numpy(pb.rhs).cuda()
gcfg = krylov.GmresConfig(restart=opts["restart"], max_iters=opts["max_iters"], rtol=opts["rtol"])
for rep in range(2):
    torch.cuda.synchronize()
    t = time.time()
    x, st = krylov.gmres(pb.A, h.apply, b, cfg=gcfg)
    torch.cuda.synchronize()
    tt = time.time() - t
print("cutoff", cut, "iterations", st.iterations, st.converged, "solve", round(tt, 3), "s", flush=True)
v = torch.randn(pb.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    h.apply(v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    h.apply(v)
e1.record()
torch.cuda.synchronize()
print("cutoff", cut, "apply ms", round(e0.elapsed_time(e1) / 10, 3), flush=True)
