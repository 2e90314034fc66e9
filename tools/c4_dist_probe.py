"""Full-size C4 (128^3) through the DISTRIBUTED setup over emulated ranks on
one GPU (loopback transport): the application against the single-GPU
hierarchy's (bitwise at the default thresholds) and the distributed GMRES's
iteration count.  The only way to run the multi-rank setup at the headline
size on a one-GPU box.
    python tools/c4_dist_probe.py [nranks] [C4|C5 [slab]]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1904_05960_b200 import dist as D, krylov, mgr, problems, sparse  # noqa: E402

nranks = int(sys.argv[1]) if len(sys.argv) > 1 else 2
name = sys.argv[2] if len(sys.argv) > 2 else "C4"
if name == "C5":  # the weak-scaling stack: a 128^3 slab per rank
    ns = int(sys.argv[3]) if len(sys.argv) > 3 else 128
    base = problems.make_c5(seed=0, nxy=ns, nz_per_gpu=ns, gpus=nranks, device=True)
else:
    base = problems.make(name, device=True)
pb, bounds = problems.rank_major(base, nranks)
del base
opts = problems.solver_options(name, pb)
cfg = mgr.config_from_options(opts)
lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
h = mgr.mgr_setup(pb.A, lay, cfg)
v = torch.randn(pb.n, dtype=torch.float64, device="cuda")
z = h.apply(v)
torch.cuda.synchronize()
b = torch.from_numpy(pb.rhs).cuda()
gcfg = krylov.GmresConfig(restart=opts["restart"], max_iters=opts["max_iters"], rtol=opts["rtol"])
x1, st = krylov.gmres(pb.A, h.apply, b, cfg=gcfg)
del h  # the emulated ranks need the memory
from paper_1904_05960_b200 import _lib  # noqa: E402
_lib.release_cached_memory()
t = time.time()
zs = D.emulate_setup_apply(pb.A, lay, cfg, bounds, v)
torch.cuda.synchronize()
print(f"{name} over {nranks} emulated ranks: distributed setup + apply {time.time() - t:.1f} s; bitwise",
      bool(torch.equal(zs, z)), "max diff", float((zs - z).abs().max()), flush=True)
del zs
torch.cuda.synchronize()
t = time.time()
xd, its, conv = D.emulate_setup_gmres(pb.A, lay, cfg, bounds, b, gcfg)
torch.cuda.synchronize()
print(f"distributed setup + GMRES {time.time() - t:.1f} s: iterations {its} (single GPU {st.iterations}) converged {conv}; "
      f"solution rel diff {float((xd - x1).norm() / x1.norm()):.2e}", flush=True)
