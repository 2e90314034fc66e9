"""Break down the e2e (host-buffer) solve overhead against the device-vector
solve at C2 (run under gpurun): python tools/e2e_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1904_05960_b200 import amg, krylov, mgr, sparse  # noqa: E402

pb, levels = bench.workload("C2", 0)
F = sparse.Field
specs = tuple(mgr.MgrLevelSpec({F(t) for t in f}, {F(t) for t in c}, f_relax=r, n_max=nm) for r, f, c, nm in levels)
cfg = mgr.MgrConfig(levels=specs,
                    amg_f_relax=amg.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=10 ** 9),
                    amg_terminal=amg.AmgConfig(strength_threshold=0.25, npartitions=10 ** 9))
A = sparse.DeviceCsr.from_arrays(pb.n, pb.n, torch.from_numpy(pb.row_offsets).cuda(),
                                 torch.from_numpy(pb.col_indices).cuda(), torch.from_numpy(pb.values).cuda())
h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of), cfg)
g = krylov.GmresConfig(restart=100, max_iters=1000, rtol=1e-6)
bd = torch.from_numpy(pb.rhs).cuda()
bp = torch.from_numpy(pb.rhs.copy()).pin_memory().numpy()
bq = pb.rhs.copy()


def tm(f, k=6):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


print("device b  (wall ms)", tm(lambda: krylov.gmres(A, h.apply, bd, cfg=g)))
print("pinned b  (wall ms)", tm(lambda: krylov.gmres(A, h.apply, bp, cfg=g)))
print("pageable b(wall ms)", tm(lambda: krylov.gmres(A, h.apply, bq, cfg=g)))
n = pb.n
print("np.zeros+any   us", 1e3 * tm(lambda: np.any(np.zeros(n)), 20) / 1)
print("np.empty+fill  us", 1e3 * tm(lambda: np.empty(n).fill(1.0), 20))
xd = torch.empty(n, dtype=torch.float64, device="cuda")
xs = torch.empty(n, dtype=torch.float64).pin_memory()
print("D2H pinned     us", 1e3 * tm(lambda: xs.copy_(xd), 20))
print("D2H pageable   us", 1e3 * tm(lambda: xd.cpu(), 20))
