"""Cost of the level-2 global smoothers (ILU(1), HBGS(3)) on the C2 solve:
iterations and solve time for several partition counts (diagnostics)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1904_05960_b200 import amg, krylov, mgr, problems, sparse  # noqa: E402

pb = problems.make_c2(seed=0, n=int(sys.argv[1]) if len(sys.argv) > 1 else 32)
A = sparse.DeviceCsr.from_arrays(pb.n, pb.n, torch.from_numpy(pb.row_offsets).cuda(),
                                 torch.from_numpy(pb.col_indices).cuda(), torch.from_numpy(pb.values).cuda())
F = sparse.Field
b = torch.from_numpy(pb.rhs).cuda()
for sm, parts in [("none", 1), ("ilu", 1), ("ilu", 256), ("ilu", 4096), ("hbgs", 256), ("hbgs", 4096)]:
    lv2 = mgr.MgrLevelSpec({F.S}, {F.P}, f_relax="jacobi", global_smoother=sm)
    cfg = mgr.MgrConfig(levels=(mgr.MgrLevelSpec({F.U}, {F.S, F.P}, f_relax="amg", n_max=4), lv2),
                        npartitions=parts,
                        amg_f_relax=amg.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=10 ** 9),
                        amg_terminal=amg.AmgConfig(strength_threshold=0.25, npartitions=10 ** 9))
    lay = sparse.FieldLayout(pb.field_of, pb.entity_of, sparse.Ordering.FLOW_INTERLEAVED)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = mgr.mgr_setup(A, lay, cfg)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    gc = krylov.GmresConfig(restart=100, max_iters=1000, rtol=1e-6)
    krylov.gmres(A, h.apply, b, cfg=gc)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    x, st = krylov.gmres(A, h.apply, b, cfg=gc)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{sm:5s} parts={parts:5d} setup {t1 - t0:7.3f}s  its {st.iterations:4d}  solve {1e3 * (t3 - t2):8.2f} ms",
          flush=True)
