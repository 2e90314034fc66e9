"""Time mgr_setup phase by phase (PMGR_SETUP_TRACE=1) on a BASELINE config."""
import os, sys, time
os.environ.setdefault("PMGR_SETUP_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1904_05960_b200 import sparse, amg, mgr, problems
F = sparse.Field
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
pb = problems.make(name)
if len(pb.cell_fields) == 3:
    lv = (mgr.MgrLevelSpec({F.U}, {F.S, F.S2, F.P}, f_relax="amg", n_max=4), mgr.MgrLevelSpec({F.S2}, {F.S, F.P}), mgr.MgrLevelSpec({F.S}, {F.P}))
elif pb.cell_fields == (2,):
    lv = (mgr.MgrLevelSpec({F.U}, {F.P}, f_relax="amg"),)
else:
    lv = (mgr.MgrLevelSpec({F.U}, {F.S, F.P}, f_relax="amg", n_max=4), mgr.MgrLevelSpec({F.S}, {F.P}))
cfg = mgr.MgrConfig(levels=lv, amg_f_relax=amg.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=10**9),
                    amg_terminal=amg.AmgConfig(strength_threshold=0.25, npartitions=10**9))
A = sparse.DeviceCsr.from_arrays(pb.n, pb.n, torch.from_numpy(pb.row_offsets).cuda(), torch.from_numpy(pb.col_indices).cuda(), torch.from_numpy(pb.values).cuda())
lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
for rep in range(2):
    torch.cuda.synchronize(); t = time.time()
    h = mgr.mgr_setup(A, lay, cfg)
    torch.cuda.synchronize()
    print(f"=== setup {rep}: {time.time()-t:.3f} s levels {h.level_sizes()}", file=sys.stderr, flush=True)
    del h
