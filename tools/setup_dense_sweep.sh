for d in 12288 6144 3072 1024; do
  for c in C2 C4; do
    PMGR_SETUP_TRACE=0 PMGR_DENSE_COLS=$d python - <<PY 2>/dev/null
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1904_05960_b200 import sparse, amg, mgr, problems
F = sparse.Field
pb = problems.make("$c", n=32 if "$c"=="C4" else 32)
if len(pb.cell_fields) == 3:
    lv = (mgr.MgrLevelSpec({F.U}, {F.S, F.S2, F.P}, f_relax="amg", n_max=4), mgr.MgrLevelSpec({F.S2}, {F.S, F.P}), mgr.MgrLevelSpec({F.S}, {F.P}))
else:
    lv = (mgr.MgrLevelSpec({F.U}, {F.S, F.P}, f_relax="amg", n_max=4), mgr.MgrLevelSpec({F.S}, {F.P}))
cfg = mgr.MgrConfig(levels=lv, amg_f_relax=amg.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=10**9), amg_terminal=amg.AmgConfig(strength_threshold=0.25, npartitions=10**9))
A = sparse.DeviceCsr.from_arrays(pb.n, pb.n, torch.from_numpy(pb.row_offsets).cuda(), torch.from_numpy(pb.col_indices).cuda(), torch.from_numpy(pb.values).cuda())
lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
best = 1e9
for rep in range(3):
    torch.cuda.synchronize(); t = time.time()
    h = mgr.mgr_setup(A, lay, cfg)
    torch.cuda.synchronize(); best = min(best, time.time() - t)
    del h
print("$d $c", round(best, 4))
PY
  done
done
