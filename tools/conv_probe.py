import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_1904_05960_b200 import sparse, amg, mgr, krylov, problems
F = sparse.Field
def cfgfor(pb):
    if pb.cell_fields == (2,):
        lv = (mgr.MgrLevelSpec({F.U}, {F.P}, f_relax="amg"),)
    elif len(pb.cell_fields) == 3:
        lv = (mgr.MgrLevelSpec({F.U}, {F.S, F.S2, F.P}, f_relax="amg", n_max=4), mgr.MgrLevelSpec({F.S2}, {F.S, F.P}), mgr.MgrLevelSpec({F.S}, {F.P}))
    else:
        lv = (mgr.MgrLevelSpec({F.U}, {F.S, F.P}, f_relax="amg", n_max=4), mgr.MgrLevelSpec({F.S}, {F.P}))
    return mgr.MgrConfig(levels=lv, amg_f_relax=amg.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=10**9),
                         amg_terminal=amg.AmgConfig(strength_threshold=0.25, npartitions=10**9))
cases = [("C1", dict(n=32)), ("C1", dict(n=48)), ("C2", dict(n=48)), ("C2", dict(n=64)), ("C3", dict(n=32)), ("C3", dict(n=48)), ("C4", dict(n=32))]
for name, kw in cases:
    pb = problems.make(name, **kw)
    A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of), cfgfor(pb))
    t = time.time()
    x, st = krylov.gmres(A, h.apply, pb.rhs, cfg=krylov.GmresConfig(restart=100, max_iters=3000))
    hist = st.residual_history
    print(json.dumps(dict(cfg=name, n=kw, dofs=pb.n, its=st.iterations, conv=st.converged, rel=float(hist[-1]/hist[0]), t=time.time()-t, levels=h.level_sizes(), amg=h.amg(0).level_sizes())), flush=True)
