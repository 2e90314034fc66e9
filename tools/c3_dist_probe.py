import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1904_05960_b200 import dist as D, krylov, mgr, problems, sparse
base = problems.make("C3", seed=0)
pb, bounds = problems.rank_major(base, 2)
A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
opts = problems.solver_options("C3", pb)
cfg = mgr.config_from_options(opts)
h = mgr.mgr_setup(A, sparse.FieldLayout(pb.field_of, pb.entity_of), cfg)
v = np.random.default_rng(7).standard_normal(pb.n)
z = h.apply(v); zd = D.emulate_apply(h, bounds, v).cpu().numpy()
print("C3 64^3 two emulated ranks: apply bitwise", np.array_equal(z, zd), "maxdiff", float(np.abs(z-zd).max()))
gcfg = krylov.GmresConfig(restart=opts["restart"], max_iters=3000, rtol=1e-6)
x1, st = krylov.gmres(A, h.apply, pb.rhs, cfg=gcfg)
t=time.time(); xd, its, conv = D.emulate_gmres(h, bounds, pb.rhs, gcfg); print("emulated gmres", its, conv, "single", st.iterations, st.converged, round(time.time()-t,2), "s",
      "rel diff", float(np.linalg.norm(xd.cpu().numpy()-x1)/np.linalg.norm(x1)))
