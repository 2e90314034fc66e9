"""Row-distributed apply against the single-GPU apply on small C5 / C4 problems
at the DEFAULT replication / collapse thresholds (the tests pin the thresholds
that keep the coarse levels distributed): prints whether the sliced and the
distributed-setup applications are bitwise equal and the largest difference.
    python tools/dist_probe.py"""
import sys, numpy as np
sys.path.insert(0, ".")
from paper_1904_05960_b200 import dist as D, mgr, problems, sparse
for name, base in (("C5", problems.make_c5(seed=4, nxy=10, nz_per_gpu=5, gpus=2)), ("C4", problems.make_c4(seed=4, n=8))):
    for variant in ("parity", "production"):
        pb, bounds = problems.rank_major(base, 2)
        opts = problems.solver_options(name, pb, variant=variant)
        cfg = mgr.config_from_options(opts)
        A = sparse.CsrMatrix(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
        lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
        h = mgr.mgr_setup(A, lay, cfg)
        v = np.random.default_rng(11).standard_normal(pb.n)
        z1 = h.apply(v)
        ze = D.emulate_apply(h, bounds, v).cpu().numpy()
        zs = D.emulate_setup_apply(A, lay, cfg, bounds, v).cpu().numpy()
        print(name, variant, "levels", h.level_sizes(), "amg0", h.amg(0).level_sizes(),
              "sliced bitwise", np.array_equal(ze, z1), "dist-setup bitwise", np.array_equal(zs, z1),
              "maxdiff", float(np.abs(zs - z1).max()), flush=True)
