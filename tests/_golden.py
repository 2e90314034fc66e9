"""Helpers shared by the parity tests: load golden fixtures, digests,
oracle hierarchies for the generated problems (test infrastructure)."""

from __future__ import annotations

import hashlib
import os

import numpy as np

from oracle import oracle as O
from paper_1904_05960_b200 import problems

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
JACOBI = 10 ** 9


def load(tag):
    return np.load(os.path.join(GOLDEN, f"ref_{tag}.npz"))


def digest(ro, ci, v=None) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(ro, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(ci, dtype=np.int32).tobytes())
    if v is not None:
        h.update((np.ascontiguousarray(v, dtype=np.float64) + 0.0).tobytes())
    return h.hexdigest()


def dcsr(m) -> str:
    return digest(m.ro, m.ci, m.v)


def vec_sha(v) -> str:
    return hashlib.sha256((np.ascontiguousarray(v, dtype=np.float64) + 0.0).tobytes()).hexdigest()


def get_csr(d, key):
    shape = d[key + "_shape"]
    return O.Csr(int(shape[0]), int(shape[1]), d[key + "_ro"], d[key + "_ci"], d[key + "_v"])


# problem tag -> (generator call, n_max, four_field)
CASES = {
    "c1_6": (lambda: problems.make_c1(seed=3, n=6), None, False),
    "c2_6": (lambda: problems.make_c2(seed=5, n=6), 4, False),
    "c4_4": (lambda: problems.make_c4(seed=9, n=4), 4, True),
    "c1_16": (lambda: problems.make_c1(seed=0, n=16), None, False),
    "c2_32": (lambda: problems.make_c2(seed=0, n=32), 4, False),
    "c4_16": (lambda: problems.make_c4(seed=0, n=16), 4, True),
    "c3_16": (lambda: problems.make_c3(seed=0, n=16), 4, False),
    # parity configuration at 32^3: C4 125 iterations, C3 2801 (the stall is the algorithm's)
    "c4_32": (lambda: problems.make_c4(seed=0, n=32), 4, True),
    "c3_32": (lambda: problems.make_c3(seed=0, n=32), 4, False),
}

# production configurations (problems.solver_options) at 32^3, goldens from the reference
PROD_CASES = {
    "c3_32p": ("C3", dict(n=32)),
    "c4_32p": ("C4", dict(n=32)),
}
# full-size production goldens from the pinned oracle (oracle/make_golden_full.py)
FULL_CASES = {
    "c3_64p": ("C3", dict(n=64)),
    "c4_128p": ("C4", dict(n=128)),
    "c5_128p": ("C5", dict(nxy=128, nz_per_gpu=128, gpus=1)),
}


def gmres_options(tag, pb=None):
    """(restart, max_iters) the golden's GMRES solve used."""
    if tag in PROD_CASES:
        name, kw = PROD_CASES[tag]
        o = problems.solver_options(name, pb if pb is not None else problems.make(name, **kw))
        return o["restart"], o["max_iters"]
    if tag == "c3_32":
        return 100, 3000
    return 100, 1000


def oracle_levels(pb, n_max, four_field):
    U, S, P, S2 = problems.FIELD_U, problems.FIELD_S, problems.FIELD_P, problems.FIELD_S2
    if four_field:
        return (O.MgrLevelSpec(frozenset({U}), frozenset({S, S2, P}), "amg", 1, n_max),
                O.MgrLevelSpec(frozenset({S2}), frozenset({S, P}), "jacobi", 1, None),
                O.MgrLevelSpec(frozenset({S}), frozenset({P}), "jacobi", 1, None))
    if pb.cell_fields == (P,):
        return (O.MgrLevelSpec(frozenset({U}), frozenset({P}), "amg", 1, n_max),)
    return (O.MgrLevelSpec(frozenset({U}), frozenset({S, P}), "amg", 1, n_max),
            O.MgrLevelSpec(frozenset({S}), frozenset({P}), "jacobi", 1, None))


# option variants (oracle/make_golden.py VARIANTS): (levels, terminal_cycles, position)
U_, S_, P_ = problems.FIELD_U, problems.FIELD_S, problems.FIELD_P
VARIANT_SPECS = {
    "c2_6_v1": ([dict(f={U_}, c={S_, P_}, f_relax="amg", f_relax_sweeps=2, interp="injection_only", n_max=4),
                 dict(f={S_}, c={P_}, f_relax="jacobi")], 1, "pre"),
    "c2_6_v2": ([dict(f={U_}, c={S_, P_}, f_relax="amg"),
                 dict(f={S_}, c={P_}, f_relax="jacobi", f_relax_sweeps=2)], 2, "post"),
    "c2_6_v3": ([dict(f={U_}, c={S_, P_}, f_relax="amg", n_max=4),
                 dict(f={S_}, c={P_}, f_relax="none")], 1, "pre"),
    # hybrid l1-GS AMG smoothing with 16 partitions (both AMGs)
    "c2_6_v4": ([dict(f={U_}, c={S_, P_}, f_relax="amg", n_max=4),
                 dict(f={S_}, c={P_}, f_relax="jacobi")], 1, "pre", dict(f_parts=16, t_parts=16)),
    # level-2 global smoothers (default_three_level, mgr.py:104-120)
    "c2_6_v5": ([dict(f={U_}, c={S_, P_}, f_relax="amg", n_max=4),
                 dict(f={S_}, c={P_}, f_relax="jacobi", global_smoother="ilu", ilu_fill=1)], 1, "pre",
                dict(npartitions=1)),
    "c2_6_v6": ([dict(f={U_}, c={S_, P_}, f_relax="amg", n_max=4),
                 dict(f={S_}, c={P_}, f_relax="jacobi", global_smoother="ilu", ilu_fill=1)], 1, "pre",
                dict(npartitions=8)),
    "c2_6_v7": ([dict(f={U_}, c={S_, P_}, f_relax="amg", n_max=4),
                 dict(f={S_}, c={P_}, f_relax="jacobi", global_smoother="hbgs", hbgs_sweeps=3)], 1, "pre",
                dict(npartitions=1, interleaved=True)),
    "c2_6_v8": ([dict(f={U_}, c={S_, P_}, f_relax="amg", n_max=4),
                 dict(f={S_}, c={P_}, f_relax="jacobi", global_smoother="hbgs", hbgs_sweeps=3)], 1, "pre",
                dict(npartitions=4, interleaved=True)),
    "c2_6_v9": ([dict(f={U_}, c={S_, P_}, f_relax="amg", n_max=4),
                 dict(f={S_}, c={P_}, f_relax="jacobi", global_smoother="ilu", ilu_fill=0)], 1, "pre",
                dict(npartitions=3)),
}


def variant_options(tag):
    spec = VARIANT_SPECS[tag]
    return spec[3] if len(spec) > 3 else {}


def oracle_variant_hierarchy(tag):
    levels, tc, pos = VARIANT_SPECS[tag][:3]
    opt = variant_options(tag)
    pb = problems.make_c2(seed=5, n=6)
    specs = tuple(O.MgrLevelSpec(frozenset(lv["f"]), frozenset(lv["c"]), lv.get("f_relax", "jacobi"),
                                 lv.get("f_relax_sweeps", 1), lv.get("n_max"), lv.get("interp", "injection_jacobi"),
                                 lv.get("global_smoother", "none"), lv.get("ilu_fill", 1), lv.get("hbgs_sweeps", 3))
                  for lv in levels)
    fp, tp = opt.get("f_parts", JACOBI), opt.get("t_parts", JACOBI)
    cfg = O.MgrConfig(levels=specs, terminal_cycles=tc,
                      amg_f_relax=O.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=fp),
                      amg_terminal=O.AmgConfig(strength_threshold=0.25, npartitions=tp),
                      f_relax_position=pos, npartitions=opt.get("npartitions", 1))
    return pb, O.mgr_setup(problem_csr(pb), pb.field_of, pb.entity_of, cfg)


def oracle_config(levels, parts=JACOBI):
    return O.MgrConfig(levels=levels,
                       amg_f_relax=O.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=parts),
                       amg_terminal=O.AmgConfig(strength_threshold=0.25, npartitions=parts))


def problem_csr(pb):
    return O.Csr(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)


def oracle_hierarchy(tag):
    if tag in PROD_CASES:
        name, kw = PROD_CASES[tag]
        pb = problems.make(name, **kw)
        cfg = O.config_from_options(problems.solver_options(name, pb))
        return pb, O.mgr_setup(problem_csr(pb), pb.field_of, pb.entity_of, cfg)
    gen, n_max, four = CASES[tag]
    pb = gen()
    cfg = oracle_config(oracle_levels(pb, n_max, four))
    h = O.mgr_setup(problem_csr(pb), pb.field_of, pb.entity_of, cfg)
    return pb, h
