"""Oracle hierarchy from a device hierarchy's exports (test / benchmark
infrastructure, never the product path).

bench.py's `cpu_baseline` leg times the oracle's solve phase on the full
workload.  The oracle's own setup at C4 (128^3, 846M nnz) takes minutes of
host time, which does not fit a bounded CPU sample; since the device setup is
bitwise equal to the oracle's (tests/test_gpu_parity.py, full-size SHA goldens
produced by oracle/make_golden_full.py), the operators are downloaded from the
device instead and wrapped into the oracle's own MgrHierarchy / AmgHierarchy
containers.  Everything the oracle then computes (l1 sweeps, SpMV, dense LU
solves, ILU substitutions, MGS GMRES) is its own C / NumPy code.
"""

from __future__ import annotations

import numpy as np

from oracle import oracle as O


def _csr(t) -> O.Csr:
    nr, nc, ro, ci, v = t
    return O.Csr(nr, nc, ro, ci, v)


def _amg(h_dev, cfg: O.AmgConfig) -> O.AmgHierarchy:
    levels_raw, coarse = h_dev.export_raw()
    levels = []
    for a, p, is_c, dt in levels_raw:
        A, P = _csr(a), _csr(p)
        starts = O.partition_starts(A.nrows, cfg.npartitions)
        levels.append(O.AmgLevel(A, P, O.transpose(P), None, is_c, dt, starts))
    C = _csr(coarse)
    return O.AmgHierarchy(levels, C, O.lu_factor(C.to_dense()), cfg)


def hierarchy(h, A_dev, field_of, entity_of, opts) -> O.MgrHierarchy:
    """O.MgrHierarchy for the device MgrHierarchy `h` built from A_dev with
    problems.solver_options `opts`."""
    cfg = O.config_from_options(opts)
    A = _csr((A_dev.nrows, A_dev.ncols) + A_dev.download())
    fo = np.asarray(field_of, dtype=np.int8)
    eo = np.asarray(entity_of, dtype=np.int32)
    levels = []
    cur = A
    views = h.levels
    for l, spec in enumerate(cfg.levels[:len(views)]):
        is_c = np.asarray(views[l].split.is_c, dtype=bool)
        f_rows = np.flatnonzero(~is_c)
        P = _csr((lambda d: (d.nrows, d.ncols) + d.download())(h._export_dev(l, 0)))
        dinv = 1.0 / cur.diagonal()[f_rows]
        if spec.f_relax == "amg":
            acfg = cfg.amg_f_relax
            nf = 3 if set(spec.f_fields) == {0} else 1
            acfg = O.AmgConfig(acfg.strength_threshold, acfg.max_levels, acfg.coarse_size_cutoff, nf,
                               acfg.npartitions, acfg.cycles)
            frelax = ("amg", _amg(h.amg(l), acfg), max(1, spec.f_relax_sweeps))
        elif spec.f_relax == "jacobi":
            a_ff = O.extract_blocks(cur, is_c)[0] if spec.f_relax_sweeps > 1 else None
            frelax = ("jacobi", a_ff, max(1, spec.f_relax_sweeps))
        else:
            frelax = None
        smoother = None
        if spec.global_smoother == "ilu":
            lu = _csr((lambda d: (d.nrows, d.ncols) + d.download())(h._export_dev(l, 2)))
            smoother = O.GlobalSmoother.__new__(O.GlobalSmoother)
            smoother.kind = "ilu"
            smoother.starts = O.partition_starts(cur.nrows, cfg.npartitions, align=2)
            smoother.lu = lu
            rows = lu.rows_of_entries()
            smoother.dpos = np.flatnonzero(lu.ci == rows).astype(np.int64)
        elif spec.global_smoother != "none":
            smoother = O.GlobalSmoother(cur, fo, eo, spec, cfg.npartitions)
        coarse = _csr((lambda d: (d.nrows, d.ncols) + d.download())(h._export_dev(l, 1)))
        levels.append(O.MgrLevel(cur, fo, eo, is_c, None, P, frelax, spec, dinv, smoother))
        fo, eo = fo[is_c], eo[is_c]
        cur = coarse
    term = _amg(h.terminal_solver, cfg.amg_terminal)
    return O.MgrHierarchy(levels, cur, term, max(1, cfg.terminal_cycles), cfg.f_relax_position)
