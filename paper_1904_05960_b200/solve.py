"""solve_file: MGR-GMRES on a system stored on disk.

    python -m paper_1904_05960_b200.solve --matrix A.mtx --rhs b.mtx \
        --layout L.json --solver S.json

* matrix / rhs: Matrix Market (sparse.read_matrix_market / read_vector);
* layout JSON: {"field_of": [...], "entity_of": [...]} -- field tags as
  integers (0 u, 1 s, 2 p, 3 s2) or names ("u", "s", "p", "s2");
* solver JSON (all keys optional): {"levels": [{"f_fields": ["u"],
  "c_fields": ["s", "p"], "f_relax": "amg", "n_max": 4, ...}, ...],
  "terminal_cycles": 1, "f_relax_position": "pre",
  "amg_f_relax": {...AmgConfig...}, "amg_terminal": {...},
  "gmres": {"restart": 100, "max_iters": 1000, "rtol": 1e-6, "atol": 1e-12}}.
  Without "levels" the default is the parity configuration for the fields
  present (U AMG -> [S Jacobi ->] P AMG, l1-Jacobi smoothing).

Returns (and the CLI prints as JSON) a report: iterations, convergence, the
residual history, setup and solve wall times, level sizes.  Exit codes as in
SPEC.md:626: 0 success, 1 solver failure, 2 input / config error.
"""

from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from . import amg, krylov, mgr, sparse

_NAMES = {"u": 0, "s": 1, "p": 2, "s2": 3}


def _field(x) -> int:
    if isinstance(x, str):
        try:
            return _NAMES[x.lower()]
        except KeyError:
            raise ValueError(f"unknown field tag {x!r}, expected one of u/s/p/s2") from None
    return int(x)


def read_layout(path) -> sparse.FieldLayout:
    with open(path) as f:
        d = json.load(f)
    if "field_of" not in d:
        raise ValueError(f"{path}: layout needs a 'field_of' list")
    fo = np.array([_field(t) for t in d["field_of"]], dtype=np.int8)
    eo = np.asarray(d.get("entity_of", np.arange(len(fo))), dtype=np.int32)
    if len(eo) != len(fo):
        raise ValueError(f"{path}: field_of and entity_of lengths differ")
    return sparse.FieldLayout(fo, eo)


def write_layout(path, field_of, entity_of) -> None:
    with open(path, "w") as f:
        json.dump({"field_of": [int(t) for t in field_of], "entity_of": [int(e) for e in entity_of]}, f)


def default_levels(fields_present):
    F = sparse.Field
    fp = set(int(f) for f in fields_present)
    if fp == {0, 2}:
        return (mgr.MgrLevelSpec({F.U}, {F.P}, f_relax="amg"),)
    if fp == {0, 1, 2}:
        return (mgr.MgrLevelSpec({F.U}, {F.S, F.P}, f_relax="amg", n_max=4),
                mgr.MgrLevelSpec({F.S}, {F.P}, f_relax="jacobi"))
    if fp == {0, 1, 2, 3}:
        return (mgr.MgrLevelSpec({F.U}, {F.S, F.S2, F.P}, f_relax="amg", n_max=4),
                mgr.MgrLevelSpec({F.S2}, {F.S, F.P}, f_relax="jacobi"),
                mgr.MgrLevelSpec({F.S}, {F.P}, f_relax="jacobi"))
    if len(fp) == 1:
        return (mgr.MgrLevelSpec(set(), {F(next(iter(fp)))}),)
    raise ValueError(f"no default MGR levels for fields {sorted(fp)}; give 'levels' in the solver config")


def solver_config(d: dict, layout: sparse.FieldLayout):
    d = dict(d or {})
    jac = 10 ** 9
    fr = amg.AmgConfig(**{"strength_threshold": 0.5, "num_functions": 3, "npartitions": jac,
                          **d.get("amg_f_relax", {})})
    te = amg.AmgConfig(**{"strength_threshold": 0.25, "npartitions": jac, **d.get("amg_terminal", {})})
    if "levels" in d:
        levels = []
        for L in d["levels"]:
            L = dict(L)
            L["f_fields"] = {_field(t) for t in L.get("f_fields", [])}
            L["c_fields"] = {_field(t) for t in L.get("c_fields", [])}
            levels.append(mgr.MgrLevelSpec(**L))
        levels = tuple(levels)
    else:
        levels = default_levels(np.unique(layout.field_of))
    cfg = mgr.MgrConfig(levels=levels, terminal_cycles=int(d.get("terminal_cycles", 1)),
                        f_relax_position=d.get("f_relax_position", "pre"), amg_f_relax=fr, amg_terminal=te)
    g = {"restart": 100, "max_iters": 1000, "rtol": 1e-6, "atol": 1e-12, **d.get("gmres", {})}
    return cfg, krylov.GmresConfig(**g)


def solve_file(matrix, rhs, layout, solver=None) -> dict:
    """Read A, b and the layout, run mgr_setup + gmres on the GPU, report."""
    A = sparse.read_matrix_market(matrix)
    b = sparse.read_vector(rhs)
    lay = read_layout(layout)
    if A.nrows != A.ncols:
        raise ValueError("the matrix must be square")
    if len(b) != A.nrows:
        raise ValueError(f"rhs length {len(b)} does not match the matrix ({A.nrows} rows)")
    if len(lay.field_of) != A.nrows:
        raise ValueError(f"layout covers {len(lay.field_of)} dofs, the matrix has {A.nrows} rows")
    if isinstance(solver, str):
        with open(solver) as f:
            solver = json.load(f)
    cfg, gcfg = solver_config(solver, lay)
    dA = A.device()
    t0 = time.perf_counter()
    h = mgr.mgr_setup(dA, lay, cfg)
    t1 = time.perf_counter()
    x, st = krylov.gmres(dA, h.apply, b, cfg=gcfg)
    t2 = time.perf_counter()
    r = b - sparse.matvec(A, x)
    return {"n": A.nrows, "nnz": A.nnz, "iterations": st.iterations, "converged": bool(st.converged),
            "residual_history": [float(v) for v in st.residual_history],
            "true_residual": float(np.linalg.norm(r)), "rhs_norm": float(np.linalg.norm(b)),
            "setup_s": t1 - t0, "solve_s": t2 - t1, "level_sizes": [int(s) for s in h.level_sizes()],
            "x": x}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1904_05960_b200.solve")
    ap.add_argument("--matrix", required=True)
    ap.add_argument("--rhs", required=True)
    ap.add_argument("--layout", required=True)
    ap.add_argument("--solver", default=None)
    ap.add_argument("--solution", default=None, help="write x as a Matrix Market vector")
    a = ap.parse_args(argv)
    try:
        rep = solve_file(a.matrix, a.rhs, a.layout, a.solver)
    except (ValueError, OSError, json.JSONDecodeError, TypeError) as e:
        print(json.dumps({"error": str(e)}), file=sys.stderr)
        return 2
    x = rep.pop("x")
    if a.solution:
        sparse.write_vector(a.solution, x)
    print(json.dumps(rep))
    return 0 if rep["converged"] else 1


if __name__ == "__main__":
    sys.exit(main())
