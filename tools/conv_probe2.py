"""Convergence probe (diagnostics, not a test): GMRES iterations of the
synthetic configs under several reference-supported preconditioner options.

    python tools/conv_probe2.py C4 64 jac gs64 fs2 gal ilu r200 ...

variants (combinable with '+', e.g. gs64+fs2):
  jac      l1-Jacobi AMG everywhere (the round-1 parity configuration)
  gsK      hybrid l1-GS AMG, partitions of ~K rows on the finest level
  fsK      K AMG V-cycles for the displacement F-relaxation
  tcK      K terminal V-cycles
  gal      Galerkin level-1 coarse grid (n_max None)
  iluK     ILU(1) global smoother on the first flow level, partitions of ~K rows
  rK       GMRES restart K
  post     F-relaxation after the coarse correction
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1904_05960_b200 import amg, krylov, mgr, problems, sparse  # noqa: E402

F = sparse.Field


def config_for(pb, var):
    opts = var.split("+")
    amg_parts_f = 10 ** 9
    amg_parts_t = 10 ** 9
    fs, tc, nmax, ilu, restart, post = 1, 1, 4, 0, 100, False
    for o in opts:
        if o.startswith("gs"):
            k = int(o[2:])
            amg_parts_f = max(1, pb.n_u // k)
            amg_parts_t = max(1, (pb.n - pb.n_u) // len(pb.cell_fields) // k)
        elif o.startswith("fs"):
            fs = int(o[2:])
        elif o.startswith("tc"):
            tc = int(o[2:])
        elif o == "gal":
            nmax = None
        elif o.startswith("ilu"):  # partitions of ~K rows on the flow level
            ilu = max(1, (pb.n - pb.n_u) // int(o[3:]))
        elif o.startswith("r"):
            restart = int(o[1:])
        elif o == "post":
            post = True
    nf = len(pb.cell_fields)
    gs = "ilu" if ilu else "none"
    if nf == 1:
        lv = (mgr.MgrLevelSpec({F.U}, {F.P}, f_relax="amg", f_relax_sweeps=fs),)
    elif nf == 3:
        lv = (mgr.MgrLevelSpec({F.U}, {F.S, F.S2, F.P}, f_relax="amg", n_max=nmax, f_relax_sweeps=fs),
              mgr.MgrLevelSpec({F.S2}, {F.S, F.P}, global_smoother=gs), mgr.MgrLevelSpec({F.S}, {F.P}))
    else:
        lv = (mgr.MgrLevelSpec({F.U}, {F.S, F.P}, f_relax="amg", n_max=nmax, f_relax_sweeps=fs),
              mgr.MgrLevelSpec({F.S}, {F.P}, global_smoother=gs))
    cfg = mgr.MgrConfig(levels=lv, terminal_cycles=tc, npartitions=max(1, ilu),
                        f_relax_position="post" if post else "pre",
                        amg_f_relax=amg.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=amg_parts_f),
                        amg_terminal=amg.AmgConfig(strength_threshold=0.25, npartitions=amg_parts_t))
    return cfg, restart


def main():
    name, n = sys.argv[1], int(sys.argv[2])
    variants = sys.argv[3:] or ["jac"]
    max_iters = int(__import__('os').environ.get('PROBE_MAX_ITERS', '3000'))
    t0 = time.perf_counter()
    if name == "C5":
        pb = problems.make(name, nxy=n, nz_per_gpu=n, gpus=int(__import__('os').environ.get('PROBE_GPUS', '1')),
                           device=True)
    else:
        pb = problems.make(name, n=n, device=True)
    torch.cuda.synchronize()
    print(f"# {name} {n}^3 n={pb.n} assembled in {time.perf_counter() - t0:.2f}s", flush=True)
    b = torch.from_numpy(pb.rhs).cuda()
    for var in variants:
        cfg, restart = config_for(pb, var)
        lay = sparse.FieldLayout(pb.field_of, pb.entity_of,
                                 sparse.Ordering.FLOW_INTERLEAVED if len(pb.cell_fields) == 2 else
                                 sparse.Ordering.FIELD_BLOCKED)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        try:
            h = mgr.mgr_setup(pb.A, lay, cfg)
        except Exception as e:  # noqa: BLE001
            print(json.dumps(dict(cfg=name, n=n, var=var, error=str(e))), flush=True)
            continue
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        gc = krylov.GmresConfig(restart=restart, max_iters=max_iters, rtol=1e-6)
        x, st = krylov.gmres(pb.A, h, b, cfg=gc)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        hist = np.asarray(st.residual_history)
        marks = {int(k): float(hist[k] / hist[0]) for k in range(0, len(hist), 100)}
        print(json.dumps(dict(cfg=name, n=n, var=var, dofs=pb.n, its=st.iterations, conv=bool(st.converged),
                              rel=float(hist[-1] / hist[0]), setup_s=round(t2 - t1, 3),
                              solve_s=round(t3 - t2, 3), ms_per_it=round(1e3 * (t3 - t2) / max(1, st.iterations), 3),
                              levels=h.level_sizes(), amg0=h.amg(0).level_sizes(), hist=marks)), flush=True)
        del h
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
