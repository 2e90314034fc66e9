"""Benchmark: MGR-preconditioned GMRES solve throughput (BASELINE.json metric
"MGR-GMRES solve MDOF/s & setup time; kernel HBM GB/s vs B200 roofline").

Workload (N=1): BASELINE.json configs[1] -- two-phase poromechanics on a
32^3 grid (173,347 dofs, 11.3M nnz), 3-level MGR (U -> S -> P, N_max=4 at
level 1, AMG F-relaxation on A_uu with l1-Jacobi, Jacobi on S, AMG on P),
right-preconditioned GMRES(100) to rtol 1e-6.  Synthetic seeded input from
paper_1904_05960_b200.problems (the reference ships no assembler).

A step = one full GMRES solve from x0 = 0 with A, the MGR hierarchy and b
resident in HBM; L2 is flushed (512 MiB write) between steps, outside the
timed region.  `value` = dofs solved per second over all ranks.
`e2e` = the same solve through the public Python API with a NumPy b/x
(host->device copy of b and device->host copy of x inside the timed call).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pmgr|reference]

N > 1 (torchrun): weak scaling of the row-distributed solve -- the global
problem is the C2 slab stacked N times in z (32 x 32 x 32N, the C5 generator,
identical to C2 at N = 1), numbered rank-major; every rank builds the global
hierarchy (replicated setup) and solves on its z-slab rows with halo
exchanges / all-reduces over NCCL inside libpmgr.  Timing is the max over
ranks; `value` = global dofs / time.  `--replicas` runs N independent C2
solves instead.  `--impl reference` times the CPU oracle (the reference
algorithm restated in C, oracle/) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "MGR-GMRES solve MDOF/s"
UNIT = "MDOF/s"


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload(cfg_name, seed, device=False):
    from paper_1904_05960_b200 import problems

    pb = problems.make(cfg_name, seed=seed, device=device)
    if pb.cell_fields == (problems.FIELD_P,):
        levels = [("amg", {0}, {2}, None)]
    elif len(pb.cell_fields) == 3:
        levels = [("amg", {0}, {1, 3, 2}, 4), ("jacobi", {3}, {1, 2}, None), ("jacobi", {1}, {2}, None)]
    else:
        levels = [("amg", {0}, {1, 2}, 4), ("jacobi", {1}, {2}, None)]
    return pb, levels


def describe(cfg_name, pb):
    names = {
        "C1": "C1: single-phase Biot 16^3, 2-level MGR (U AMG -> P AMG)",
        "C2": "C2: two-phase poromechanics 32^3, 3-level MGR (U AMG, N_max=4 -> S Jacobi -> P AMG)",
        "C3": "C3: two-phase layered 64^3, 3-level MGR (U AMG, N_max=4 -> S Jacobi -> P AMG)",
        "C4": "C4: three-phase 128^3, 4-level MGR (U AMG, N_max=4 -> S2 -> S1 -> P AMG)",
        "C5": "C5: two-phase 128^3 slab, 3-level MGR",
    }
    return names.get(cfg_name, cfg_name)


# ---------------------------------------------------------------------------
# CPU reference arm (oracle port)
# ---------------------------------------------------------------------------


def oracle_solve(pb, levels, restart, rtol):
    import logging

    logging.disable(logging.WARNING)
    from oracle import oracle as O

    O.build()
    specs = tuple(O.MgrLevelSpec(frozenset(f), frozenset(c), relax, 1, nm) for relax, f, c, nm in levels)
    cfg = O.MgrConfig(levels=specs,
                      amg_f_relax=O.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=10 ** 9),
                      amg_terminal=O.AmgConfig(strength_threshold=0.25, npartitions=10 ** 9))
    A = O.Csr(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    t = time.perf_counter()
    h = O.mgr_setup(A, pb.field_of, pb.entity_of, cfg)
    setup = time.perf_counter() - t

    def solve():
        t0 = time.perf_counter()
        _, its, _, conv = O.gmres(lambda v: O.spmv(A, v), h.apply, pb.rhs, restart=restart, max_iters=1000,
                                  rtol=rtol)
        return time.perf_counter() - t0, its, conv

    return setup, solve


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank):
    if rank != 0:
        return
    threads = cpu_threads()
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    pb, levels = workload(args.config, args.seed)
    setup, solve = oracle_solve(pb, levels, args.restart, args.rtol)
    w = min(args.warmup, 1)
    k = max(1, min(args.steps, 3))
    for _ in range(w):
        solve()
    times, its = [], 0
    for _ in range(k):
        t, its, conv = solve()
        times.append(t)
    mean = statistics.mean(times)
    v = pb.n / mean / 1e6
    sample = (f"{k} full {args.config} GMRES({args.restart}) solves to rtol {args.rtol} ({its} iterations) "
              f"after {w} untimed warm-up solve(s); oracle setup {setup:.2f} s untimed")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": k,
        "warmup": w, "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generator, paper_1904_05960_b200/problems.py)",
        "config": {"workload": describe(args.config, pb), "n_dofs": pb.n, "nnz": pb.nnz, "restart": args.restart,
                   "rtol": args.rtol, "gmres_iterations": its, "parallelism": "host cores"},
        "setup_s": setup,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.f.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def run_gpu_dist(args, rank, world, local_rank):
    """Row-distributed weak-scaling solve, NCCL transport."""
    import ctypes

    import torch
    import torch.distributed as tdist

    from paper_1904_05960_b200 import _lib, amg, dist as D, krylov, mgr, problems, sparse

    torch.cuda.set_device(local_rank)
    if world > 1:
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    # the global slab stack assembled on the GPU and renumbered rank-major there
    base = problems.make_c5(seed=args.seed, nxy=32, nz_per_gpu=32, gpus=world, device=True)
    pb, bounds = problems.rank_major(base, world)
    del base
    _, levels = workload("C2", args.seed)
    F = sparse.Field
    specs = tuple(mgr.MgrLevelSpec({F(t) for t in f}, {F(t) for t in c}, f_relax=relax, n_max=nm)
                  for relax, f, c, nm in levels)
    cfg = mgr.MgrConfig(levels=specs,
                        amg_f_relax=amg.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=10 ** 9),
                        amg_terminal=amg.AmgConfig(strength_threshold=0.25, npartitions=10 ** 9))
    stream = torch.cuda.current_stream()
    A = pb.A
    lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
    tr = D.nccl_transport(rank, world, tdist)
    torch.cuda.synchronize()
    levels_info = None
    if args.replicated_setup:
        # every rank builds the global hierarchy, then keeps its rows
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h = mgr.mgr_setup(A, lay, cfg)
        e1.record(stream)
        torch.cuda.synchronize()
        setup_s = e0.elapsed_time(e1) / 1e3
        levels_info = h.level_sizes()
        t0 = time.perf_counter()
        solver = D.DeviceDistSolver(h, bounds, rank, world, tr)
        torch.cuda.synchronize()
        dist_setup_s = time.perf_counter() - t0
    else:
        # distributed setup: each rank sets up from its own rows (warm-up build
        # first, then the timed one; wall time max over ranks)
        lo_r, hi_r = int(bounds[rank]), int(bounds[rank + 1])
        A_rows = D.row_slice(A, lo_r, hi_r)
        solver = D.DeviceDistSetupSolver(A_rows, lay, cfg, bounds, rank, world, tr)
        del solver
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        solver = D.DeviceDistSetupSolver(A_rows, lay, cfg, bounds, rank, world, tr)
        torch.cuda.synchronize()
        setup_s = time.perf_counter() - t0
        dist_setup_s = None
    lo, no = solver.lo, solver.n_own
    b_own = torch.from_numpy(pb.rhs[lo:lo + no].copy()).cuda()
    gcfg = krylov.GmresConfig(restart=args.restart, max_iters=1000, rtol=args.rtol)
    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    def barrier():
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        x, st = solver.gmres(b_own, gcfg)
    clocks = Clocks(local_rank)
    launches0 = _lib.launch_count()
    times = []
    for k in range(args.steps):
        flush.fill_(float(k))
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        x, st = solver.gmres(b_own, gcfg)
        s1.record(stream)
        s1.synchronize()
        times.append(s0.elapsed_time(s1) / 1e3)
    barrier()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()

    def tmax(v):
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        if world > 1:
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        return float(t)

    t_max = tmax(statistics.mean(times))
    setup_s = tmax(setup_s)
    # e2e: host b slice in, host x slice out, inside the timed region
    e2e_times = []
    bh = pb.rhs[lo:lo + no].copy()
    for k in range(max(1, args.steps)):
        flush.fill_(float(k))
        barrier()
        t0 = time.perf_counter()
        xd, st2 = solver.gmres(torch.from_numpy(bh).cuda(), gcfg)
        xh = xd.cpu().numpy()
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_mean = tmax(statistics.mean(e2e_times))
    # true residual of the gathered solution on rank 0
    r_own = b_own - solver.spmv(x)
    rr = torch.tensor([float(torch.dot(r_own, r_own)), float(torch.dot(b_own, b_own))], dtype=torch.float64,
                      device="cuda")
    if world > 1:
        tdist.all_reduce(rr)
    rel = float(torch.sqrt(rr[0] / rr[1]))
    if rank == 0:
        line = {
            "metric": METRIC, "value": pb.n / t_max / 1e6, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, paper_1904_05960_b200/problems.py)",
            "config": {"workload": f"C2 slab x{world}: two-phase poromechanics 32x32x{32 * world} (C5 generator, "
                                   "rank-major z-slabs), 3-level MGR (U AMG, N_max=4 -> S Jacobi -> P AMG)",
                       "n_dofs": pb.n, "n_dofs_per_gpu": int(np.diff(bounds).max()), "nnz": pb.nnz,
                       "restart": args.restart, "rtol": args.rtol, "gmres_iterations": st.iterations,
                       "true_relative_residual": rel, "mgr_levels": levels_info,
                       "l2": "flushed between steps (512 MiB write, untimed)",
                       "parallelism": f"row-distributed z-slabs over {world} GPU(s): "
                                      + ("replicated setup" if args.replicated_setup else
                                         "distributed setup (pmgr_dist_setup)")
                                      + ", NCCL halo exchange / all-gather / all-reduce inside libpmgr"},
            "setup_s": setup_s, "setup_timing": "max over ranks" + ("" if args.replicated_setup else
                                                                     ", host wall clock around pmgr_dist_setup"),
            "dist_setup_s": dist_setup_s,
            "e2e": {"value": pb.n / e2e_mean / 1e6, "unit": UNIT, "h2d_bytes_per_step": 8 * no,
                    "d2h_bytes_per_step": 8 * no, "ms_per_step": e2e_mean * 1e3, "note": "per-rank slices"},
            "gpu_launches": launches, "clocks": clk, "roofline": None, "cpu_baseline": None,
            "kernel_timing": "not instrumented on the distributed path (see the N = 1 line)",
        }
        print(json.dumps(line), flush=True)
    del solver, tr
    if world > 1:
        tdist.destroy_process_group()


def run_gpu(args, rank, world, local_rank):
    import torch

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    from paper_1904_05960_b200 import _lib, amg, krylov, mgr, sparse

    device_asm = args.config not in ("C1", "C2")  # large systems: assemble on the GPU (problems.py, bitwise)
    pb, levels = workload(args.config, args.seed, device=device_asm)
    F = sparse.Field
    specs = tuple(mgr.MgrLevelSpec({F(t) for t in f}, {F(t) for t in c}, f_relax=relax, n_max=nm)
                  for relax, f, c, nm in levels)
    cfg = mgr.MgrConfig(levels=specs,
                        amg_f_relax=amg.AmgConfig(strength_threshold=0.5, num_functions=3, npartitions=10 ** 9),
                        amg_terminal=amg.AmgConfig(strength_threshold=0.25, npartitions=10 ** 9))
    stream = torch.cuda.current_stream()
    if device_asm:
        A = pb.A
    else:
        A = sparse.DeviceCsr.from_arrays(pb.n, pb.n, torch.from_numpy(pb.row_offsets).cuda(),
                                         torch.from_numpy(pb.col_indices).cuda(), torch.from_numpy(pb.values).cuda())
    lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
    b = torch.from_numpy(pb.rhs).cuda()
    gcfg = krylov.GmresConfig(restart=args.restart, max_iters=1000, rtol=args.rtol)
    L = _lib.lib()

    # ---- setup (one warm-up build, then a timed build)
    h = mgr.mgr_setup(A, lay, cfg)
    del h
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_host = time.perf_counter()
    e0.record(stream)
    h = mgr.mgr_setup(A, lay, cfg)
    e1.record(stream)
    torch.cuda.synchronize()
    setup_s = max(e0.elapsed_time(e1) / 1e3, 0.0)
    setup_wall = time.perf_counter() - t_host

    flush = torch.empty(512 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    def solve():
        x, st = krylov.gmres(A, h.apply, b, cfg=gcfg)
        return st

    for _ in range(args.warmup):
        st = solve()
    its = st.iterations
    if args.ncu:
        # one solve bracketed for `ncu --profile-from-start off`
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        st = solve()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        if rank == 0:
            print(json.dumps({"ncu_solve": True, "gmres_iterations": st.iterations, "n_dofs": pb.n}))
        return

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(local_rank)
    launches0 = _lib.launch_count()
    times = []
    for k in range(args.steps):
        flush.fill_(float(k))
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        st = solve()
        s1.record(stream)
        s1.synchronize()
        times.append(s0.elapsed_time(s1) / 1e3)
        its = st.iterations
    barrier()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    # kernel timing: the same solves again with CUDA events around the hot
    # kernels (event nodes cannot live in the production graph's WHILE body,
    # so these solves step the Arnoldi loop from the host)
    L.pmgr_prof_enable(1)
    nprof = max(1, min(args.steps, 3))
    for k in range(nprof):
        flush.fill_(float(k))
        barrier()
        solve()
    torch.cuda.synchronize()
    prof = {}
    import ctypes

    for kind, name in ((0, "outer_spmv"), (1, "frelax_l0_sweep0_residual"), (2, "frelax_l0_jacobi"),
                       (3, "mgr_apply"), (4, "cgs2_step")):
        c, ms, by = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        _lib.check(L.pmgr_prof_query(kind, ctypes.byref(c), ctypes.byref(ms), ctypes.byref(by)))
        prof[name] = {"launches": c.value, "ms_total": ms.value, "bytes_total": by.value,
                      "avg_us": (ms.value * 1e3 / c.value) if c.value else None,
                      "gbs": (by.value / (ms.value / 1e3) / 1e9) if ms.value > 0 and by.value > 0 else None}
    L.pmgr_prof_enable(0)
    # SURVEY 8(d)'s algorithmic bytes of an Arnoldi step, 8 n (2 (j+1) + 5): the
    # basis read for the projections and again for the update.  The library
    # records the compulsory bytes 8 n ((j+1) + 4) (the basis once: the update
    # pass re-reads it from L2 when it fits); both are reported.
    o = prof["cgs2_step"]
    if o["launches"]:
        comp = o["bytes_total"]
        o["bytes_total_compulsory"] = comp
        o["gbs_compulsory"] = o["gbs"]
        o["bytes_total"] = 2.0 * comp - 24.0 * pb.n * o["launches"]
        o["gbs"] = o["bytes_total"] / (o["ms_total"] / 1e3) / 1e9 if o["ms_total"] > 0 else None
        o["bytes_rule"] = "8 n (2 (j+1) + 5) per step (SURVEY 8(d)); *_compulsory: 8 n ((j+1) + 4)"

    mean = statistics.mean(times)
    t_max = mean
    if dist is not None:
        tt = torch.tensor([mean], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt)
    value = world * pb.n / t_max / 1e6

    # ---- e2e through the public API with host buffers
    e2e_times = []
    bh_pinned = torch.from_numpy(pb.rhs.copy()).pin_memory()  # the step's input in pinned host memory
    bh = bh_pinned.numpy()
    for k in range(max(1, args.steps)):
        flush.fill_(float(k))
        barrier()
        t0 = time.perf_counter()
        xh, st2 = krylov.gmres(A, h.apply, bh, cfg=gcfg)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_mean = statistics.mean(e2e_times)
    if dist is not None:
        tt = torch.tensor([e2e_mean], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_mean = float(tt)
    e2e = {"value": world * pb.n / e2e_mean / 1e6, "unit": UNIT, "h2d_bytes_per_step": 8 * pb.n,
           "d2h_bytes_per_step": 8 * pb.n + 8 * len(st2.residual_history), "ms_per_step": e2e_mean * 1e3}

    # ---- roofline of the dominant memory-bound kernel
    peak, peak_kind = peaks()
    cands = {k: v for k, v in prof.items() if k in ("outer_spmv", "frelax_l0_sweep0_residual", "frelax_l0_jacobi",
                                                     "cgs2_step") and v["gbs"]}
    dom = max(cands, key=lambda k: cands[k]["ms_total"]) if cands else None
    roof = None
    traffic = args.traffic
    tfile = os.path.join(REPO, "profiles", "roofline_traffic.json")
    if traffic is None and os.path.exists(tfile):
        try:
            with open(tfile) as f:
                tj = json.load(f)
            if tj.get("kernel") == dom and tj.get("config") == args.config:
                traffic = float(tj["dram_bytes_per_launch"])
        except Exception:
            traffic = None
    if dom:
        d = prof[dom]
        roof = {"kernel": dom, "bound": "hbm", "achieved": d["gbs"], "peak": peak, "unit": "GB/s",
                "frac": d["gbs"] / peak, "peak_source": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json)",
                "bytes_per_launch": d["bytes_total"] / d["launches"], "avg_launch_us": d["avg_us"],
                "bytes_rule": d.get("bytes_rule", "SURVEY 8(d)"),
                "traffic": traffic, "traffic_source": "profiles/roofline_traffic.json (ncu --set full, "
                                                       "dram__bytes_read.sum + dram__bytes_write.sum)"}

    if roof and prof[dom].get("gbs_compulsory"):
        roof["achieved_compulsory"] = prof[dom]["gbs_compulsory"]
        roof["frac_compulsory"] = prof[dom]["gbs_compulsory"] / peak

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline and not device_asm:
        os.environ.setdefault("OMP_NUM_THREADS", str(cpu_threads()))
        setup_c, solve_c = oracle_solve(pb, levels, args.restart, args.rtol)
        tc, its_c, _ = solve_c()
        cpu = {"value": pb.n / tc / 1e6, "unit": UNIT, "cores": int(os.environ["OMP_NUM_THREADS"]), "kind": "port",
               "sample": f"one full {args.config} GMRES({args.restart}) solve to rtol {args.rtol} ({its_c} iterations) "
                         f"by the C oracle (oracle/oracle.c), setup {setup_c:.2f} s untimed",
               "setup_s": setup_c, "gmres_iterations": its_c}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, paper_1904_05960_b200/problems.py)",
        "config": {"workload": describe(args.config, pb), "n_dofs": pb.n, "nnz": pb.nnz, "restart": args.restart,
                   "rtol": args.rtol, "gmres_iterations": its, "mgr_levels": h.level_sizes(),
                   "l2": "flushed between steps (512 MiB write, untimed)",
                   "parallelism": "replicas" if world > 1 else "single GPU"},
        "setup_s": setup_s, "setup_wall_s": setup_wall,
        "e2e": e2e, "gpu_launches": launches, "clocks": clk, "roofline": roof, "cpu_baseline": cpu,
        "kernels": prof, "kernel_timing": f"CUDA events around each launch over {nprof} extra solves "
                                          "(host-stepped Arnoldi loop, same kernels)",
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["pmgr", "reference"], default="pmgr")
    ap.add_argument("--config", default="C2")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--restart", type=int, default=100)
    ap.add_argument("--rtol", type=float, default=1e-6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ncu", action="store_true", help="profile one solve between cudaProfilerStart/Stop and exit")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent C2 solves instead of the "
                                                                "row-distributed slab stack")
    ap.add_argument("--dist", action="store_true", help="use the row-distributed path even at N = 1")
    ap.add_argument("--replicated-setup", action="store_true",
                    help="distributed path: build the global hierarchy on every rank instead of the "
                         "distributed setup")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the roofline kernel (profiles/), echoed into the JSON")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if args.dist or (world > 1 and not args.replicas and not args.ncu):
        run_gpu_dist(args, rank, world, local_rank)
        return
    run_gpu(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
