"""Benchmark: MGR-preconditioned GMRES solve throughput (BASELINE.json metric
"MGR-GMRES solve MDOF/s & setup time; kernel HBM GB/s vs B200 roofline").

Workload (N=1, default): BASELINE.json configs[3] -- C4, three-phase
poromechanics on a 128^3 grid (12,731,523 dofs, 843M nnz, assembled on the
device from the seeded generator), 4-level MGR (U -> S2 -> S1 -> P; three AMG
V-cycles of l1-Jacobi F-relaxation on A_uu, N_max=4 at level 1, Jacobi on the
saturations, AMG on the pressure), right-preconditioned GMRES(300) to rtol
1e-6 (problems.solver_options("C4")).  C4 is the largest config
that fits one GPU; the other configs are parity-test cases (--config).

A step = one full GMRES solve from x0 = 0 with A, the MGR hierarchy and b
resident in HBM; the inputs are far larger than L2 and a 512 MiB write flushes
L2 between steps anyway (outside the timed region).  `value` = dofs solved per
second over all ranks.  `e2e` = the same solve through the public Python API
with NumPy b / x (host->device copy of b, device->host copy of x and of the
residual history inside the timed call).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl pmgr|reference] [--config C4]

N > 1 (torchrun): strong scaling of the row-distributed C4 solve (the N = 1
workload split into rank-major z-slabs, distributed setup, NCCL halo
exchanges / all-gathers / all-reduces inside libpmgr); --weak runs the C5
weak-scaling stack instead (a 128^3 slab per GPU stacked in z).  `--impl reference` times the CPU oracle (the
reference algorithm restated in C, oracle/) on the host cores, rank 0 only.
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
DEFAULT_CONFIG = "C4"
DATA = "synthetic (seeded generator, paper_1904_05960_b200/problems.py; device-assembled from C3 up)"

# GMRES iterations of the production configurations at full size (GPU solves,
# tests/test_gpu_parity.py::test_full_size_solve_converges; the CPU oracle's
# count is the same +-1 wherever it has been run to convergence).  Used only to
# scale the CPU arm's per-iteration sample to a solve rate.
FULL_ITERATIONS = {"C3": 580, "C4": 276, "C5": 220}
# the CPU sample of configs above this size is a z-slab of the same generator
CPU_SAMPLE_MAX_DOFS = 2_500_000


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def make_problem(cfg_name, seed, device=False, slab_nz=None):
    from paper_1904_05960_b200 import problems

    if slab_nz is not None:
        if cfg_name == "C4":
            return problems.make_c4(seed=seed, n=128, nz=slab_nz, device=device)
        if cfg_name == "C5":
            return problems.make_c5(seed=seed, nxy=128, nz_per_gpu=slab_nz, gpus=1, device=device)
        raise ValueError(f"no slab sample for {cfg_name}")
    return problems.make(cfg_name, seed=seed, device=device)


def solver_summary(opts):
    names = {0: "U", 1: "S", 2: "P", 3: "S2"}
    lv = []
    for L in opts["levels"]:
        f = "+".join(names[t] for t in sorted(L["f"]))
        c = "+".join(names[t] for t in sorted(L["c"]))
        item = f"{f}|{c}: {L['f_relax']}"
        if L.get("f_relax_sweeps", 1) > 1:
            item += f" x{L['f_relax_sweeps']}"
        if L.get("n_max") is not None:
            item += f", N_max={L['n_max']}"
        if L.get("global_smoother", "none") != "none":
            item += f", global {L['global_smoother']}(1) over {opts['npartitions']} partitions"
        lv.append(item)
    return {"mgr_levels": lv, "terminal": "AMG (theta 0.25, l1-Jacobi)", "f_relax_amg": "theta 0.5, 3 functions, "
            "l1-Jacobi", "restart": opts["restart"], "rtol": opts["rtol"], "max_iters": opts["max_iters"],
            "variant": opts["variant"]}


def config_block(cfg_name, n, nnz, opts, level_sizes):
    """The `config` object both arms print (identical keys and values)."""
    names = {
        "C1": "C1: single-phase Biot 16^3",
        "C2": "C2: two-phase poromechanics 32^3",
        "C3": "C3: two-phase layered poromechanics 64^3",
        "C4": "C4: three-phase poromechanics 128^3",
        "C5": "C5: two-phase poromechanics 128^3 slab (per GPU)",
    }
    return {"workload": names.get(cfg_name, cfg_name) + " -- MGR-preconditioned GMRES to rtol 1e-6",
            "n_dofs": int(n), "nnz": int(nnz), "solver": solver_summary(opts), "mgr_level_sizes": level_sizes,
            "parallelism": "single GPU / host cores"}


def mean_arnoldi_index(its, restart):
    return float(np.mean([k % restart for k in range(max(1, its))]))


# ---------------------------------------------------------------------------
# CPU arm: the oracle (reference algorithm restated in C + NumPy, oracle/)
# ---------------------------------------------------------------------------


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_sample(cfg_name, seed, n_full, its, steps, warmup, log=None):
    """Time the oracle's solve phase.  Small configs: full solves (a step = one
    solve).  Large configs: a step = one Arnoldi step of the oracle (M^-1 v,
    A z, modified Gram-Schmidt against j+1 basis vectors with j the solve's
    mean Arnoldi index, normalisation), on the full problem when it has at most
    CPU_SAMPLE_MAX_DOFS dofs, else on a z-slab of the same generator scaled to
    the full size by rows; the rate is n / (its * step time)."""
    import logging

    logging.disable(logging.WARNING)
    from oracle import oracle as O
    from paper_1904_05960_b200 import problems

    O.build()
    slab = None
    if n_full > CPU_SAMPLE_MAX_DOFS and cfg_name in ("C4", "C5"):
        slab = 16
    t0 = time.perf_counter()
    pb = make_problem(cfg_name, seed, device=False, slab_nz=slab)
    gen_s = time.perf_counter() - t0
    opts = problems.solver_options(cfg_name, pb)
    cfg = O.config_from_options(opts)
    A = O.Csr(pb.n, pb.n, pb.row_offsets, pb.col_indices, pb.values)
    t0 = time.perf_counter()
    h = O.mgr_setup(A, pb.field_of, pb.entity_of, cfg)
    setup_s = time.perf_counter() - t0
    scale = n_full / pb.n
    if log:
        log(f"cpu sample: {pb.name} n={pb.n} generated in {gen_s:.1f}s, oracle setup {setup_s:.1f}s")
    full_solves = cfg_name in ("C1", "C2")
    if full_solves:
        def step():
            t = time.perf_counter()
            _, k, _, conv = O.gmres(lambda y: O.spmv(A, y), h.apply, pb.rhs, restart=opts["restart"],
                                    max_iters=opts["max_iters"], rtol=opts["rtol"])
            return time.perf_counter() - t, k
    else:
        j = int(round(mean_arnoldi_index(its, opts["restart"])))
        rng = np.random.default_rng(7)
        V = rng.standard_normal((j + 2, pb.n))
        V /= np.linalg.norm(V, axis=1)[:, None]
        v0 = V[0].copy()

        def step():
            t = time.perf_counter()
            w = O.spmv(A, h.apply(v0))
            for i in range(j + 1):  # the oracle's MGS (krylov.py:66-70)
                hij = float(V[i] @ w)
                w = w - hij * V[i]
            hn = float(np.linalg.norm(w))
            V[j + 1] = w / hn
            return time.perf_counter() - t, None

    for _ in range(warmup):
        step()
    times, k_its = [], its
    for _ in range(steps):
        t, k = step()
        times.append(t)
        if k is not None:
            k_its = k
    mean = statistics.mean(times)
    if full_solves:
        value = n_full / mean / 1e6
        sample = (f"{steps} full {cfg_name} GMRES solves by the oracle ({k_its} iterations each) after {warmup} "
                  f"untimed warm-up solve(s); oracle setup {setup_s:.2f} s untimed")
    else:
        value = n_full / (mean * scale * its) / 1e6
        where = (f"a {pb.nx}x{pb.ny}x{pb.nz} z-slab of the {cfg_name} generator ({pb.n} dofs, scaled by rows x"
                 f"{scale:.2f})" if slab else f"the full {cfg_name} problem ({pb.n} dofs)")
        sample = (f"{steps} oracle Arnoldi steps (M^-1 v, A z, MGS against {j + 1} vectors = the mean index of a "
                  f"{its}-iteration GMRES({opts['restart']}) solve, normalisation) on {where}, after {warmup} "
                  f"warm-up step(s); rate = n / ({its} iterations x step time); oracle setup {setup_s:.1f} s untimed")
    return {"value": value, "unit": UNIT, "ms_per_step": mean * 1e3, "steps": steps, "warmup": warmup,
            "setup_s": setup_s, "sample": sample, "sample_dofs": pb.n, "scale": scale,
            "level_sizes": [int(x) for x in h.level_sizes()], "iterations_used": k_its}


def run_reference(args, rank):
    if rank != 0:
        return
    threads = cpu_threads()
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    from paper_1904_05960_b200 import problems

    # the full problem's size and configuration (host generator metadata only
    # for the large configs: n and nnz follow from the grid)
    pb_meta = full_problem_meta(args.config, args.seed)
    if args.restart:
        pb_meta["opts"]["restart"] = args.restart
    its = FULL_ITERATIONS.get(args.config, 0)
    res = cpu_sample(args.config, args.seed, pb_meta["n"], its, args.steps, args.warmup,
                     log=lambda m: print(m, file=sys.stderr, flush=True))
    if res["scale"] == 1.0:
        pb_meta["level_sizes"] = res["level_sizes"]
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": config_block(args.config, pb_meta["n"], pb_meta["nnz"], pb_meta["opts"], pb_meta["level_sizes"]),
        "gmres_iterations": res["iterations_used"],
        "setup_s": res["setup_s"],
        "cpu_baseline": {"value": res["value"], "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": res["sample"]},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def full_problem_meta(cfg_name, seed):
    """n, nnz, solver options and MGR level sizes of the full problem without
    building it on the host when it is large (the grid determines them;
    pinned by the tests: problems.py's generators and the goldens)."""
    from paper_1904_05960_b200 import problems

    if cfg_name in ("C1", "C2", "C3"):
        pb = problems.make(cfg_name, seed=seed)
        opts = problems.solver_options(cfg_name, pb)
        return {"n": pb.n, "nnz": pb.nnz, "opts": opts, "level_sizes": None}
    known = {  # (n, nnz, MGR level sizes) of the device-assembled full problems (bench GPU lines)
        "C4": (12731523, 843347322, [12731523, 6291456, 4194304, 2097152]),
        "C5": (10634371, None, [10634371, 4194304, 2097152]),
    }
    n, nnz, sizes = known[cfg_name]

    class _Meta:  # what solver_options reads
        pass

    m = _Meta()
    m.cell_fields = (1, 3, 2) if cfg_name == "C4" else (1, 2)
    m.n = n
    m.n_u = 3 * 129 ** 3
    return {"n": n, "nnz": nnz, "opts": problems.solver_options(cfg_name, m), "level_sizes": sizes}


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
    # the global problem assembled on every GPU and renumbered rank-major there:
    # weak scaling = the C5 slab stack (ns^3 cells per GPU), strong scaling =
    # the fixed C4 128^3 problem
    ns = args.slab
    c3 = (not args.weak) and args.config == "C3"
    if c3:
        # C3 (64^3, "1 GPU and 2 GPUs"): its production configuration has an
        # ILU(1) global smoother, which the row distribution takes from a
        # hierarchy built whole on every rank (the partitions of 16 flow rows
        # fall on the z-slab boundaries); 1.3M dofs set up in 0.13 s
        base = problems.make("C3", seed=args.seed, device=True)
        opts = problems.solver_options("C3", base, variant=args.dist_variant)
        args.replicated_setup = True
    elif not args.weak:
        base = problems.make_c4(seed=args.seed, n=128, device=True)
        opts = problems.solver_options("C4", base, variant=args.dist_variant)
    else:
        base = problems.make_c5(seed=args.seed, nxy=ns, nz_per_gpu=ns, gpus=world, device=True)
        opts = problems.solver_options("C5", base, variant=args.dist_variant)
    pb, bounds = problems.rank_major(base, world)
    del base
    cfg = mgr.config_from_options(opts)
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
    gcfg = krylov.GmresConfig(restart=opts["restart"], max_iters=opts["max_iters"], rtol=opts["rtol"])
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
            "warmup": args.warmup, "ms_per_step": t_max * 1e3, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, paper_1904_05960_b200/problems.py)",
            "config": {"workload": ("C3: two-phase layered poromechanics 64^3 over " + f"{world} GPU(s) (rank-major z-slabs)"
                                    if c3 else
                                    "C4: three-phase poromechanics 128^3 over " + f"{world} GPU(s) (rank-major z-slabs)"
                                    if not args.weak else
                                    f"C5: two-phase poromechanics {ns}x{ns}x{ns * world} ({ns}^3 cells per GPU, "
                                    "rank-major z-slabs)") + " -- MGR-preconditioned GMRES to rtol 1e-6",
                       "n_dofs": pb.n, "n_dofs_per_gpu": int(np.diff(bounds).max()), "nnz": pb.nnz,
                       "solver": solver_summary(opts), "gmres_iterations": st.iterations,
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
    import ctypes

    import torch

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    from paper_1904_05960_b200 import _lib, krylov, mgr, problems, sparse

    device_asm = args.config not in ("C1", "C2")  # large systems: assembled on the GPU (problems.py, bitwise)
    t_asm = time.perf_counter()
    pb = make_problem(args.config, args.seed, device=device_asm)
    torch.cuda.synchronize()
    asm_s = time.perf_counter() - t_asm
    opts = problems.solver_options(args.config, pb)
    if args.restart:
        opts["restart"] = args.restart
    cfg = mgr.config_from_options(opts)
    stream = torch.cuda.current_stream()
    if device_asm:
        A = pb.A
    else:
        A = sparse.DeviceCsr.from_arrays(pb.n, pb.n, torch.from_numpy(pb.row_offsets).cuda(),
                                         torch.from_numpy(pb.col_indices).cuda(), torch.from_numpy(pb.values).cuda())
    lay = sparse.FieldLayout(pb.field_of, pb.entity_of)
    b = torch.from_numpy(pb.rhs).cuda()
    gcfg = krylov.GmresConfig(restart=opts["restart"], max_iters=opts["max_iters"], rtol=opts["rtol"])
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
        x, st = krylov.gmres(A, h, b, cfg=gcfg)
        return st

    st = None
    for _ in range(args.warmup):
        st = solve()
    its = st.iterations if st is not None else 0
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
    times, conv = [], True
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
        conv = conv and st.converged
    barrier()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    hist = np.asarray(st.residual_history)

    # ---- kernel timing: one more solve with CUDA events around the hot
    # launches (event nodes cannot live in the production graph's WHILE body,
    # so this solve steps the Arnoldi loop from the host; same kernels)
    L.pmgr_prof_enable(1)
    flush.fill_(-1.0)
    barrier()
    solve()
    torch.cuda.synchronize()
    prof = {}
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
    # records the compulsory bytes 8 n ((j+1) + 4); both are reported.
    o = prof["cgs2_step"]
    if o["launches"]:
        comp = o["bytes_total"]
        o["bytes_total_compulsory"] = comp
        o["gbs_compulsory"] = o["gbs"]
        o["bytes_total"] = 2.0 * comp - 24.0 * pb.n * o["launches"]
        o["gbs"] = o["bytes_total"] / (o["ms_total"] / 1e3) / 1e9 if o["ms_total"] > 0 else None
        o["bytes_rule"] = "8 n (2 (j+1) + 5) per step (SURVEY 8(d)); *_compulsory: 8 n ((j+1) + 4)"
    # the whole MGR application: algorithmic bytes from the library's ledger
    apply_bytes, apply_kernels = h.apply_bytes()
    m = prof["mgr_apply"]
    m["bytes_per_launch"] = apply_bytes
    m["kernels_per_launch"] = apply_kernels
    if m["launches"] and m["ms_total"] > 0:
        m["bytes_total"] = apply_bytes * m["launches"]
        m["gbs"] = m["bytes_total"] / (m["ms_total"] / 1e3) / 1e9

    mean = statistics.mean(times)
    t_max = mean
    if dist is not None:
        tt = torch.tensor([mean], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt)
    value = world * pb.n / t_max / 1e6

    # ---- solve GB/s = sum over the iterations of
    # B_SpMV(A) + B_MGR_apply + B_orth(j), plus each restart's combine, apply
    # and true residual, over the solve time
    spmv_b = prof["outer_spmv"]["bytes_total"] / max(1, prof["outer_spmv"]["launches"])
    m_r = opts["restart"]
    solve_bytes = 0.0
    for k in range(its):
        j = k % m_r
        solve_bytes += spmv_b + apply_bytes + 8.0 * pb.n * (2 * (j + 1) + 5)
    cycles = (its + m_r - 1) // m_r
    solve_bytes += cycles * (apply_bytes + spmv_b + 8.0 * pb.n * (m_r + 3))
    solve_gbs = solve_bytes / t_max / 1e9

    # ---- e2e through the public API with host buffers
    e2e_times = []
    bh_pinned = torch.from_numpy(pb.rhs.copy()).pin_memory()  # the step's input in pinned host memory
    bh = bh_pinned.numpy()
    for k in range(max(1, min(args.steps, 3))):
        flush.fill_(float(k))
        barrier()
        t0 = time.perf_counter()
        xh, st2 = krylov.gmres(A, h, bh, cfg=gcfg)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_mean = statistics.mean(e2e_times)
    if dist is not None:
        tt = torch.tensor([e2e_mean], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_mean = float(tt)
    e2e = {"value": world * pb.n / e2e_mean / 1e6, "unit": UNIT, "h2d_bytes_per_step": 8 * pb.n,
           "d2h_bytes_per_step": 8 * pb.n + 8 * len(st2.residual_history), "ms_per_step": e2e_mean * 1e3,
           "steps": len(e2e_times)}
    # true residual of the last solution (host arrays)
    r = b - sparse.matvec(A, torch.from_numpy(xh).cuda())
    true_rel = float(torch.linalg.vector_norm(r) / torch.linalg.vector_norm(b))

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
                                                       "dram__bytes_read.sum + dram__bytes_write.sum, per launch)",
                "solve_gbs": solve_gbs, "solve_frac": solve_gbs / peak,
                "solve_rule": "sum_k [B_SpMV(A) + B_MGR_apply + 8n(2(j_k+1)+5)] + per restart "
                              "[B_MGR_apply + B_SpMV(A) + 8n(m+3)], over the solve time (SURVEY 8(d))"}
        if d.get("gbs_compulsory"):
            roof["achieved_compulsory"] = d["gbs_compulsory"]
            roof["frac_compulsory"] = d["gbs_compulsory"] / peak
        if roof["frac"] > 1.0:
            roof["note"] = ("frac > 1: the peak is a COPY bandwidth (half reads, half writes); this kernel's traffic "
                            "is almost all reads, which HBM3e serves faster than a copy (8.19 TB/s raw)")

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        os.environ.setdefault("OMP_NUM_THREADS", str(cpu_threads()))
        res = cpu_sample(args.config, args.seed, pb.n, its, steps=2, warmup=1,
                         log=lambda m: print(m, file=sys.stderr, flush=True))
        cpu = {"value": res["value"], "unit": UNIT, "cores": int(os.environ["OMP_NUM_THREADS"]), "kind": "port",
               "sample": res["sample"], "setup_s": res["setup_s"]}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": config_block(args.config, pb.n, pb.nnz, opts, [int(x) for x in h.level_sizes()]),
        "gmres_iterations": its, "converged": conv, "true_relative_residual": true_rel,
        "final_residual_history_ratio": float(hist[-1] / hist[0]),
        "l2": "inputs far larger than L2; 512 MiB L2 flush write between steps (untimed)",
        "setup_s": setup_s, "setup_wall_s": setup_wall, "assembly_s": asm_s,
        "dofs_iterations_per_s": pb.n * its / t_max,
        "e2e": e2e, "gpu_launches": launches, "clocks": clk, "roofline": roof, "cpu_baseline": cpu,
        "kernels": prof, "kernel_timing": "CUDA events around each launch over 1 extra solve "
                                          "(host-stepped Arnoldi loop, same kernels)",
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["pmgr", "reference"], default="pmgr")
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--restart", type=int, default=None, help="override the configuration's GMRES restart")
    ap.add_argument("--slab", type=int, default=128, help="distributed path: cells per side of each GPU's slab")
    ap.add_argument("--weak", action="store_true",
                    help="N > 1: weak scaling of the C5 slab stack (--slab^3 cells per GPU) instead of the default "
                         "strong scaling of the C4 problem (the N = 1 workload)")
    ap.add_argument("--dist-variant", default="production", choices=["parity", "production"],
                    help="distributed path: solver configuration (problems.solver_options)")
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
    if args.dist or args.weak or (world > 1 and not args.replicas and not args.ncu):
        run_gpu_dist(args, rank, world, local_rank)
        return
    run_gpu(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
