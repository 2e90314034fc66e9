"""z-slab domain decomposition: ownership, halo plans and the distributed
Krylov plumbing.

One process per GPU.  Rank r owns the node planes and cell layers
z in [z0_r, z1_r) of the structured poromechanics grid (the last rank also
owns the top node plane) and every dof living on them.  Rows stay in the
global ordering's relative order, columns keep their global stored order
inside each row, so a row's products are summed in the same order on any
number of ranks.  Communication happens only where the path has a real
exchange step:

* halo exchange of x before every SpMV / smoother / transfer (point-to-point
  with the z-neighbours; NCCL over NVLink on the GPU, gloo in CPU tests);
* all-reduce of the Arnoldi projections and norms.

The local compute is pluggable (`local_matvec`): the oracle in the CPU
tests (gloo, world_size 2).  The device path (`DeviceDistSolver`, bottom of
this file) is libpmgr's row distribution: replicated setup of a rank-major
problem, every operator sliced to the rank's rows, halo exchanges over NCCL
inside libpmgr; `emulate_apply` / `emulate_gmres` run N ranks on one GPU
(loopback transport) for the parity tests.
"""

from __future__ import annotations

import ctypes
import sys
from dataclasses import dataclass, field

import numpy as np


def slab_bounds(nz: int, nranks: int):
    """Cell-layer ranges [z0, z1) per rank (near-equal, contiguous)."""
    if nranks < 1 or nranks > nz:
        raise ValueError(f"cannot split {nz} cell layers over {nranks} ranks")
    b = [(r * nz) // nranks for r in range(nranks + 1)]
    return [(b[r], b[r + 1]) for r in range(nranks)]


def dof_owner(pb, nranks: int) -> np.ndarray:
    """Owning rank of every dof of a generated problem (problems.Problem)."""
    bounds = slab_bounds(pb.nz, nranks)
    zcell_owner = np.empty(pb.nz, dtype=np.int32)
    for r, (z0, z1) in enumerate(bounds):
        zcell_owner[z0:z1] = r
    # node plane k belongs to the rank owning cell layer k (top plane -> last rank)
    znode_owner = np.empty(pb.nz + 1, dtype=np.int32)
    znode_owner[:pb.nz] = zcell_owner
    znode_owner[pb.nz] = nranks - 1
    n_u = pb.n_u
    owner = np.empty(pb.n, dtype=np.int32)
    node = pb.entity_of[:n_u].astype(np.int64)
    owner[:n_u] = znode_owner[node // ((pb.nx + 1) * (pb.ny + 1))]
    cell = pb.entity_of[n_u:].astype(np.int64)
    owner[n_u:] = zcell_owner[cell // (pb.nx * pb.ny)]
    return owner


@dataclass
class HaloPlan:
    """What rank `rank` owns, what it must receive, and what it must send."""

    rank: int
    nranks: int
    owned: np.ndarray                    # global ids, ascending
    ghosts: np.ndarray                   # global ids needed but not owned, ascending
    recv_from: dict = field(default_factory=dict)   # peer -> positions in ghosts (ascending global id)
    send_to: dict = field(default_factory=dict)     # peer -> local owned indices to send
    # local CSR over owned rows; columns index [owned | ghosts]
    ro: np.ndarray = None
    ci: np.ndarray = None
    v: np.ndarray = None

    @property
    def n_own(self) -> int:
        return len(self.owned)

    @property
    def n_ext(self) -> int:
        return len(self.owned) + len(self.ghosts)


def build_halo_plan(ro, ci, v, owner: np.ndarray, rank: int, nranks: int) -> HaloPlan:
    """Local rows, ghost columns and the send/recv lists of one rank.

    The send lists are derived symmetrically (every rank computes what each
    peer needs from it), so no communication is needed to build the plan.
    """
    ro = np.asarray(ro, dtype=np.int64)
    ci = np.asarray(ci, dtype=np.int64)
    owned = np.flatnonzero(owner == rank)
    gl2own = np.full(len(owner), -1, dtype=np.int64)
    gl2own[owned] = np.arange(len(owned))
    starts, ends = ro[owned], ro[owned + 1]
    cnt = ends - starts
    take = np.repeat(starts - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt) + np.arange(cnt.sum())
    cols = ci[take]
    ghosts = np.unique(cols[owner[cols] != rank])
    plan = HaloPlan(rank, nranks, owned, ghosts)
    gpos = np.searchsorted(ghosts, cols)
    local = np.where(owner[cols] == rank, gl2own[cols], len(owned) + gpos)
    plan.ro = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    plan.ci = local.astype(np.int32)
    plan.v = np.asarray(v)[take] if v is not None else None
    for peer in range(nranks):
        if peer == rank:
            continue
        mine = np.flatnonzero(owner[ghosts] == peer)
        if len(mine):
            plan.recv_from[peer] = mine
        # what `peer` needs from me: ghosts of peer that I own, ascending
        p_owned = np.flatnonzero(owner == peer)
        p_cnt = ro[p_owned + 1] - ro[p_owned]
        p_take = np.repeat(ro[p_owned] - np.concatenate([[0], np.cumsum(p_cnt)[:-1]]), p_cnt) + np.arange(p_cnt.sum())
        p_cols = np.unique(ci[p_take])
        need = p_cols[owner[p_cols] == rank]
        if len(need):
            plan.send_to[peer] = gl2own[need]
    return plan


def halo_exchange(x_ext, plan: HaloPlan, dist, group=None):
    """Fill the ghost part of x_ext (torch tensor of length n_ext) from the
    owning ranks: one isend/irecv pair per neighbour."""
    import torch

    n = plan.n_own
    reqs, bufs = [], []
    for peer, idx in plan.recv_from.items():
        buf = torch.empty(len(idx), dtype=x_ext.dtype, device=x_ext.device)
        bufs.append((peer, idx, buf))
        reqs.append(dist.irecv(buf, src=peer, group=group))
    for peer, idx in plan.send_to.items():
        sidx = torch.as_tensor(idx, device=x_ext.device)
        reqs.append(dist.isend(x_ext[:n].index_select(0, sidx).contiguous(), dst=peer, group=group))
    for r in reqs:
        r.wait()
    for peer, idx, buf in bufs:
        x_ext[n + torch.as_tensor(idx, device=x_ext.device)] = buf
    return x_ext


def dist_dots(V_rows, w, dist, group=None):
    """Global dot products of the rows of V with w (one all-reduce)."""
    import torch

    local = V_rows @ w
    dist.all_reduce(local, group=group)
    return local


def dist_norm(w, dist, group=None) -> float:
    import torch

    s = torch.dot(w, w).reshape(1)
    dist.all_reduce(s, group=group)
    return float(torch.sqrt(s))


class DistOperator:
    """v (owned part) -> A v (owned rows) with a halo exchange first."""

    def __init__(self, plan: HaloPlan, local_matvec, dist, group=None):
        self.plan, self.local_matvec, self.dist, self.group = plan, local_matvec, dist, group

    def __call__(self, v_own):
        import torch

        x_ext = torch.zeros(self.plan.n_ext, dtype=v_own.dtype, device=v_own.device)
        x_ext[:self.plan.n_own] = v_own
        halo_exchange(x_ext, self.plan, self.dist, self.group)
        return self.local_matvec(x_ext)


class DistVectors:
    """krylov.gmres_loop's vector algebra on row-distributed slices: local
    torch arithmetic plus one all-reduce per projection pass / norm."""

    def __init__(self, dist, group, like):
        self.dist, self.group, self.like = dist, group, like

    def zeros(self, shape):
        import torch

        return torch.zeros(shape, dtype=self.like.dtype, device=self.like.device)

    def norm(self, v) -> float:
        return dist_norm(v, self.dist, self.group)

    def axpby(self, a, x, b, y):
        if b == 0.0:
            y.copy_(x).mul_(a)
        else:
            y.mul_(b).add_(x, alpha=a)
        return y

    def project(self, V, k, w):
        h = np.zeros(k)
        for _ in range(2):  # CGS2, one all-reduce per pass
            c = dist_dots(V[:k], w, self.dist, self.group)
            w -= c @ V[:k]
            h += c.cpu().numpy()
        return h

    def combine(self, V, j, y):
        import torch

        return torch.as_tensor(y, dtype=V.dtype, device=V.device) @ V[:j]


def dist_gmres(apply_A, apply_M_inv, b, dist, group=None, restart=50, max_iters=500, rtol=1e-6, atol=1e-12):
    """Right-preconditioned restarted GMRES (reference krylov.py:39-117) on
    row-distributed vectors: krylov.gmres_loop with classical Gram-Schmidt
    plus one re-orthogonalisation (one all-reduce per pass); the small
    Hessenberg algebra is replicated on every rank."""
    from .krylov import gmres_loop

    return gmres_loop(DistVectors(dist, group, b), apply_A, apply_M_inv, b, b.new_zeros(b.numel()), False,
                      restart, max_iters, rtol, atol)


# ---------------------------------------------------------------------------
# device path: libpmgr's row distribution (include/pmgr.h, csrc/dist.cu)
# ---------------------------------------------------------------------------
#
# Every rank builds the global hierarchy of a rank-major numbered problem
# (problems.rank_major) on its own GPU, then keeps its rows of every
# operator.  Vectors are the rank's owned slices (float64 CUDA tensors).


def nccl_transport(rank: int, nranks: int, dist):
    """NCCL communicator inside libpmgr; the unique id travels through the
    caller's torch.distributed process group (any backend)."""
    from . import _lib

    L = _lib.lib()
    nid = _lib.NcclId()
    if rank == 0:
        _lib.check(L.pmgr_nccl_get_id(ctypes.byref(nid)))
    if nranks > 1:
        box = [ctypes.string_at(ctypes.addressof(nid), 128) if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        ctypes.memmove(ctypes.addressof(nid), box[0], 128)
    out = ctypes.c_void_p()
    _lib.check(L.pmgr_transport_nccl_create(ctypes.byref(nid), rank, nranks, ctypes.byref(out)))
    return _Handle(out, "pmgr_transport_destroy")


def host_transport(rank: int, nranks: int, dist, group=None):
    """Host-staged transport inside libpmgr over the caller's torch.distributed
    group (any backend with point-to-point and all_reduce, e.g. gloo): every
    exchange stages through host memory and synchronises, so several
    processes may share one GPU.  Used by the multi-process tests."""
    import torch

    from . import _lib

    def a2a(_ctx, sptr, sbytes, rptr, rbytes):
        try:
            reqs, keep = [], []
            for p in range(nranks):
                if p == rank:
                    continue
                if sbytes[p] > 0:
                    buf = (ctypes.c_uint8 * sbytes[p]).from_address(sptr[p])
                    t = torch.frombuffer(buf, dtype=torch.uint8)
                    keep.append(t)
                    reqs.append(dist.isend(t, dst=p, group=group))
                if rbytes[p] > 0:
                    buf = (ctypes.c_uint8 * rbytes[p]).from_address(rptr[p])
                    t = torch.frombuffer(buf, dtype=torch.uint8)
                    keep.append(t)
                    reqs.append(dist.irecv(t, src=p, group=group))
            for r in reqs:
                r.wait()
            return 0
        except Exception:  # noqa: BLE001 -- reported as a library error
            import traceback

            traceback.print_exc()
            return 1

    def ared(_ctx, buf, n):
        try:
            arr = (ctypes.c_double * n).from_address(ctypes.addressof(buf.contents))
            t = torch.frombuffer(arr, dtype=torch.float64)
            dist.all_reduce(t, group=group)
            return 0
        except Exception:  # noqa: BLE001
            import traceback

            traceback.print_exc()
            return 1

    fa, fr = _lib.ALLTOALLV_FN(a2a), _lib.ALLREDUCE_FN(ared)
    out = ctypes.c_void_p()
    _lib.check(_lib.lib().pmgr_transport_host_create(rank, nranks, ctypes.cast(fa, ctypes.c_void_p),
                                                     ctypes.cast(fr, ctypes.c_void_p), None, ctypes.byref(out)))
    h = _Handle(out, "pmgr_transport_destroy")
    h._callbacks = (fa, fr)  # keep the trampolines alive with the transport
    return h


class _Handle:
    def __init__(self, h, destroy):
        self.h, self._destroy = h, destroy

    def __del__(self):
        from . import _lib

        if sys.is_finalizing():  # the process is exiting: the driver reclaims everything
            return
        if getattr(self, "h", None) and _lib is not None and _lib._lib is not None:
            getattr(_lib._lib, self._destroy)(self.h)
            self.h = None


class DeviceDistSolver:
    """Rank `rank`'s slice of an MgrHierarchy (and its matrix) for the
    distributed solve: `apply` / `spmv` / `gmres` on owned slices."""

    def __init__(self, h, bounds, rank: int, nranks: int, transport=None):
        from . import _lib
        from .sparse import current_stream

        self.h, self.rank, self.nranks = h, rank, nranks
        self.transport = transport
        self.bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        if len(self.bounds) != nranks + 1:
            raise ValueError("bounds must have nranks + 1 entries")
        out = ctypes.c_void_p()
        th = transport.h if transport is not None else None
        _lib.check(_lib.lib().pmgr_dist_create(h._A.handle, h.handle, self.bounds.ctypes.data, rank, nranks, th,
                                               current_stream(), ctypes.byref(out)))
        self._d = _Handle(out, "pmgr_dist_destroy")
        lo, no = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().pmgr_dist_info(self._d.h, ctypes.byref(lo), ctypes.byref(no)))
        self.lo, self.n_own = lo.value, no.value

    def _vec(self, v):
        from .sparse import to_device

        return to_device(v, self.n_own).contiguous()

    def apply(self, v_own):
        from . import _lib
        from .sparse import current_stream, empty_device, ptr

        v = self._vec(v_own)
        z = empty_device(self.n_own)
        _lib.check(_lib.lib().pmgr_dist_apply(self._d.h, ptr(v), ptr(z), current_stream()))
        return z

    def spmv(self, x_own):
        from . import _lib
        from .sparse import current_stream, empty_device, ptr

        x = self._vec(x_own)
        y = empty_device(self.n_own)
        _lib.check(_lib.lib().pmgr_dist_spmv(self._d.h, ptr(x), ptr(y), current_stream()))
        return y

    def gmres(self, b_own, cfg=None):
        from . import _lib
        from .krylov import GmresConfig, SolveStats
        from .sparse import current_stream, empty_device, ptr

        cfg = cfg or GmresConfig()
        b = self._vec(b_own)
        x = empty_device(self.n_own).zero_()
        c = _lib.GmresCfg(int(cfg.restart), int(cfg.max_iters), float(cfg.rtol), float(cfg.atol))
        st = _lib.GmresStats()
        cap = int(cfg.max_iters) + 2
        hist = np.zeros(cap)
        _lib.check(_lib.lib().pmgr_dist_gmres(self._d.h, ptr(b), ptr(x), 0, ctypes.byref(c), ctypes.byref(st),
                                              hist.ctypes.data, cap, current_stream()))
        return x, SolveStats(int(st.iterations), hist[:st.history_len].copy(), bool(st.converged))


def row_slice(A, lo: int, hi: int):
    """Rows [lo, hi) of A in A's global row space, every other row empty (a
    rank's input to the distributed setup), as a device matrix."""
    from . import _lib
    from .sparse import DeviceCsr, as_device_csr, current_stream

    dA = as_device_csr(A)
    out = ctypes.c_void_p()
    _lib.check(_lib.lib().pmgr_csr_rows(dA.handle, int(lo), int(hi), current_stream(), ctypes.byref(out)))
    nr, nc, nz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.lib().pmgr_csr_info(out, ctypes.byref(nr), ctypes.byref(nc), ctypes.byref(nz)))
    return DeviceCsr(out, nr.value, nc.value, nz.value)


class DeviceDistSetupSolver(DeviceDistSolver):
    """Rank `rank`'s solver from the DISTRIBUTED setup (pmgr_dist_setup):
    `A_rows` holds only this rank's rows (global row space), the layout is
    global; every rank calls this collectively.  Each rank builds the owned
    rows of every operator of the hierarchy (bitwise equal to the single-GPU
    setup) and the small coarse levels redundantly."""

    def __init__(self, A_rows, layout, config, bounds, rank: int, nranks: int, transport=None):
        from . import _lib
        from .mgr import setup_args
        from .sparse import as_device_csr, current_stream

        self.h, self.rank, self.nranks = None, rank, nranks
        self.transport = transport
        self.bounds = np.ascontiguousarray(bounds, dtype=np.int64)
        if len(self.bounds) != nranks + 1:
            raise ValueError("bounds must have nranks + 1 entries")
        dA = as_device_csr(A_rows)
        self._A = dA
        specs, cfg, fo0, eo0 = setup_args(dA, layout, config)
        out = ctypes.c_void_p()
        th = transport.h if transport is not None else None
        _lib.check(_lib.lib().pmgr_dist_setup(dA.handle, fo0.ctypes.data, eo0.ctypes.data, specs,
                                              len(config.levels), ctypes.byref(cfg), self.bounds.ctypes.data,
                                              rank, nranks, th, current_stream(), ctypes.byref(out)))
        self._d = _Handle(out, "pmgr_dist_destroy")
        lo, no = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.lib().pmgr_dist_info(self._d.h, ctypes.byref(lo), ctypes.byref(no)))
        self.lo, self.n_own = lo.value, no.value


def _emulate_setup(A, layout, config, bounds, what, vin, cfg=None):
    from . import _lib
    from .krylov import GmresConfig
    from .mgr import setup_args
    from .sparse import as_device_csr, current_stream, empty_device, ptr, to_device

    dA = as_device_csr(A)
    specs, mcfg, fo0, eo0 = setup_args(dA, layout, config)
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    vd = to_device(vin, dA.nrows).contiguous()
    z = empty_device(dA.nrows).zero_()
    c = st = None
    if what == 1:
        cfg = cfg or GmresConfig()
        c = _lib.GmresCfg(int(cfg.restart), int(cfg.max_iters), float(cfg.rtol), float(cfg.atol))
        st = _lib.GmresStats()
    _lib.check(_lib.lib().pmgr_dist_setup_emulate(dA.handle, fo0.ctypes.data, eo0.ctypes.data, specs,
                                                  len(config.levels), ctypes.byref(mcfg), b.ctypes.data, len(b) - 1,
                                                  what, ptr(vd), ptr(z), ctypes.byref(c) if c else None,
                                                  ctypes.byref(st) if st else None, current_stream()))
    return z, st


def emulate_setup_apply(A, layout, config, bounds, v):
    """z = M v where M comes from the distributed setup over len(bounds)-1
    ranks emulated on this GPU (each rank sets up from its row slice)."""
    return _emulate_setup(A, layout, config, bounds, 0, v)[0]


def emulate_setup_gmres(A, layout, config, bounds, rhs, cfg=None):
    """Distributed setup + distributed GMRES(MGR) from x0 = 0 over emulated ranks."""
    x, st = _emulate_setup(A, layout, config, bounds, 1, rhs, cfg)
    return x, int(st.iterations), bool(st.converged)


def emulate_apply(h, bounds, v):
    """z = M v with the hierarchy row-distributed over len(bounds)-1 ranks
    emulated on this GPU (loopback transport): the parity harness of §8e."""
    from . import _lib
    from .sparse import current_stream, empty_device, ptr, to_device

    b = np.ascontiguousarray(bounds, dtype=np.int64)
    vd = to_device(v, h.n).contiguous()
    z = empty_device(h.n)
    _lib.check(_lib.lib().pmgr_dist_emulate(h._A.handle, h.handle, b.ctypes.data, len(b) - 1, 0, ptr(vd), ptr(z),
                                            None, None, current_stream()))
    return z


def emulate_gmres(h, bounds, rhs, cfg=None):
    """Distributed GMRES(MGR) from x0 = 0 over emulated ranks; returns the
    gathered solution and the iteration count / convergence flag."""
    from . import _lib
    from .krylov import GmresConfig
    from .sparse import current_stream, empty_device, ptr, to_device

    cfg = cfg or GmresConfig()
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    bd = to_device(rhs, h.n).contiguous()
    x = empty_device(h.n).zero_()
    c = _lib.GmresCfg(int(cfg.restart), int(cfg.max_iters), float(cfg.rtol), float(cfg.atol))
    st = _lib.GmresStats()
    _lib.check(_lib.lib().pmgr_dist_emulate(h._A.handle, h.handle, b.ctypes.data, len(b) - 1, 1, ptr(bd), ptr(x),
                                            ctypes.byref(c), ctypes.byref(st), current_stream()))
    return x, int(st.iterations), bool(st.converged)
