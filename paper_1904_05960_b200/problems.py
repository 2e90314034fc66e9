"""Seeded synthetic poromechanics Jacobians for the BASELINE.json configs.

The reference ships no assembler (SPEC `poromech`, is absent
from the code), so this host-side NumPy generator stands in for it.  It is an
input fixture, not part of the timed path.  It follows SURVEY.md §8(d):

* layout: displacement dofs node-blocked first (dof = 3*node + component,
  node = i + (nx+1)*(j + (ny+1)*k)), then flow dofs interleaved per cell
  (cell = i + nx*(j + ny*k)), exactly the ordering SPEC.md:500 prescribes;
* mechanics: trilinear (Q1) hexahedra, 2x2x2 Gauss, isotropic elasticity with
  per-cell Young's modulus E and Poisson ratio 0.25 (K_e = E * K_ref);
* flow: cell-centred TPFA with harmonic transmissibilities, first-order
  upwinding by a seeded "linear plus noise" pressure state, Corey quadratic
  (two-phase) or Stone-I-like (three-phase) mobilities;
* coupling: Biot b=1, A_up = -b * int(div N_u) per cell, the mass rows get
  +b * S_l * int(div N_u) / dt ("A_pu = -A_up^T" up to 1/dt);
* Dirichlet: bottom-face displacement rows replaced by identity rows, columns
  kept ("impose Dirichlet on rows only");
* randomness: one seed, spawned with SeedSequence into independent streams
  in the fixed order E, perm, saturation, pressure noise, RHS.

Every row's column indices come out strictly increasing, so the arrays are a
valid reference `CsrMatrix` (sparse.py:65-101) without sorting.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

FIELD_U = 0
FIELD_S = 1      # wetting saturation (S_1 in the three-phase config)
FIELD_P = 2
FIELD_S2 = 3     # second saturation (three-phase config only)

# (dz, dy, dx) in lexicographic order => ascending neighbour node id
_OFFSETS27 = np.array([(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)])


@dataclass
class Problem:
    """One seeded linear system A x = b with its field layout."""

    name: str
    nx: int
    ny: int
    nz: int
    row_offsets: np.ndarray   # int64, n+1
    col_indices: np.ndarray   # int32, nnz
    values: np.ndarray        # float64, nnz
    field_of: np.ndarray      # int8, n
    entity_of: np.ndarray     # int32, n
    rhs: np.ndarray           # float64, n
    cell_fields: tuple        # per-cell flow field tags in dof order
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return len(self.row_offsets) - 1

    @property
    def nnz(self) -> int:
        return len(self.values)

    @property
    def n_u(self) -> int:
        return 3 * (self.nx + 1) * (self.ny + 1) * (self.nz + 1)


# ---------------------------------------------------------------------------
# element matrices
# ---------------------------------------------------------------------------


def element_matrices(h: float, nu: float):
    """Unit-E Q1 stiffness K_ref (24x24) and Biot vector int(dN_l/dx_a) (24,).

    Local node ln = a + 2b + 4c for corner offsets (a, b, c); dof 3*ln + comp.
    """
    gp = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
    lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = 1.0 / (2.0 * (1.0 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[0, 0] += 2 * mu
    D[1, 1] += 2 * mu
    D[2, 2] += 2 * mu
    D[3, 3] = D[4, 4] = D[5, 5] = mu
    K = np.zeros((24, 24))
    bvec = np.zeros(24)
    w = h ** 3 / 8.0
    for gz in gp:
        for gy in gp:
            for gx in gp:
                dN = np.zeros((8, 3))
                for ln in range(8):
                    a, b, c = ln & 1, (ln >> 1) & 1, (ln >> 2) & 1
                    fx, dfx = (gx, 1.0) if a else (1.0 - gx, -1.0)
                    fy, dfy = (gy, 1.0) if b else (1.0 - gy, -1.0)
                    fz, dfz = (gz, 1.0) if c else (1.0 - gz, -1.0)
                    dN[ln] = np.array([dfx * fy * fz, fx * dfy * fz, fx * fy * dfz]) / h
                B = np.zeros((6, 24))
                for ln in range(8):
                    B[0, 3 * ln] = dN[ln, 0]
                    B[1, 3 * ln + 1] = dN[ln, 1]
                    B[2, 3 * ln + 2] = dN[ln, 2]
                    B[3, 3 * ln] = dN[ln, 1]
                    B[3, 3 * ln + 1] = dN[ln, 0]
                    B[4, 3 * ln + 1] = dN[ln, 2]
                    B[4, 3 * ln + 2] = dN[ln, 1]
                    B[5, 3 * ln] = dN[ln, 2]
                    B[5, 3 * ln + 2] = dN[ln, 0]
                K += w * (B.T @ D @ B)
                bvec += w * dN.ravel()
    return K, bvec


# ---------------------------------------------------------------------------
# random fields
# ---------------------------------------------------------------------------


def _gaussian_smooth2d(noise, corr):
    from scipy.ndimage import gaussian_filter

    f = gaussian_filter(noise, sigma=corr, mode="wrap")
    s = f.std()
    return (f - f.mean()) / (s if s > 0 else 1.0)


def _layered_logperm(rng, nx, ny, nz, layer, corr):
    """Per-cell N(0,1) log-field, constant over z-layers of `layer` cells,
    smoothed in (x, y) with a Gaussian filter of length `corr` cells."""
    nlay = (nz + layer - 1) // layer
    out = np.empty((nz, ny, nx))
    for L in range(nlay):
        f = _gaussian_smooth2d(rng.standard_normal((ny, nx)), corr)
        out[L * layer:(L + 1) * layer] = f[None]
    return out


# ---------------------------------------------------------------------------
# mobility models
# ---------------------------------------------------------------------------


def _mobilities(kind, sats, mu):
    """Phase mobilities and their derivatives w.r.t. the saturation unknowns.

    sats: (nsat, ...) unknown saturations.  Returns lam (nph, ...) and
    dlam (nph, nsat, ...), phases ordered as the mass equations.
    """
    if kind == "single":
        one = np.ones(sats.shape[1:]) if sats.ndim > 1 else np.ones(())
        return one[None], np.zeros((1, 0) + one.shape)
    if kind == "two":
        s = sats[0]
        # Corey quadratic, zero residuals: krw=s^2, kro=(1-s)^2
        lw = s * s / mu[0]
        lo = (1.0 - s) ** 2 / mu[1]
        dlw = 2.0 * s / mu[0]
        dlo = -2.0 * (1.0 - s) / mu[1]
        return np.stack([lw, lo]), np.stack([dlw[None], dlo[None]])
    # three-phase (water, gas, oil); unknowns (s_w, s_g); Stone-I-like oil
    sw, sg = sats[0], sats[1]
    so = 1.0 - sw - sg
    krw, krg = sw * sw, sg * sg
    kro = so * (1.0 - sw) * (1.0 - sg)
    dkro_dsw = -(1.0 - sw) * (1.0 - sg) - so * (1.0 - sg)
    dkro_dsg = -(1.0 - sw) * (1.0 - sg) - so * (1.0 - sw)
    z = np.zeros_like(sw)
    lam = np.stack([krw / mu[0], krg / mu[1], kro / mu[2]])
    dlam = np.stack([
        np.stack([2 * sw / mu[0], z]),
        np.stack([z, 2 * sg / mu[1]]),
        np.stack([dkro_dsw / mu[2], dkro_dsg / mu[2]]),
    ])
    return lam, dlam


# ---------------------------------------------------------------------------
# assembly
# ---------------------------------------------------------------------------


def assemble(nx, ny, nz, *, E, kx, ky, kz, phases="single", sats=None,
             pstate=None, mu=(1.0,), phi=0.2, ct=1e-3, dt=1.0, biot=1.0,
             nu=0.25, h=None, rhs_rng=None, name="custom"):
    """Assemble the coupled Jacobian on an nx*ny*nz cube-cell grid.

    E, kx, ky, kz: per-cell arrays shaped (nz, ny, nx).  sats: (nsat, nz, ny, nx)
    unknown saturations (two-phase: s_w; three-phase: s_w, s_g).  pstate:
    (nz, ny, nx) pressure state used only for upwind directions and
    potential differences.
    """
    if h is None:
        h = 1.0 / max(nx, ny)
    NX, NY, NZ = nx + 1, ny + 1, nz + 1
    nn = NX * NY * NZ
    nc = nx * ny * nz
    n_u = 3 * nn
    if phases == "single":
        cell_fields = (FIELD_P,)
    elif phases == "two":
        cell_fields = (FIELD_S, FIELD_P)
    else:
        cell_fields = (FIELD_S, FIELD_S2, FIELD_P)
    nf = len(cell_fields)
    p_slot = nf - 1          # pressure is the last unknown of each cell
    nsat = nf - 1
    n = n_u + nf * nc

    K0, bvec = element_matrices(h, nu)

    # ---- displacement rows: 27 neighbour nodes x 3 comps, then 8 cells x nf
    Ep = np.zeros((nz + 2, ny + 2, nx + 2))
    Ep[1:-1, 1:-1, 1:-1] = E
    kk, jj, ii = np.meshgrid(np.arange(NZ), np.arange(NY), np.arange(NX), indexing="ij")
    uu = np.zeros((NZ, NY, NX, 27, 3, 3))
    uvalid = np.zeros((NZ, NY, NX, 27), dtype=bool)
    ucol_node = np.zeros((NZ, NY, NX, 27), dtype=np.int64)
    for o, (dz, dy, dx) in enumerate(_OFFSETS27):
        mi, mj, mk = ii + dx, jj + dy, kk + dz
        uvalid[..., o] = (mi >= 0) & (mi < NX) & (mj >= 0) & (mj < NY) & (mk >= 0) & (mk < NZ)
        ucol_node[..., o] = mi + NX * (mj + NY * mk)
        for ck in (0, 1):
            for cj in (0, 1):
                for ci in (0, 1):
                    lx, ly, lz = 1 - ci, 1 - cj, 1 - ck
                    mx, my, mz = lx + dx, ly + dy, lz + dz
                    if not (0 <= mx <= 1 and 0 <= my <= 1 and 0 <= mz <= 1):
                        continue
                    ln = lx + 2 * ly + 4 * lz
                    lm = mx + 2 * my + 4 * mz
                    blk = K0[3 * ln:3 * ln + 3, 3 * lm:3 * lm + 3]
                    Es = Ep[ck:ck + NZ, cj:cj + NY, ci:ci + NX]
                    uu[..., o, :, :] += Es[..., None, None] * blk
    # coupling of displacement rows to the pressure of the 8 adjacent cells
    ucell = np.zeros((NZ, NY, NX, 8), dtype=np.int64)
    ucell_valid = np.zeros((NZ, NY, NX, 8), dtype=bool)
    ucoup = np.zeros((NZ, NY, NX, 8, 3))
    q = 0
    for ck in (0, 1):
        for cj in (0, 1):
            for ci in (0, 1):
                ci_, cj_, ck_ = ii - 1 + ci, jj - 1 + cj, kk - 1 + ck
                ok = (ci_ >= 0) & (ci_ < nx) & (cj_ >= 0) & (cj_ < ny) & (ck_ >= 0) & (ck_ < nz)
                ucell_valid[..., q] = ok
                ucell[..., q] = ci_ + nx * (cj_ + ny * ck_)
                ln = (1 - ci) + 2 * (1 - cj) + 4 * (1 - ck)
                ucoup[..., q, :] = -biot * bvec[3 * ln:3 * ln + 3]
                q += 1

    Wu = 27 * 3 + 8 * nf
    ucols = np.empty((nn, 3, Wu), dtype=np.int64)
    uvals = np.zeros((nn, 3, Wu))
    umask = np.zeros((nn, 3, Wu), dtype=bool)
    cn = ucol_node.reshape(nn, 27)
    ucols[:, :, :81] = (3 * cn[:, None, :, None] + np.arange(3)[None, None, None, :]).reshape(nn, 1, 81)
    uvals[:, :, :81] = uu.reshape(nn, 27, 3, 3).transpose(0, 2, 1, 3).reshape(nn, 3, 81)
    umask[:, :, :81] = np.repeat(uvalid.reshape(nn, 27), 3, axis=1)[:, None, :]
    cc = ucell.reshape(nn, 8)
    ucols[:, :, 81:] = (n_u + nf * cc[:, None, :, None] + np.arange(nf)[None, None, None, :]).reshape(nn, 1, 8 * nf)
    cv = np.zeros((nn, 3, 8, nf))
    cv[..., p_slot] = ucoup.reshape(nn, 8, 3).transpose(0, 2, 1)
    uvals[:, :, 81:] = cv.reshape(nn, 3, 8 * nf)
    cm = np.zeros((nn, 8, nf), dtype=bool)
    cm[..., p_slot] = ucell_valid.reshape(nn, 8)
    umask[:, :, 81:] = cm.reshape(nn, 1, 8 * nf)
    # Dirichlet (rows only): bottom node plane -> identity rows
    bottom = np.arange(NX * NY)
    umask[bottom] = False
    uvals[bottom] = 0.0
    diag_slot = 13 * 3  # offset (0,0,0) is index 13; + component b == a
    for a in range(3):
        umask[bottom, a, diag_slot + a] = True
        uvals[bottom, a, diag_slot + a] = 1.0
    del uu, ucol_node, uvalid

    # ---- flow rows: 8 cell nodes x 3 comps, then 7-point cells x nf
    ck3, cj3, ci3 = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    V = h ** 3
    if phases == "single":
        lam = np.ones((1, nz, ny, nx))
        dlam = np.zeros((1, 0, nz, ny, nx))
        Sph = np.ones((1, nz, ny, nx))
        dS = np.zeros((1, 0))
    else:
        lam, dlam = _mobilities(phases, sats, mu)
        if phases == "two":
            Sph = np.stack([sats[0], 1.0 - sats[0]])
            dS = np.array([[1.0], [-1.0]])
        else:
            Sph = np.stack([sats[0], sats[1], 1.0 - sats[0] - sats[1]])
            dS = np.array([[1.0, 0.0], [0.0, 1.0], [-1.0, -1.0]])
    neq = nf
    # Jf[eq, slot(7), field, z, y, x]; slots -z,-y,-x,self,+x,+y,+z
    Jf = np.zeros((neq, 7, nf, nz, ny, nx))
    for e in range(neq):
        for f in range(nsat):
            Jf[e, 3, f] += V * phi / dt * dS[e, f]
        Jf[e, 3, p_slot] += V * phi * Sph[e] * ct / dt
    fvalid = np.ones((7, nz, ny, nx), dtype=bool)
    fvalid[0, 0] = False
    fvalid[6, -1] = False
    fvalid[1, :, 0] = False
    fvalid[5, :, -1] = False
    fvalid[2, :, :, 0] = False
    fvalid[4, :, :, -1] = False
    for axis, kdir, sK, sL in ((2, kx, 4, 2), (1, ky, 5, 1), (0, kz, 6, 0)):
        # faces between K (lower) and L (upper) along this axis
        sl_K = [slice(None)] * 3
        sl_L = [slice(None)] * 3
        sl_K[axis] = slice(0, -1)
        sl_L[axis] = slice(1, None)
        sl_K, sl_L = tuple(sl_K), tuple(sl_L)
        tK = 2.0 * kdir[sl_K] * h
        tL = 2.0 * kdir[sl_L] * h
        T = tK * tL / (tK + tL)
        dphi = pstate[sl_K] - pstate[sl_L]
        upK = dphi >= 0.0
        for e in range(neq):
            lup = np.where(upK, lam[e][sl_K], lam[e][sl_L])
            g = T * lup
            # row K (+F) and row L (-F), pressure derivatives
            Jf[(e, 3, p_slot) + sl_K] += g
            Jf[(e, sK, p_slot) + sl_K] -= g
            Jf[(e, 3, p_slot) + sl_L] += g
            Jf[(e, sL, p_slot) + sl_L] -= g
            for f in range(nsat):
                dK = T * dlam[e, f][sl_K] * dphi
                dL = T * dlam[e, f][sl_L] * dphi
                Jf[(e, 3, f) + sl_K] += np.where(upK, dK, 0.0)
                Jf[(e, sK, f) + sl_K] += np.where(upK, 0.0, dL)
                Jf[(e, sL, f) + sl_L] -= np.where(upK, dK, 0.0)
                Jf[(e, 3, f) + sl_L] -= np.where(upK, 0.0, dL)
    # neighbour cell ids per slot
    nbr = np.stack([
        ci3 + nx * (cj3 + ny * (ck3 - 1)),
        ci3 + nx * (cj3 - 1 + ny * ck3),
        ci3 - 1 + nx * (cj3 + ny * ck3),
        ci3 + nx * (cj3 + ny * ck3),
        ci3 + 1 + nx * (cj3 + ny * ck3),
        ci3 + nx * (cj3 + 1 + ny * ck3),
        ci3 + nx * (cj3 + ny * (ck3 + 1)),
    ])
    # Biot coupling of the mass rows to the 8 cell nodes
    cnode = np.zeros((8, nz, ny, nx), dtype=np.int64)
    for ln in range(8):
        a, b, c = ln & 1, (ln >> 1) & 1, (ln >> 2) & 1
        cnode[ln] = (ci3 + a) + NX * ((cj3 + b) + NY * (ck3 + c))

    Wf = 24 + 7 * nf
    fcols = np.empty((nc, neq, Wf), dtype=np.int64)
    fvals = np.zeros((nc, neq, Wf))
    fmask = np.zeros((nc, neq, Wf), dtype=bool)
    cn8 = cnode.reshape(8, nc).T  # (nc, 8)
    fcols[:, :, :24] = (3 * cn8[:, None, :, None] + np.arange(3)[None, None, None, :]).reshape(nc, 1, 24)
    fmask[:, :, :24] = True
    for e in range(neq):
        coef = (biot * Sph[e] / dt).reshape(nc)
        fvals[:, e, :24] = coef[:, None] * bvec[None, :]
    nb = nbr.reshape(7, nc).T  # (nc, 7)
    fcols[:, :, 24:] = (n_u + nf * nb[:, None, :, None] + np.arange(nf)[None, None, None, :]).reshape(nc, 1, 7 * nf)
    fvals[:, :, 24:] = Jf.reshape(neq, 7, nf, nc).transpose(3, 0, 1, 2).reshape(nc, neq, 7 * nf)
    fm = np.repeat(fvalid.reshape(7, nc).T[:, :, None], nf, axis=2)  # (nc, 7, nf)
    fmask[:, :, 24:] = fm.reshape(nc, 1, 7 * nf)
    del Jf

    um = umask.reshape(n_u, Wu)
    fm2 = fmask.reshape(nf * nc, Wf)
    counts = np.concatenate([um.sum(axis=1), fm2.sum(axis=1)])
    ro = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=ro[1:])
    ci = np.concatenate([ucols.reshape(n_u, Wu)[um], fcols.reshape(nf * nc, Wf)[fm2]]).astype(np.int32)
    va = np.concatenate([uvals.reshape(n_u, Wu)[um], fvals.reshape(nf * nc, Wf)[fm2]])
    del ucols, uvals, umask, fcols, fvals, fmask

    field_of = np.concatenate([np.full(n_u, FIELD_U, dtype=np.int8),
                               np.tile(np.array(cell_fields, dtype=np.int8), nc)])
    entity_of = np.concatenate([(np.arange(n_u) // 3).astype(np.int32),
                                np.repeat(np.arange(nc, dtype=np.int32), nf)])
    rhs = rhs_rng.standard_normal(n) if rhs_rng is not None else np.zeros(n)
    return Problem(name, nx, ny, nz, ro, ci, va, field_of, entity_of, rhs, cell_fields,
                   dict(h=h, dt=dt, phases=phases))


@dataclass
class DeviceProblem:
    """A generated system whose matrix was assembled on the GPU (libpmgr,
    SURVEY.md §8f row 3): `A` is a sparse.DeviceCsr; layout and rhs on the host."""

    name: str
    nx: int
    ny: int
    nz: int
    A: object
    field_of: np.ndarray
    entity_of: np.ndarray
    rhs: np.ndarray
    cell_fields: tuple
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.A.nrows

    @property
    def nnz(self) -> int:
        return self.A.nnz

    @property
    def n_u(self) -> int:
        return 3 * (self.nx + 1) * (self.ny + 1) * (self.nz + 1)


def assemble_device(nx, ny, nz, *, E, kx, ky, kz, phases="single", sats=None,
                    pstate=None, mu=(1.0,), phi=0.2, ct=1e-3, dt=1.0, biot=1.0,
                    nu=0.25, h=None, rhs_rng=None, name="custom") -> DeviceProblem:
    """`assemble` with the matrix built on the device (pmgr_assemble_poromech):
    same arguments, bitwise the same CSR, no host matrix and no host-to-device
    copy of it (only the per-cell fields travel)."""
    import ctypes

    from . import _lib
    from .sparse import DeviceCsr, current_stream

    if h is None:
        h = 1.0 / max(nx, ny)
    K0, bvec = element_matrices(h, nu)
    nph = {"single": 1, "two": 2, "three": 3}[phases]
    cell_fields = {1: (FIELD_P,), 2: (FIELD_S, FIELD_P), 3: (FIELD_S, FIELD_S2, FIELD_P)}[nph]
    shape = (nz, ny, nx)
    arr = lambda a: np.ascontiguousarray(np.broadcast_to(np.asarray(a, dtype=np.float64), shape))  # noqa: E731
    Ea, kxa, kya, kza = arr(E), arr(kx), arr(ky), arr(kz)
    pa = arr(pstate if pstate is not None else np.zeros(shape))
    sa = np.ascontiguousarray(sats, dtype=np.float64).reshape(nph - 1, *shape) if nph > 1 else None
    K0 = np.ascontiguousarray(K0)
    bvec = np.ascontiguousarray(bvec)
    a = _lib.Assembly()
    a.nx, a.ny, a.nz, a.phases = nx, ny, nz, nph
    a.h, a.V = float(h), float(h ** 3)
    a.phi, a.ct, a.dt, a.biot = float(phi), float(ct), float(dt), float(biot)
    for t in range(3):
        a.mu[t] = float(mu[t]) if t < len(mu) else 1.0
    a.E, a.kx, a.ky, a.kz = Ea.ctypes.data, kxa.ctypes.data, kya.ctypes.data, kza.ctypes.data
    a.sats = sa.ctypes.data if sa is not None else None
    a.pstate, a.K0, a.bvec = pa.ctypes.data, K0.ctypes.data, bvec.ctypes.data
    out = ctypes.c_void_p()
    _lib.check(_lib.lib().pmgr_assemble_poromech(ctypes.byref(a), current_stream(), ctypes.byref(out)))
    nr, nc_, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.lib().pmgr_csr_info(out, ctypes.byref(nr), ctypes.byref(nc_), ctypes.byref(nnz)))
    A = DeviceCsr(out, nr.value, nc_.value, nnz.value)
    n_u = 3 * (nx + 1) * (ny + 1) * (nz + 1)
    ncell = nx * ny * nz
    nf = len(cell_fields)
    n = n_u + nf * ncell
    field_of = np.concatenate([np.full(n_u, FIELD_U, dtype=np.int8),
                               np.tile(np.array(cell_fields, dtype=np.int8), ncell)])
    entity_of = np.concatenate([(np.arange(n_u) // 3).astype(np.int32),
                                np.repeat(np.arange(ncell, dtype=np.int32), nf)])
    rhs = rhs_rng.standard_normal(n) if rhs_rng is not None else np.zeros(n)
    return DeviceProblem(name, nx, ny, nz, A, field_of, entity_of, rhs, cell_fields,
                         dict(h=h, dt=dt, phases=phases, device=True))


# ---------------------------------------------------------------------------
# the BASELINE.json configurations
# ---------------------------------------------------------------------------


def _streams(seed):
    ss = np.random.SeedSequence(seed).spawn(5)
    return [np.random.default_rng(s) for s in ss]  # E, perm, sat, pnoise, rhs


def _pressure_state(rng, nx, ny, nz, h, noise=0.3):
    x = (np.arange(nx) + 0.5) * h
    base = np.broadcast_to(1.0 - x[None, None, :], (nz, ny, nx))
    return base + noise * h * rng.standard_normal((nz, ny, nx))


# Time step of the two/three-phase configs: chosen so the accumulation term
# phi*V/dt is comparable to the upwind flux derivatives (an implicit step at a
# moderate CFL number), recorded in DESIGN.md.
_DT_MULTIPHASE = 0.002


def make_c1(seed=0, n=16, device=False):
    """C1: single-phase Biot on n^3 (BASELINE.json configs[0])."""
    rE, rk, _rs, _rp, rb = _streams(seed)
    E = np.exp(0.5 * rE.standard_normal((n, n, n)))
    k = np.exp(1.0 * rk.standard_normal((n, n, n)))
    p = np.zeros((n, n, n))
    return (assemble_device if device else assemble)(n, n, n, E=E, kx=k, ky=k, kz=k, phases="single", pstate=p,
                    phi=0.2, ct=1e-3, dt=1.0, rhs_rng=rb, name=f"C1-{n}^3")


def make_c2(seed=0, n=32, device=False):
    """C2: two-phase Corey, mu ratio 10, s ~ U(0.2, 0.8) (configs[1])."""
    rE, rk, rs, rp, rb = _streams(seed)
    E = np.exp(0.5 * rE.standard_normal((n, n, n)))
    k = np.exp(1.0 * rk.standard_normal((n, n, n)))
    s = rs.uniform(0.2, 0.8, (1, n, n, n))
    h = 1.0 / n
    p = _pressure_state(rp, n, n, n, h)
    return (assemble_device if device else assemble)(n, n, n, E=E, kx=k, ky=k, kz=k, phases="two", sats=s, pstate=p,
                    mu=(1.0, 10.0), phi=0.2, ct=1e-3, dt=_DT_MULTIPHASE, rhs_rng=rb,
                    name=f"C2-{n}^3")


def make_c3(seed=0, n=64, device=False):
    """C3: layered lognormal sigma=2 (4-cell z-layers, corr 8), kz=0.1 kx,
    E contrast 1e3 between alternating layer pairs (configs[2])."""
    rE, rk, rs, rp, rb = _streams(seed)
    logk = _layered_logperm(rk, n, n, n, layer=4, corr=8.0)
    kx = np.exp(2.0 * logk)
    kz = 0.1 * kx
    layer = np.arange(n) // 4
    Ez = np.where((layer // 2) % 2 == 1, 1e3, 1.0)
    E = np.broadcast_to(Ez[:, None, None], (n, n, n)).copy()
    s = rs.uniform(0.2, 0.8, (1, n, n, n))
    h = 1.0 / n
    p = _pressure_state(rp, n, n, n, h)
    return (assemble_device if device else assemble)(n, n, n, E=E, kx=kx, ky=kx, kz=kz, phases="two", sats=s, pstate=p,
                    mu=(1.0, 10.0), phi=0.2, ct=1e-3, dt=_DT_MULTIPHASE, rhs_rng=rb,
                    name=f"C3-{n}^3")


def make_c4(seed=0, n=128, device=False, nz=None):
    """C4: three-phase, Stone-I-like, saturations ~ Dirichlet(2,2,2),
    perm sigma=1.5 (configs[3]).  nz < n: an n x n x nz slab of the same
    generator (the bounded CPU-baseline sample, bench.py)."""
    nz = n if nz is None else nz
    rE, rk, rs, rp, rb = _streams(seed)
    E = np.exp(0.5 * rE.standard_normal((nz, n, n)))
    k = np.exp(1.5 * rk.standard_normal((nz, n, n)))
    d = rs.dirichlet((2.0, 2.0, 2.0), size=(nz, n, n))  # (…, 3): w, g, o
    sats = np.stack([d[..., 0], d[..., 1]])
    h = 1.0 / n
    p = _pressure_state(rp, n, n, nz, h)
    return (assemble_device if device else assemble)(n, n, nz, E=E, kx=k, ky=k, kz=k, phases="three", sats=sats,
                                                     pstate=p, mu=(1.0, 0.2, 5.0), phi=0.2, ct=1e-3,
                                                     dt=_DT_MULTIPHASE, rhs_rng=rb,
                                                     name=f"C4-{n}^3" if nz == n else f"C4-{n}x{n}x{nz}")


def make_c5(seed=0, nxy=128, nz_per_gpu=128, gpus=1, device=False):
    """C5: weak-scaling slab stack nxy x nxy x (nz_per_gpu * gpus) (configs[4]).

    The random fields are drawn for the global grid, so a slab does not depend
    on how many GPUs share the stack.
    """
    nz = nz_per_gpu * gpus
    rE, rk, rs, rp, rb = _streams(seed)
    E = np.exp(0.5 * rE.standard_normal((nz, nxy, nxy)))
    k = np.exp(1.0 * rk.standard_normal((nz, nxy, nxy)))
    s = rs.uniform(0.2, 0.8, (1, nz, nxy, nxy))
    h = 1.0 / nxy
    p = _pressure_state(rp, nxy, nxy, nz, h)
    return (assemble_device if device else assemble)(nxy, nxy, nz, E=E, kx=k, ky=k, kz=k, phases="two", sats=s, pstate=p,
                    mu=(1.0, 10.0), phi=0.2, ct=1e-3, dt=_DT_MULTIPHASE, rhs_rng=rb,
                    name=f"C5-{nxy}x{nxy}x{nz}")


def rank_major(pb: Problem, nranks: int):
    """Renumber a problem so that each rank's z-slab is one contiguous range.

    Rank r owns the node planes and cell layers z in [z0_r, z1_r) of
    `dist.slab_bounds` (the last rank also owns the top node plane).  The new
    order is rank after rank; inside a rank: its displacement dofs
    (node-blocked, nodes in their original order) then its flow dofs (cells
    in their original order, fields interleaved).  For nranks == 1 this is the
    original layout.  Row and column numbering change together (P A P^T) and
    each row's columns are re-sorted, so the result is again a valid
    reference CsrMatrix.  Returns (problem, bounds) with bounds[r] the first
    row of rank r (bounds[nranks] = n): the row ranges libpmgr's row
    distribution takes.
    """
    from .dist import slab_bounds

    slabs = slab_bounds(pb.nz, nranks)
    plane = (pb.nx + 1) * (pb.ny + 1)
    layer = pb.nx * pb.ny
    nf = len(pb.cell_fields)
    n_u = pb.n_u
    parts, bounds = [], [0]
    for r, (z0, z1) in enumerate(slabs):
        zn1 = z1 + 1 if r == nranks - 1 else z1
        parts.append(np.arange(3 * plane * z0, 3 * plane * zn1, dtype=np.int64))
        parts.append(n_u + np.arange(nf * layer * z0, nf * layer * z1, dtype=np.int64))
        bounds.append(bounds[-1] + len(parts[-2]) + len(parts[-1]))
    perm = np.concatenate(parts)  # new -> old
    n = pb.n
    if len(perm) != n:
        raise AssertionError("rank-major permutation does not cover the dofs")
    if isinstance(pb, DeviceProblem):  # permute the device matrix in place on the GPU
        import ctypes

        from . import _lib
        from .sparse import DeviceCsr, current_stream

        perm = np.ascontiguousarray(perm, dtype=np.int64)
        out = ctypes.c_void_p()
        _lib.check(_lib.lib().pmgr_csr_permute(pb.A.handle, perm.ctypes.data, current_stream(), ctypes.byref(out)))
        A = DeviceCsr(out, pb.A.nrows, pb.A.ncols, pb.A.nnz)
        new = DeviceProblem(pb.name + f"-rm{nranks}", pb.nx, pb.ny, pb.nz, A, pb.field_of[perm],
                            pb.entity_of[perm], pb.rhs[perm], pb.cell_fields,
                            dict(pb.meta, rank_bounds=list(bounds), perm=perm))
        return new, np.array(bounds, dtype=np.int64)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    ro = pb.row_offsets
    cnt = np.diff(ro)[perm]
    new_ro = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=new_ro[1:])
    take = np.repeat(ro[perm] - new_ro[:-1], cnt) + np.arange(new_ro[-1])
    rows = np.repeat(np.arange(n, dtype=np.int64), cnt)
    cols = inv[pb.col_indices[take]]
    order = np.lexsort((cols, rows))
    new = Problem(pb.name + f"-rm{nranks}", pb.nx, pb.ny, pb.nz, new_ro, cols[order].astype(np.int32),
                  pb.values[take][order], pb.field_of[perm], pb.entity_of[perm], pb.rhs[perm], pb.cell_fields,
                  dict(pb.meta, rank_bounds=list(bounds), perm=perm))
    return new, np.array(bounds, dtype=np.int64)


CONFIGS = {"C1": make_c1, "C2": make_c2, "C3": make_c3, "C4": make_c4, "C5": make_c5}


# ---------------------------------------------------------------------------
# solver configurations
# ---------------------------------------------------------------------------
#
# "parity": the round-1 configuration every golden up to 32^3 pins -- l1-Jacobi
# AMG (npartitions >= n), one AMG V-cycle of F-relaxation, no global smoother,
# GMRES(100).  It converges at full size for C1, C2, C4 (1249 iterations) and
# C5 (635), not for C3 (stalls above 32^3: 2801 iterations at 32^3, the
# oracle's count exactly).
#
# "production": reference-supported options chosen per config from the
# measured iteration counts (tools/conv_probe2.py, profiles/r02_convergence.md)
# so that every config converges at full size:
#   C3 -- ILU(1) level-2 global smoother over partitions of 16 flow rows (the
#         paper's production smoother, default_three_level mgr.py:104-120),
#         two AMG V-cycles of displacement F-relaxation, GMRES(400);
#   C4 -- three AMG V-cycles of displacement F-relaxation, GMRES(300);
#   C5 -- two AMG V-cycles of displacement F-relaxation, GMRES(200);
#   C1, C2 -- the parity configuration.
# GMRES restart is unspecified by BASELINE.json for C2-C5.

ILU_PART_ROWS = 16


def solver_options(name: str, pb, variant: str = "production") -> dict:
    """Plain-data description of the MGR + GMRES configuration of a config:
    `levels` (f/c field sets, f_relax, f_relax_sweeps, n_max, global_smoother),
    `npartitions` (global smoother partitions), AMG options, GMRES restart /
    max_iters / rtol, and the flow ordering.  Turned into library objects by
    mgr.config_from_options (and into oracle objects by the tests)."""
    nf = len(pb.cell_fields)
    fs, restart, smoother, nparts = 1, 100, "none", 1
    if variant == "production":
        if name == "C3":
            fs, restart, smoother = 2, 400, "ilu"
            nparts = max(1, (pb.n - pb.n_u) // ILU_PART_ROWS)
        elif name == "C4":
            fs, restart = 3, 300
        elif name == "C5":
            fs, restart = 2, 200
    elif variant != "parity":
        raise ValueError(f"unknown solver variant {variant!r}")
    if nf == 1:
        levels = [dict(f={FIELD_U}, c={FIELD_P}, f_relax="amg", f_relax_sweeps=fs, n_max=None)]
    elif nf == 3:
        levels = [dict(f={FIELD_U}, c={FIELD_S, FIELD_S2, FIELD_P}, f_relax="amg", f_relax_sweeps=fs, n_max=4),
                  dict(f={FIELD_S2}, c={FIELD_S, FIELD_P}, f_relax="jacobi", global_smoother=smoother),
                  dict(f={FIELD_S}, c={FIELD_P}, f_relax="jacobi")]
    else:
        levels = [dict(f={FIELD_U}, c={FIELD_S, FIELD_P}, f_relax="amg", f_relax_sweeps=fs, n_max=4),
                  dict(f={FIELD_S}, c={FIELD_P}, f_relax="jacobi", global_smoother=smoother)]
    for lv in levels:
        lv.setdefault("f_relax_sweeps", 1)
        lv.setdefault("n_max", None)
        lv.setdefault("global_smoother", "none")
    return dict(levels=levels, npartitions=nparts, terminal_cycles=1, f_relax_position="pre",
                amg_f_relax=dict(strength_threshold=0.5, num_functions=3, npartitions=10 ** 9),
                amg_terminal=dict(strength_threshold=0.25, npartitions=10 ** 9),
                restart=restart, max_iters=3000, rtol=1e-6,
                interleaved=(nf == 2 and smoother == "hbgs"), variant=variant)


def make(name: str, seed: int = 0, **kw) -> Problem:
    return CONFIGS[name](seed=seed, **kw)
