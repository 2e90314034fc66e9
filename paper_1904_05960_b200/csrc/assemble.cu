// assemble.cu -- on-device Jacobian assembly of the synthetic poromechanics
// systems (the reference's SPEC poromech, SPEC.md:412-545,
// has no code).  Restates paper_1904_05960_b200/problems.py:assemble on the
// GPU: one thread per row writes its CSR entries in the host generator's slot
// order with the host generator's arithmetic (explicit _rn intrinsics, no FMA
// contraction), so the device matrix is bitwise the host one.  Inputs are the
// per-cell fields (E, k, saturations, pressure state) and the 24x24 reference
// element matrix / Biot vector; the matrix never touches the host.
#include "hier.cuh"

namespace pmgr {
namespace {

struct AsmP {
    int nx, ny, nz, nf, phases;  // phases: 1 single, 2 two, 3 three
    double h, V, phi, ct, dt, biot, mu[3];
    const double *E, *kx, *ky, *kz, *sats, *pst, *K0, *bvec;
    const double *lam, *dlam, *sph;  // per phase / per (phase, sat) / per phase, x nc
};

__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dv(double a, double b) { return __ddiv_rn(a, b); }

// _mobilities (problems.py): lam[e], dlam[e][f], Sph[e] per cell
__global__ void k_asm_mob(AsmP P, int64_t nc, double *lam, double *dlam, double *sph) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= nc) return;
    if (P.phases == 1) {
        lam[c] = 1.0;
        sph[c] = 1.0;
        return;
    }
    if (P.phases == 2) {
        const double s = P.sats[c];
        const double om = sub(1.0, s);
        lam[c] = dv(mul(s, s), P.mu[0]);
        lam[nc + c] = dv(mul(om, om), P.mu[1]);
        dlam[c] = dv(mul(2.0, s), P.mu[0]);
        dlam[nc + c] = dv(mul(-2.0, om), P.mu[1]);
        sph[c] = s;
        sph[nc + c] = om;
        return;
    }
    const double sw = P.sats[c], sg = P.sats[nc + c];
    const double so = sub(sub(1.0, sw), sg);
    const double a = sub(1.0, sw), b = sub(1.0, sg);
    const double krw = mul(sw, sw), krg = mul(sg, sg);
    const double kro = mul(mul(so, a), b);
    const double dsw = sub(mul(-a, b), mul(so, b));
    const double dsg = sub(mul(-a, b), mul(so, a));
    lam[c] = dv(krw, P.mu[0]);
    lam[nc + c] = dv(krg, P.mu[1]);
    lam[2 * nc + c] = dv(kro, P.mu[2]);
    // dlam[e][f] at (e * 2 + f) * nc
    dlam[(0 * 2 + 0) * nc + c] = dv(mul(2.0, sw), P.mu[0]);
    dlam[(0 * 2 + 1) * nc + c] = 0.0;
    dlam[(1 * 2 + 0) * nc + c] = 0.0;
    dlam[(1 * 2 + 1) * nc + c] = dv(mul(2.0, sg), P.mu[1]);
    dlam[(2 * 2 + 0) * nc + c] = dv(dsw, P.mu[2]);
    dlam[(2 * 2 + 1) * nc + c] = dv(dsg, P.mu[2]);
    sph[c] = sw;
    sph[nc + c] = sg;
    sph[2 * nc + c] = so;
}

__device__ __forceinline__ int64_t cell_id(const AsmP &P, int i, int j, int k) {
    return i + (int64_t)P.nx * (j + (int64_t)P.ny * k);
}

// row lengths: displacement rows (valid neighbour nodes x 3 + valid cells),
// Dirichlet bottom rows 1, flow rows 24 + valid 7-point slots x nf
__global__ void k_asm_count(AsmP P, int64_t n_u, int64_t nc, int64_t *cnt) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int NX = P.nx + 1, NY = P.ny + 1, NZ = P.nz + 1;
    if (r < n_u) {
        const int64_t node = r / 3;
        const int i = (int)(node % NX), j = (int)((node / NX) % NY), k = (int)(node / ((int64_t)NX * NY));
        if (k == 0) {
            cnt[r] = 1;
            return;
        }
        int c = 0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int mi = i + dx, mj = j + dy, mk = k + dz;
                    c += (mi >= 0 && mi < NX && mj >= 0 && mj < NY && mk >= 0 && mk < NZ) ? 3 : 0;
                }
        for (int ck = 0; ck < 2; ++ck)
            for (int cj = 0; cj < 2; ++cj)
                for (int ci = 0; ci < 2; ++ci) {
                    const int a = i - 1 + ci, b = j - 1 + cj, d = k - 1 + ck;
                    c += (a >= 0 && a < P.nx && b >= 0 && b < P.ny && d >= 0 && d < P.nz) ? 1 : 0;
                }
        cnt[r] = c;
        return;
    }
    const int64_t q = r - n_u;
    if (q >= (int64_t)P.nf * nc) return;
    const int64_t cell = q / P.nf;
    const int i = (int)(cell % P.nx), j = (int)((cell / P.nx) % P.ny), k = (int)(cell / ((int64_t)P.nx * P.ny));
    int slots = 1 + (k > 0) + (k < P.nz - 1) + (j > 0) + (j < P.ny - 1) + (i > 0) + (i < P.nx - 1);
    cnt[r] = 24 + (int64_t)slots * P.nf;
}

__global__ void k_asm_urows(AsmP P, int64_t n_u, const int64_t *ro, int32_t *ci_out, double *v_out) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= n_u) return;
    const int NX = P.nx + 1, NY = P.ny + 1, NZ = P.nz + 1;
    const int64_t node = r / 3;
    const int a = (int)(r % 3);
    const int i = (int)(node % NX), j = (int)((node / NX) % NY), k = (int)(node / ((int64_t)NX * NY));
    int64_t w = ro[r];
    if (k == 0) {  // Dirichlet: identity row, columns kept elsewhere
        ci_out[w] = (int32_t)r;
        v_out[w] = 1.0;
        return;
    }
    for (int dz = -1; dz <= 1; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int mi = i + dx, mj = j + dy, mk = k + dz;
                if (!(mi >= 0 && mi < NX && mj >= 0 && mj < NY && mk >= 0 && mk < NZ)) continue;
                const int64_t mnode = mi + (int64_t)NX * (mj + (int64_t)NY * mk);
                for (int b = 0; b < 3; ++b) {
                    double s = 0.0;
                    for (int ck = 0; ck < 2; ++ck)
                        for (int cj = 0; cj < 2; ++cj)
                            for (int cii = 0; cii < 2; ++cii) {
                                const int lx = 1 - cii, ly = 1 - cj, lz = 1 - ck;
                                const int mx = lx + dx, my = ly + dy, mz = lz + dz;
                                if (!(mx >= 0 && mx <= 1 && my >= 0 && my <= 1 && mz >= 0 && mz <= 1)) continue;
                                const int ln = lx + 2 * ly + 4 * lz, lm = mx + 2 * my + 4 * mz;
                                const int ca = i - 1 + cii, cb = j - 1 + cj, cd = k - 1 + ck;
                                const bool in = ca >= 0 && ca < P.nx && cb >= 0 && cb < P.ny && cd >= 0 && cd < P.nz;
                                const double e = in ? P.E[cell_id(P, ca, cb, cd)] : 0.0;
                                s = add(s, mul(e, P.K0[(3 * ln + a) * 24 + 3 * lm + b]));
                            }
                    ci_out[w] = (int32_t)(3 * mnode + b);
                    v_out[w] = s;
                    ++w;
                }
            }
    const int64_t n_u_total = n_u;
    const int pslot = P.nf - 1;
    for (int ck = 0; ck < 2; ++ck)
        for (int cj = 0; cj < 2; ++cj)
            for (int cii = 0; cii < 2; ++cii) {
                const int ca = i - 1 + cii, cb = j - 1 + cj, cd = k - 1 + ck;
                if (!(ca >= 0 && ca < P.nx && cb >= 0 && cb < P.ny && cd >= 0 && cd < P.nz)) continue;
                const int ln = (1 - cii) + 2 * (1 - cj) + 4 * (1 - ck);
                ci_out[w] = (int32_t)(n_u_total + (int64_t)P.nf * cell_id(P, ca, cb, cd) + pslot);
                v_out[w] = mul(-P.biot, P.bvec[3 * ln + a]);
                ++w;
            }
}

// flow rows: Biot coupling to the 8 cell nodes, then the 7-point TPFA slots
// (-z, -y, -x, self, +x, +y, +z) x fields; contributions to each entry in the
// host generator's order: accumulation, then per axis x, y, z the face where
// the cell is the lower one, then the face where it is the upper one
__global__ void k_asm_frows(AsmP P, int64_t n_u, int64_t nc, const int64_t *ro, int32_t *ci_out, double *v_out) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= (int64_t)P.nf * nc) return;
    const int nf = P.nf, pslot = nf - 1, nsat = nf - 1;
    const int64_t c = q / nf;
    const int e = (int)(q % nf);
    const int i = (int)(c % P.nx), j = (int)((c / P.nx) % P.ny), k = (int)(c / ((int64_t)P.nx * P.ny));
    const int NX = P.nx + 1, NY = P.ny + 1;
    const double h = P.h, V = P.V;
    int64_t w = ro[n_u + q];
    // Biot coupling: coef * bvec
    const double coef = dv(mul(P.biot, P.sph[(int64_t)e * nc + c]), P.dt);
    for (int ln = 0; ln < 8; ++ln) {
        const int a = ln & 1, b = (ln >> 1) & 1, cc = (ln >> 2) & 1;
        const int64_t nd = (i + a) + (int64_t)NX * ((j + b) + (int64_t)NY * (k + cc));
        for (int comp = 0; comp < 3; ++comp) {
            ci_out[w] = (int32_t)(3 * nd + comp);
            v_out[w] = mul(coef, P.bvec[3 * ln + comp]);
            ++w;
        }
    }
    // J[slot][field]
    double J[7][3];
    for (int s = 0; s < 7; ++s)
        for (int f = 0; f < 3; ++f) J[s][f] = 0.0;
    // dS: two-phase [[1], [-1]]; three-phase [[1,0],[0,1],[-1,-1]]
    for (int f = 0; f < nsat; ++f) {
        double ds;
        if (P.phases == 2) ds = (e == 0) ? 1.0 : -1.0;
        else ds = (e == 2) ? -1.0 : (e == f ? 1.0 : 0.0);
        J[3][f] = add(J[3][f], mul(dv(mul(V, P.phi), P.dt), ds));
    }
    J[3][pslot] = add(J[3][pslot], dv(mul(mul(mul(V, P.phi), P.sph[(int64_t)e * nc + c]), P.ct), P.dt));
    const double *lam = P.lam + (int64_t)e * nc;
    for (int axis = 0; axis < 3; ++axis) {  // x, y, z
        const double *kd = axis == 0 ? P.kx : axis == 1 ? P.ky : P.kz;
        const int sK = 4 + axis, sL = 2 - axis;
        const int di = axis == 0, dj = axis == 1, dk = axis == 2;
        const bool has_up = axis == 0 ? i < P.nx - 1 : axis == 1 ? j < P.ny - 1 : k < P.nz - 1;
        const bool has_lo = axis == 0 ? i > 0 : axis == 1 ? j > 0 : k > 0;
        const int64_t cu = has_up ? cell_id(P, i + di, j + dj, k + dk) : -1;
        const int64_t cl = has_lo ? cell_id(P, i - di, j - dj, k - dk) : -1;
        double gK = 0.0, gL = 0.0, TK = 0.0, TL = 0.0, phK = 0.0, phL = 0.0;
        bool upK = false, upL = false;
        if (has_up) {  // face (c, cu): c is the lower cell K
            const double tK = mul(mul(2.0, kd[c]), h), tL = mul(mul(2.0, kd[cu]), h);
            TK = dv(mul(tK, tL), add(tK, tL));
            phK = sub(P.pst[c], P.pst[cu]);
            upK = phK >= 0.0;
            gK = mul(TK, upK ? lam[c] : lam[cu]);
        }
        if (has_lo) {  // face (cl, c): c is the upper cell L
            const double tK = mul(mul(2.0, kd[cl]), h), tL = mul(mul(2.0, kd[c]), h);
            TL = dv(mul(tK, tL), add(tK, tL));
            phL = sub(P.pst[cl], P.pst[c]);
            upL = phL >= 0.0;
            gL = mul(TL, upL ? lam[cl] : lam[c]);
        }
        // pressure derivatives (K statements, then L statements)
        if (has_up) {
            J[3][pslot] = add(J[3][pslot], gK);
            J[sK][pslot] = sub(J[sK][pslot], gK);
        }
        if (has_lo) {
            J[3][pslot] = add(J[3][pslot], gL);
            J[sL][pslot] = sub(J[sL][pslot], gL);
        }
        // saturation derivatives
        for (int f = 0; f < nsat; ++f) {
            const double *dl = P.dlam + ((int64_t)e * nsat + f) * nc;
            if (has_up) {
                const double dK = mul(mul(TK, dl[c]), phK), dL = mul(mul(TK, dl[cu]), phK);
                J[3][f] = add(J[3][f], upK ? dK : 0.0);
                J[sK][f] = add(J[sK][f], upK ? 0.0 : dL);
            }
            if (has_lo) {
                const double dK = mul(mul(TL, dl[cl]), phL), dL = mul(mul(TL, dl[c]), phL);
                J[sL][f] = sub(J[sL][f], upL ? dK : 0.0);
                J[3][f] = sub(J[3][f], upL ? 0.0 : dL);
            }
        }
    }
    const bool valid[7] = {k > 0, j > 0, i > 0, true, i < P.nx - 1, j < P.ny - 1, k < P.nz - 1};
    const int64_t nb[7] = {c - (int64_t)P.nx * P.ny, c - P.nx, c - 1, c, c + 1, c + P.nx, c + (int64_t)P.nx * P.ny};
    for (int s = 0; s < 7; ++s) {
        if (!valid[s]) continue;
        for (int f = 0; f < nf; ++f) {
            ci_out[w] = (int32_t)(n_u + (int64_t)nf * nb[s] + f);
            v_out[w] = J[s][f];
            ++w;
        }
    }
}

}  // namespace

std::shared_ptr<Csr> assemble_poromech(const pmgr_assembly &A, cudaStream_t s) {
    if (A.nx < 1 || A.ny < 1 || A.nz < 1) fail(PMGR_ERR_INVALID, "grid must have at least one cell per axis");
    if (A.phases < 1 || A.phases > 3) fail(PMGR_ERR_INVALID, "phases must be 1, 2 or 3");
    const int64_t nc = (int64_t)A.nx * A.ny * A.nz;
    const int64_t n_u = 3 * (int64_t)(A.nx + 1) * (A.ny + 1) * (A.nz + 1);
    const int nf = A.phases;
    const int nsat = nf - 1;
    const int64_t n = n_u + nf * nc;
    if (n >= (int64_t)INT32_MAX) fail(PMGR_ERR_INVALID, "system too large for int32 columns");
    // device copies of the per-cell fields
    DBuf<double> E(nc), kx(nc), ky(nc), kz(nc), pst(nc), sats(nsat > 0 ? nsat * nc : 1), K0(576), bv(24);
    auto up = [&](DBuf<double> &d, const double *h, int64_t cnt) {
        if (cnt > 0) PMGR_CUDA(cudaMemcpyAsync(d.p, h, sizeof(double) * cnt, cudaMemcpyHostToDevice, s));
    };
    up(E, A.E, nc);
    up(kx, A.kx, nc);
    up(ky, A.ky, nc);
    up(kz, A.kz, nc);
    up(pst, A.pstate, nc);
    if (nsat > 0) up(sats, A.sats, nsat * nc);
    up(K0, A.K0, 576);
    up(bv, A.bvec, 24);
    DBuf<double> lam((int64_t)nf * nc), dlam(nsat > 0 ? (int64_t)nf * nsat * nc : 1), sph((int64_t)nf * nc);
    AsmP P{};
    P.nx = A.nx;
    P.ny = A.ny;
    P.nz = A.nz;
    P.nf = nf;
    P.phases = A.phases;
    P.h = A.h;
    P.V = A.V;
    P.phi = A.phi;
    P.ct = A.ct;
    P.dt = A.dt;
    P.biot = A.biot;
    for (int t = 0; t < 3; ++t) P.mu[t] = A.mu[t];
    P.E = E.p;
    P.kx = kx.p;
    P.ky = ky.p;
    P.kz = kz.p;
    P.sats = sats.p;
    P.pst = pst.p;
    P.K0 = K0.p;
    P.bvec = bv.p;
    P.lam = lam.p;
    P.dlam = dlam.p;
    P.sph = sph.p;
    k_asm_mob<<<grid_for(nc, 256), 256, 0, s>>>(P, nc, lam.p, dlam.p, sph.p);
    PMGR_LAUNCHED();
    auto M = std::make_shared<Csr>();
    TBuf<int64_t> cnt(n, s);
    k_asm_count<<<grid_for(n, 256), 256, 0, s>>>(P, n_u, nc, cnt.p);
    PMGR_LAUNCHED();
    M->nrows = M->ncols = n;
    M->ro.alloc(n + 1);
    M->nnz = exclusive_scan_total(cnt.p, M->ro.p, n, s);
    if (M->nnz >= (int64_t)INT32_MAX) fail(PMGR_ERR_INVALID, "nnz exceeds the per-device int32 limit");
    M->ci.alloc(M->nnz);
    M->v.alloc(M->nnz);
    k_asm_urows<<<grid_for(n_u, 128), 128, 0, s>>>(P, n_u, M->ro.p, M->ci.p, M->v.p);
    PMGR_LAUNCHED();
    k_asm_frows<<<grid_for((int64_t)nf * nc, 128), 128, 0, s>>>(P, n_u, nc, M->ro.p, M->ci.p, M->v.p);
    PMGR_LAUNCHED();
    csr_finalize(*M, s, false);  // sliced jagged copy: at first use (capi.cu ensure_sj)
    PMGR_CUDA(cudaStreamSynchronize(s));
    return M;
}

}  // namespace pmgr
