// mgr.cu -- MGR setup and application on the device (reference mgr.py).
//
// Setup per level (mgr.py:329-371):
//   split      is_c from the level's field tags; C/F row lists and index maps
//   blocks     A_FF, A_FC, A_CF, A_CC with order-preserving renumbering and
//              explicit zeros kept (extract_blocks, sparse.py:269-288)
//   transfers  dinv = 1.0/diag(A_FF); P = [W_p; I] with W_p = A_FC*(-dinv)
//              row-scaled; R = [0 I] is an injection and never stored
//              (build_transfers, mgr.py:131-187, injection_jacobi/injection)
//   F-relax    AMG on A_FF (num_functions 3 for F={U}) or Jacobi (mgr.py:374-386)
//   coarse     T = (R A) P with the structural pattern (spgemm keeps
//              cancellations as +0.0); with n_max the non-Galerkin
//              A_CC - sparsify(A_CC - T) (build_coarse, mgr.py:212-231)
// Apply per level (mgr.py:405-429), with f_relax_position "pre":
//   z_F = M_FF^{-1} v_F ; r_C = v_C - A_CF z_F ; e_C = next level ;
//   z = [z_F; 0] + P e_C
// The residual is only formed on C rows (R is an injection) and only
// against A_CF, which reads a fraction of A: the same numbers, since the
// skipped terms multiply exact zeros of z.
#include <cstdlib>
#include <set>

#include "dsetup.cuh"
#include "hier.cuh"

namespace pmgr {

namespace {

__global__ void k_split(int64_t n, const int8_t *field, uint64_t cmask, int8_t *is_c, int64_t *c64,
                        int64_t *f64) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int8_t c = (cmask >> (field[i] & 63)) & 1ull;
    is_c[i] = c;
    c64[i] = c;
    f64[i] = 1 - c;
}

// which field tags occur, and how many rows the C mask selects
__global__ void k_field_stats(int64_t n, const int8_t *field, uint64_t cmask, int *seen, unsigned long long *nc) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long c = 0;
    if (i < n) {
        const int8_t t = field[i];
        if (!seen[(uint8_t)t]) seen[(uint8_t)t] = 1;  // benign race: every writer stores 1
        c = (cmask >> (t & 63)) & 1ull;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(FULL, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(nc, c);
}

// the next level's layout: field / entity of the C rows, in order
__global__ void k_restrict_layout(int64_t nc, const int64_t *c_rows, const int8_t *field, const int32_t *entity,
                                  int8_t *field2, int32_t *entity2) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= nc) return;
    const int64_t i = c_rows[k];
    field2[k] = field[i];
    entity2[k] = entity[i];
}

__global__ void k_index_maps(int64_t n, const int8_t *is_c, const int64_t *cscan, const int64_t *fscan,
                             int64_t *c_index, int64_t *f_index, int64_t *c_rows, int64_t *f_rows) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (is_c[i]) {
        c_index[i] = cscan[i];
        f_index[i] = -1;
        c_rows[cscan[i]] = i;
    } else {
        c_index[i] = -1;
        f_index[i] = fscan[i];
        f_rows[fscan[i]] = i;
    }
}

// block extraction: rows from `rows` (k-th output row = A row rows[k]),
// columns with colmap[j] >= 0 and is_c[j] == want_c, renumbered by colmap
template <bool FILL>
__global__ void k_extract(int64_t nout, const int64_t *rows, const int64_t *ro, const int32_t *ci,
                          const double *v, const int8_t *is_c, int8_t want_c, const int64_t *colmap,
                          int64_t *cnt, const int64_t *oro, int32_t *oci, double *ov) {
    int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (k >= nout) return;
    const int64_t i = rows[k];
    int64_t w = FILL ? oro[k] : 0;
    for (int64_t q0 = ro[i]; q0 < ro[i + 1]; q0 += 32) {
        int64_t q = q0 + lane;
        bool keep = false;
        int32_t j = 0;
        if (q < ro[i + 1]) {
            j = ci[q];
            keep = is_c[j] == want_c;
        }
        unsigned m = __ballot_sync(FULL, keep);
        if (FILL && keep) {
            int pos = __popc(m & ((1u << lane) - 1u));
            oci[w + pos] = (int32_t)colmap[j];
            ov[w + pos] = v[q];
        }
        w += __popc(m);
    }
    if (!FILL && lane == 0) cnt[k] = w;
}

// rows of A (all columns), -0.0 normalised to +0.0 (R A = 1.0*a summed from 0.0)
template <bool FILL>
__global__ void k_rows_of(int64_t nout, const int64_t *rows, const int64_t *ro, const int32_t *ci,
                          const double *v, int64_t *cnt, const int64_t *oro, int32_t *oci, double *ov) {
    int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (k >= nout) return;
    const int64_t i = rows[k];
    if (!FILL) {
        if (lane == 0) cnt[k] = ro[i + 1] - ro[i];
        return;
    }
    const int64_t off = oro[k] - ro[i];
    for (int64_t q = ro[i] + lane; q < ro[i + 1]; q += 32) {
        oci[q + off] = ci[q];
        double a = v[q];
        ov[q + off] = (a == 0.0) ? 0.0 : a;
    }
}

// P = [W_p; I] in level order
template <bool FILL>
__global__ void k_build_p(int64_t lo, int64_t n, const int8_t *is_c, const int64_t *c_index, const int64_t *f_index,
                          const int64_t *fc_ro, const int32_t *fc_ci, const double *fc_v, const double *dinv,
                          int with_wp, int64_t *cnt, const int64_t *pro, int32_t *pci, double *pv) {
    int64_t i = lo + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    if (is_c[i]) {
        if (lane == 0) {
            if (FILL) {
                pci[pro[i]] = (int32_t)c_index[i];
                pv[pro[i]] = 1.0;
            } else {
                cnt[i] = 1;
            }
        }
        return;
    }
    const int64_t f = f_index[i];
    if (!FILL) {
        if (lane == 0) cnt[i] = with_wp ? fc_ro[f + 1] - fc_ro[f] : 0;
        return;
    }
    if (!with_wp) return;
    const double s = -dinv[f];
    const int64_t off = pro[i] - fc_ro[f];
    for (int64_t q = fc_ro[f] + lane; q < fc_ro[f + 1]; q += 32) {
        pci[q + off] = fc_ci[q];
        pv[q + off] = __dmul_rn(fc_v[q], s);
    }
}

__global__ void k_scatter_add(const double *src, const int64_t *idx, int64_t n, double *dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[idx[i]] += src[i];
}

__global__ void k_jacobi_dinv(int64_t n, const int64_t *ro, const int32_t *ci, const double *v,
                              const double *x, const double *b, const double *dinv, double *xo) {
    // x' = x + dinv * (b - A x)  (mgr.py:249), warp per row
    int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    double s = 0.0;
    for (int64_t q = ro[i] + lane; q < ro[i + 1]; q += 32) s = fma(v[q], x[ci[q]], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0) xo[i] = x[i] + dinv[i] * (b[i] - s);
}

// Extract one block: rows given by `rows` (count nout), columns on the
// `want_c` side renumbered through colmap.
void extract_block(const CsrView &A, const int64_t *rows, int64_t nout, const int8_t *is_c, bool want_c,
                   const int64_t *colmap, int64_t ncols_out, Csr &B, cudaStream_t s) {
    TBuf<int64_t> cnt(nout, s);
    B.nrows = nout;
    B.ncols = ncols_out;
    B.ro.alloc(nout + 1);
    if (nout) {
        k_extract<false><<<grid_for(nout * 32, 256), 256, 0, s>>>(nout, rows, A.ro, A.ci, A.v, is_c, want_c ? 1 : 0,
                                                                 colmap, cnt.p, nullptr, nullptr, nullptr);
        PMGR_LAUNCHED();
    }
    B.nnz = exclusive_scan_total(cnt.p, B.ro.p, nout, s);
    B.ci.alloc(B.nnz);
    B.v.alloc(B.nnz);
    if (nout) {
        k_extract<true><<<grid_for(nout * 32, 256), 256, 0, s>>>(nout, rows, A.ro, A.ci, A.v, is_c, want_c ? 1 : 0,
                                                                colmap, nullptr, B.ro.p, B.ci.p, B.v.p);
        PMGR_LAUNCHED();
    }
}

void rows_of(const CsrView &A, const int64_t *rows, int64_t nout, Csr &B, cudaStream_t s) {
    TBuf<int64_t> cnt(nout, s);
    B.nrows = nout;
    B.ncols = A.ncols;
    B.ro.alloc(nout + 1);
    if (nout) {
        k_rows_of<false><<<grid_for(nout * 32, 256), 256, 0, s>>>(nout, rows, A.ro, A.ci, A.v, cnt.p, nullptr,
                                                                 nullptr, nullptr);
        PMGR_LAUNCHED();
    }
    B.nnz = exclusive_scan_total(cnt.p, B.ro.p, nout, s);
    B.ci.alloc(B.nnz);
    B.v.alloc(B.nnz);
    if (nout) {
        k_rows_of<true><<<grid_for(nout * 32, 256), 256, 0, s>>>(nout, rows, A.ro, A.ci, A.v, nullptr, B.ro.p,
                                                                B.ci.p, B.v.p);
        PMGR_LAUNCHED();
    }
}

std::string field_names(const std::set<int> &f) {
    std::string out = "[";
    bool first = true;
    for (int t : f) {
        if (!first) out += ", ";
        first = false;
        const char *nm = t == 0 ? "'U'" : t == 1 ? "'S'" : t == 2 ? "'P'" : nullptr;
        out += nm ? nm : ("'F" + std::to_string(t) + "'");
    }
    return out + "]";
}

void apply_level(pmgr_mgr &h, size_t l, const double *v, double *z, cudaStream_t s, bool prefilled = false);

void f_relax_apply(MgrLevel &L, const double *vf, double *zf, cudaStream_t s) {
    if (L.f_relax == PMGR_FRELAX_AMG) {
        amg_cycle(*L.amg, vf, nullptr, zf, s);
        for (int c = 1; c < L.f_relax_sweeps; ++c) {  // ext layout: owned range at off_f
            vec_copy(zf + L.off_f, L.tmpf.p + L.off_f, L.nf, s);
            amg_cycle(*L.amg, vf, L.tmpf.p, zf, s);
        }
    } else {
        vec_mul(L.dinv_ff.p, vf, zf, L.nf, s);
        for (int c = 1; c < L.f_relax_sweeps; ++c) {
            const CsrView F = L.A_ff->view();
            ledger(csr_pass_bytes(F) + 24.0 * L.nf);
            k_jacobi_dinv<<<grid_for(L.nf * 32, 256), 256, 0, s>>>(L.nf, F.ro, F.ci, F.v, zf, vf, L.dinv_ff.p,
                                                                   L.tmpf.p);
            PMGR_LAUNCHED();
            vec_copy(L.tmpf.p, zf, L.nf, s);
        }
    }
}

// A level with a global smoother (mgr.py:411-429): z = S v; F-relaxation on
// the residual v - A z; C residual of the smoothed z; coarse correction.
void apply_level_smoothed(pmgr_mgr &h, size_t l, const double *v, double *z, cudaStream_t s) {
    // vectors in the level's ext layout (row-distributed: owned range at
    // L.off, the smoother local to the rank's partitions, ghosts of zs
    // exchanged before A and A_c read them; offsets 0 and no-ops on one GPU)
    MgrLevel &L = h.levels[l];
    const int64_t o = L.off, of = L.off_f;
    smoother_apply(*L.smoother, v + o, L.zs.p + o, s);
    auto f_relax_on = [&](const double *r, double *zacc) {  // zacc[F] += M_FF^{-1} r[F]
        bool done = false;
        if (L.f_relax_sweeps == 1) {
            if (L.f_relax == PMGR_FRELAX_AMG) {
                done = amg_cycle_rows(*L.amg, r, L.f_rows.p, L.zf.p, s);
            } else {
                vec_scale_gather(r, L.f_rows.p + of, L.dinv_ff.p + of, L.nf, L.zf.p + of, s);
                done = true;
            }
        }
        if (!done) {
            vec_gather(r, L.f_rows.p + of, L.nf, L.vf.p + of, s);
            f_relax_apply(L, L.vf.p, L.zf.p, s);
        }
        ledger(32.0 * L.nf);
        k_scatter_add<<<grid_for(L.nf, 256), 256, 0, s>>>(L.zf.p + of, L.f_rows.p + of, L.nf, zacc);
        PMGR_LAUNCHED();
    };
    if (!h.f_relax_post && L.f_relax != PMGR_FRELAX_NONE) {
        with_halo(*L.A, L.halo_m.get(), L.zs.p, s,
                  [&](const CsrView &V) { spmv_residual(V, L.zs.p, v, L.rr.p, s); });
        f_relax_on(L.rr.p, L.zs.p);
    }
    with_halo(L.A_c, L.halo_m.get(), L.zs.p, s,
              [&](const CsrView &V) { spmv_resid_rows(V, L.zs.p, v, L.c_rows.p, L.rc.p, ResidNext{}, s); });
    apply_level(h, l + 1, L.rc.p, L.zc.p, s, false);
    vec_copy(L.zs.p + o, z + o, L.n, s);
    with_halo(L.P, L.halo_c.get(), L.zc.p, s, [&](const CsrView &V) { spmv_add(V, L.zc.p, z, s); });
    if (h.f_relax_post && L.f_relax != PMGR_FRELAX_NONE) {
        spmv_residual(L.A->view(), z, v, L.rr.p, s);
        f_relax_on(L.rr.p, z);
    }
}

// prefilled: the producer of v already ran this level's first step (the
// terminal AMG's l1-Jacobi entry, or a single Jacobi F-relaxation)
void apply_level(pmgr_mgr &h, size_t l, const double *v, double *z, cudaStream_t s, bool prefilled) {
    if (l == h.levels.size()) {
        if (prefilled) {
            amg_cycle_prefilled(*h.terminal, z, s);
            return;
        }
        amg_cycle(*h.terminal, v, nullptr, z, s);
        for (int c = 1; c < h.terminal_cycles; ++c) {
            vec_copy(z, h.tz.p, h.terminal_A->nrows, s);
            amg_cycle(*h.terminal, v, h.tz.p, z, s);
        }
        return;
    }
    MgrLevel &L = h.levels[l];
    if (L.smoother) {
        apply_level_smoothed(h, l, v, z, s);
        return;
    }
    const bool pre = !h.f_relax_post && L.f_relax != PMGR_FRELAX_NONE;
    double *rc = L.rc.p;
    bool next_prefilled = false;
    if (pre) {
        // single sweep: the F gather is fused into the relaxation's first kernel
        bool done = prefilled;
        if (!done && L.f_relax_sweeps == 1) {
            if (L.f_relax == PMGR_FRELAX_AMG) {
                done = amg_cycle_rows(*L.amg, v, L.f_rows.p, L.zf.p, s);
            } else {
                const int64_t o = L.off_f;
                vec_scale_gather(v, L.f_rows.p + o, L.dinv_ff.p + o, L.nf, L.zf.p + o, s);
                done = true;
            }
        }
        if (!done) {
            vec_gather(v, L.f_rows.p + L.off_f, L.nf, L.vf.p + L.off_f, s);
            f_relax_apply(L, L.vf.p, L.zf.p, s);
        }
        // the consumer's first step rides on the residual kernel
        ResidNext nx;
        if (l + 1 == h.levels.size()) {
            const double *d = nullptr;
            double *b = nullptr, *x = nullptr;
            if (h.terminal_cycles == 1 && amg_entry(*h.terminal, &b, &x, &d)) {
                rc = b;
                nx.x2 = x;
                nx.d2 = d;
                next_prefilled = true;
            }
        } else {
            MgrLevel &N = h.levels[l + 1];
            if (N.f_relax == PMGR_FRELAX_JACOBI && N.f_relax_sweeps == 1 && !N.smoother) {
                nx.sidx = N.f_index.p;
                nx.sd = N.dinv_ff.p;
                nx.sz = N.zf.p;
                next_prefilled = true;
            }
        }
        with_halo(L.A_cf, L.halo_f.get(), L.zf.p, s,
                  [&](const CsrView &V) { spmv_resid_rows(V, L.zf.p, v, L.c_rows.p, rc, nx, s); });
    } else {
        vec_gather(v, L.c_rows.p + L.off_c, L.nc, L.rc.p + L.off_c, s);
    }
    apply_level(h, l + 1, rc, L.zc.p, s, next_prefilled);
    with_halo(L.P, L.halo_c.get(), L.zc.p, s, [&](const CsrView &V) {
        spmv_prolong_combine(V, L.zc.p, pre ? L.zf.p : nullptr, pre ? L.f_index.p : nullptr, z, s);
    });
    if (h.f_relax_post && L.f_relax != PMGR_FRELAX_NONE) {
        // r = v - A z ; z[F] += M_FF^{-1} r[F]
        DBuf<double> &r = L.tmpf;  // reuse: needs n, allocated as max(n, nf)
        spmv_residual(L.A->view(), z, v, r.p, s);
        vec_gather(r.p, L.f_rows.p, L.nf, L.vf.p, s);
        f_relax_apply(L, L.vf.p, L.zf.p, s);
        ledger(32.0 * L.nf);
        k_scatter_add<<<grid_for(L.nf, 256), 256, 0, s>>>(L.zf.p, L.f_rows.p, L.nf, z);
        PMGR_LAUNCHED();
    }
}

}  // namespace

std::unique_ptr<pmgr_mgr> mgr_build(std::shared_ptr<const Csr> A0, const int8_t *field_of_host,
                                    const int32_t *entity_of_host, const pmgr_level_spec *specs, int nlevels,
                                    const pmgr_mgr_cfg &cfg, cudaStream_t s, const DistSetup *dist) {
    if (A0->nrows != A0->ncols) fail(PMGR_ERR_INVALID, "mgr_setup requires a square matrix");
    setup_trace("mgr begin", -1, s);
    host_trace_report("before");
    // distributed setup (dsetup.cuh): every operator keeps the owned rows of
    // its global row space; dd tracks the owned ranges of the level space
    std::unique_ptr<DistSetup> dd;
    if (dist && dist->nranks > 1) dd.reset(new DistSetup(*dist));
    auto h = std::make_unique<pmgr_mgr>();
    h->n = A0->nrows;
    h->terminal_cycles = cfg.terminal_cycles > 1 ? cfg.terminal_cycles : 1;
    if (const char *e = getenv("PMGR_NO_GRAPHS")) h->use_graphs = (e[0] == '0');
    h->f_relax_post = cfg.f_relax_post;
    // the layout (field tag and entity per row) lives on the device and is
    // restricted to the C rows level by level there; the host copies exist
    // only while a global smoother needs them (12.7M-row host loops cost
    // ~100 ms per C4 setup)
    TBuf<int8_t> dfo(A0->nrows, s);
    TBuf<int32_t> deo(A0->nrows, s);
    PMGR_CUDA(cudaMemcpyAsync(dfo.p, field_of_host, (size_t)A0->nrows, cudaMemcpyHostToDevice, s));
    PMGR_CUDA(cudaMemcpyAsync(deo.p, entity_of_host, sizeof(int32_t) * (size_t)A0->nrows, cudaMemcpyHostToDevice, s));
    bool any_smoother = false;
    for (int lj = 0; lj < nlevels; ++lj) any_smoother |= specs[lj].global_smoother != PMGR_SMOOTHER_NONE;
    std::vector<int8_t> fo;
    std::vector<int32_t> eo;
    if (any_smoother) {
        fo.assign(field_of_host, field_of_host + A0->nrows);
        eo.assign(entity_of_host, entity_of_host + A0->nrows);
    }
    std::shared_ptr<const Csr> cur = A0;
    // FieldLayout ordering: interleaved while every restriction keeps the S/P
    // pairing, else downgraded (the mgr.py:359 x sparse.py:180-189 shim)
    bool interleaved = cfg.flow_interleaved != 0;
    for (int li = 0; li < nlevels; ++li) {
        const pmgr_level_spec &sp = specs[li];
        // (only a global smoother reads the flag: levels with none at or after
        // them skip the check -- two host sorts of the flow rows, ~40 ms per
        // level at C4)
        bool smoother_ahead = false;
        for (int lj = li; lj < nlevels; ++lj) smoother_ahead |= specs[lj].global_smoother != PMGR_SMOOTHER_NONE;
        if (interleaved && smoother_ahead) {
            std::vector<int64_t> sv, pv;
            for (int64_t i = 0; i < (int64_t)fo.size(); ++i) {
                if (fo[i] == 1) sv.push_back(i);
                else if (fo[i] == 2) pv.push_back(i);
            }
            auto by_ent = [&](std::vector<int64_t> &v) {
                auto less = [&](int64_t a, int64_t b) { return eo[a] < eo[b]; };
                if (!std::is_sorted(v.begin(), v.end(), less)) std::stable_sort(v.begin(), v.end(), less);
            };
            by_ent(sv);
            by_ent(pv);
            bool ok = sv.size() == pv.size();
            for (size_t t = 0; ok && t < sv.size(); ++t) ok = (sv[t] - pv[t] == 1 || pv[t] - sv[t] == 1);
            if (!ok) interleaved = false;
        }
        std::set<int> present;
        int64_t nc_h = 0;
        {
            const int64_t nl = cur->nrows;
            TBuf<int> dseen(256, s);
            TBuf<unsigned long long> dnc(1, s);
            PMGR_CUDA(cudaMemsetAsync(dseen.p, 0, sizeof(int) * 256, s));
            PMGR_CUDA(cudaMemsetAsync(dnc.p, 0, sizeof(unsigned long long), s));
            if (nl > 0) {
                k_field_stats<<<grid_for(nl, 256), 256, 0, s>>>(nl, dfo.p, sp.c_mask, dseen.p, dnc.p);
                PMGR_LAUNCHED();
            }
            int seen[256];
            unsigned long long ncv = 0;
            PMGR_CUDA(cudaMemcpyAsync(seen, dseen.p, sizeof(seen), cudaMemcpyDeviceToHost, s));
            PMGR_CUDA(cudaMemcpyAsync(&ncv, dnc.p, sizeof(ncv), cudaMemcpyDeviceToHost, s));
            PMGR_CUDA(cudaStreamSynchronize(s));
            nc_h = (int64_t)ncv;
            for (int t = 0; t < 256; ++t)
                if (seen[t]) present.insert((int)(int8_t)t);
        }
        std::set<int> spec_f;
        for (int t = 0; t < 64; ++t)
            if (((sp.f_mask | sp.c_mask) >> t) & 1ull) spec_f.insert(t);
        if (sp.f_mask & sp.c_mask) fail(PMGR_ERR_INVALID, "f_fields and c_fields must be disjoint");
        if (spec_f != present)
            fail(PMGR_ERR_FIELDS, "level spec fields " + field_names(spec_f) + " do not cover the fields present " +
                                      field_names(present));
        if (!sp.c_mask) fail(PMGR_ERR_INVALID, "empty C set: nothing to reduce onto");
        if (sp.global_smoother != PMGR_SMOOTHER_NONE && sp.global_smoother != PMGR_SMOOTHER_ILU &&
            sp.global_smoother != PMGR_SMOOTHER_HBGS)
            fail(PMGR_ERR_INVALID, "unknown global smoother");
        if (sp.interp == PMGR_INTERP_IDEAL || sp.restrict_ != PMGR_RESTRICT_INJECTION)
            fail(PMGR_ERR_NOT_SUPPORTED, "only injection restriction with injection/injection_jacobi "
                                         "interpolation is on the device path");
        if (sp.f_relax == PMGR_FRELAX_EXACT) fail(PMGR_ERR_NOT_SUPPORTED, "exact F-relaxation is not on the device path");
        if (sp.quasi_impes) fail(PMGR_ERR_NOT_SUPPORTED, "quasi-IMPES is not on the device path");
        const int64_t n = cur->nrows;
        if (nc_h == n) {
            if (present.size() != 1) fail(PMGR_ERR_INVALID, "an all-C level requires a single remaining field");
            break;  // reduction-free limit (mgr.py:347-352)
        }
        MgrLevel L;
        L.A = cur;
        L.n = n;
        L.nc = nc_h;
        L.nf = n - nc_h;
        // ---- split and index maps
        L.is_c.alloc(n);
        TBuf<int64_t> c64(n, s), f64(n, s), cscan(n + 1, s), fscan(n + 1, s), c_index(n, s);
        k_split<<<grid_for(n, 256), 256, 0, s>>>(n, dfo.p, sp.c_mask, L.is_c.p, c64.p, f64.p);
        PMGR_LAUNCHED();
        exclusive_scan_total(c64.p, cscan.p, n, s);
        exclusive_scan_total(f64.p, fscan.p, n, s);
        L.c_rows.alloc(L.nc);
        L.f_rows.alloc(L.nf);
        L.f_index.alloc(n);
        k_index_maps<<<grid_for(n, 256), 256, 0, s>>>(n, L.is_c.p, cscan.p, fscan.p, c_index.p, L.f_index.p,
                                                     L.c_rows.p, L.f_rows.p);
        PMGR_LAUNCHED();
        setup_trace("mgr split", li, s);
        // owned ranges of the level, F and C spaces (distributed setup)
        std::unique_ptr<DistSetup> dF, dC;
        if (dd) {
            dF.reset(new DistSetup(dd->with(ds_sub_bounds(dd->start, L.is_c.p, n, false, s))));
            dC.reset(new DistSetup(dd->with(ds_sub_bounds(dd->start, L.is_c.p, n, true, s))));
            if (sp.global_smoother != PMGR_SMOOTHER_NONE)
                fail(PMGR_ERR_NOT_SUPPORTED, "distributed setup of a level with a global smoother");
        }
        // ---- blocks (extract_blocks, sparse.py:269-288)
        const CsrView Av = cur->view();
        auto A_ff = std::make_shared<Csr>();
        Csr A_fc, A_cc;
        extract_block(Av, L.f_rows.p, L.nf, L.is_c.p, false, L.f_index.p, L.nf, *A_ff, s);
        extract_block(Av, L.f_rows.p, L.nf, L.is_c.p, true, c_index.p, L.nc, A_fc, s);
        extract_block(Av, L.c_rows.p, L.nc, L.is_c.p, false, L.f_index.p, L.nf, L.A_cf, s);
        if (sp.n_max >= 0) extract_block(Av, L.c_rows.p, L.nc, L.is_c.p, true, c_index.p, L.nc, A_cc, s);
        setup_trace("mgr blocks", li, s);
        // ---- transfers (build_transfers, mgr.py:131-187)
        const bool need_dinv = sp.interp == PMGR_INTERP_INJECTION_JACOBI || sp.f_relax == PMGR_FRELAX_JACOBI;
        // (the sliced jagged copy of A_FF is built from its block copy when it gets one)
        ds_finalize(dF.get(), *A_ff, s, false);
        if (sp.f_relax == PMGR_FRELAX_AMG && sp.amg_num_functions == 3)
            csr_make_bsr3(*A_ff, A_ff->nrows, A_ff->ncols, s, false, dF.get());
        if (!dd && !A_ff->sj) csr_make_sj(*A_ff, s);
        if (li == 0 && A_ff->nbrows > 0) {
            // F rows first, then C rows: the same blocks lead A0 itself
            // (the C rows are the last nc rows exactly when the first of them is row nf)
            const bool prefix = L.nc > 0 && read_scalar(L.c_rows.p, s) == L.nf;
            if (prefix) {
                h->block_prefix = L.nf;
                if (!dd) h->block_src = A_ff;
            }
        }
        ds_finalize(dC.get(), L.A_cf, s);
        if (need_dinv) {
            L.dinv_ff.alloc(L.nf);
            int64_t bad;
            if (dd) {  // owned F rows; the first singular row over all ranks
                bad = ds_diag_inverse(*A_ff, dF->lo(), dF->hi(), L.dinv_ff.p, s);
                const int64_t g = ds_allmax(*dd, bad < 0 ? INT64_MIN : -bad, s);
                bad = g == INT64_MIN ? -1 : -g;
            } else {
                bad = csr_diag_inverse(A_ff->view(), L.dinv_ff.p, s);
            }
            if (bad >= 0)
                fail(PMGR_ERR_SINGULAR_DIAG, "singular diagonal: zero or missing entry at row " + std::to_string(bad),
                     bad);
        }
        const int with_wp = sp.interp == PMGR_INTERP_INJECTION_JACOBI ? 1 : 0;
        {
            TBuf<int64_t> cnt(n, s);
            L.P.nrows = n;
            L.P.ncols = L.nc;
            L.P.ro.alloc(n + 1);
            const int64_t plo = dd ? dd->lo() : 0, phi = dd ? dd->hi() : n;
            PMGR_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t) * (size_t)(n > 0 ? n : 1), s));
            if (phi > plo) {
                k_build_p<false><<<grid_for((phi - plo) * 32, 256), 256, 0, s>>>(
                    plo, phi, L.is_c.p, c_index.p, L.f_index.p, A_fc.ro.p, A_fc.ci.p, A_fc.v.p, L.dinv_ff.p, with_wp,
                    cnt.p, nullptr, nullptr, nullptr);
                PMGR_LAUNCHED();
            }
            L.P.nnz = exclusive_scan_total(cnt.p, L.P.ro.p, n, s);
            L.P.ci.alloc(L.P.nnz);
            L.P.v.alloc(L.P.nnz);
            if (phi > plo) {
                k_build_p<true><<<grid_for((phi - plo) * 32, 256), 256, 0, s>>>(
                    plo, phi, L.is_c.p, c_index.p, L.f_index.p, A_fc.ro.p, A_fc.ci.p, A_fc.v.p, L.dinv_ff.p, with_wp,
                    nullptr, L.P.ro.p, L.P.ci.p, L.P.v.p);
                PMGR_LAUNCHED();
            }
        }
        ds_finalize(dd.get(), L.P, s);
        setup_trace("mgr transfers", li, s);
        // ---- F-relaxation (_build_f_relax, mgr.py:374-386)
        L.f_relax = sp.f_relax;
        L.f_relax_sweeps = sp.f_relax_sweeps > 1 ? sp.f_relax_sweeps : 1;
        if (sp.f_relax == PMGR_FRELAX_AMG) {
            pmgr_amg_cfg acfg = cfg.amg_f_relax;
            acfg.num_functions = sp.amg_num_functions > 0 ? sp.amg_num_functions : 1;
            L.amg = amg_build(A_ff, acfg, s, dF.get());
            L.amg->prof_tag = (li == 0);
        }
        if (sp.f_relax == PMGR_FRELAX_JACOBI && L.f_relax_sweeps > 1) L.A_ff = A_ff;
        setup_trace("mgr F-relax AMG", li, s);
        // ---- global smoother (_build_global_smoother, mgr.py:388-396)
        if (sp.global_smoother != PMGR_SMOOTHER_NONE) {
            L.smoother = smoother_build(cur, sp.global_smoother, sp.ilu_fill, sp.hbgs_sweeps,
                                        cfg.npartitions > 0 ? cfg.npartitions : 1, interleaved, fo.data(), eo.data(), s);
            rows_of(Av, L.c_rows.p, L.nc, L.A_c, s);
            csr_finalize(L.A_c, s);
            L.zs.alloc(n);
            L.rr.alloc(n);
            setup_trace("mgr global smoother", li, s);
        }
        // ---- coarse operator (build_coarse, mgr.py:212-231)
        auto coarse = std::make_shared<Csr>();
        {
            Csr RA, T;
            rows_of(Av, L.c_rows.p, L.nc, RA, s);
            // distributed: the rows of P behind RA's columns, fetched from their owners
            Csr Pext;
            if (dd) ds_fetch_rows(*dd, L.P, ds_cols_outside(RA, dC->lo(), dC->hi(), dd->lo(), dd->hi(), s), Pext, s);
            const CsrView Pv = dd ? Pext.view() : L.P.view();
            if (sp.n_max < 0) {
                spgemm(RA.view(), Pv, 1, *coarse, s);
            } else {
                spgemm(RA.view(), Pv, 1, T, s);
                Csr corr, kept;
                csr_subtract(A_cc.view(), T.view(), corr, s);
                TBuf<int32_t> ent(L.nc, s);
                TBuf<int8_t> fdummy(L.nc, s);
                k_restrict_layout<<<grid_for(L.nc, 256), 256, 0, s>>>(L.nc, L.c_rows.p, dfo.p, deo.p, fdummy.p, ent.p);
                PMGR_LAUNCHED();
                csr_sparsify(corr.view(), ent.p, sp.n_max, kept, s);
                csr_subtract(A_cc.view(), kept.view(), *coarse, s);
                PMGR_CUDA(cudaStreamSynchronize(s));
            }
        }
        ds_finalize(dC.get(), *coarse, s);
        setup_trace("mgr coarse RAP", li, s);
        // ---- workspace
        L.vf.alloc(L.nf);
        L.zf.alloc(L.nf);
        L.rc.alloc(L.nc);
        L.zc.alloc(L.nc);
        L.tmpf.alloc(n > L.nf ? n : L.nf);
        // ---- next layout
        {
            TBuf<int8_t> dfo2(L.nc, s);
            TBuf<int32_t> deo2(L.nc, s);
            if (L.nc > 0) {
                k_restrict_layout<<<grid_for(L.nc, 256), 256, 0, s>>>(L.nc, L.c_rows.p, dfo.p, deo.p, dfo2.p, deo2.p);
                PMGR_LAUNCHED();
            }
            dfo = std::move(dfo2);
            deo = std::move(deo2);
        }
        if (any_smoother) {
            std::vector<int8_t> fo2;
            std::vector<int32_t> eo2;
            fo2.reserve((size_t)L.nc);
            eo2.reserve((size_t)L.nc);
            for (int64_t i = 0; i < n; ++i)
                if ((sp.c_mask >> (fo[i] & 63)) & 1ull) {
                    fo2.push_back(fo[i]);
                    eo2.push_back(eo[i]);
                }
            fo.swap(fo2);
            eo.swap(eo2);
        }
        h->levels.push_back(std::move(L));
        cur = coarse;
        if (dd) dd->start = dC->start;
        PMGR_CUDA(cudaStreamSynchronize(s));
    }
    h->terminal_A = cur;
    h->terminal = amg_build(cur, cfg.amg_terminal, s, dd.get());
    h->tz.alloc(cur->nrows);
    PMGR_CUDA(cudaStreamSynchronize(s));
    return h;
}

void mgr_apply(pmgr_mgr &h, const double *v, double *z, cudaStream_t s) {
    if (!h.use_graphs) {
        apply_level(h, 0, v, z, s);
        return;
    }
    // one CUDA graph per (v, z) pair: ~100 small launches of the multilevel
    // cycle replay back to back instead of paying host launch latency each
    const bool prof = prof_on();
    ApplyGraph *g = nullptr;
    for (auto &e : h.graphs)
        if (e.v == v && e.z == z && e.prof == prof) g = &e;
    if (!g) {
        if (h.graphs.size() >= 8) {
            auto old = h.graphs.begin();
            for (auto it = h.graphs.begin(); it != h.graphs.end(); ++it)
                if (it->last_use < old->last_use) old = it;
            if (old->pending) prof_collect(old->recs);
            prof_release(old->recs);
            cudaGraphExecDestroy(old->exec);
            h.graphs.erase(old);
        }
        if (!h.cap_stream) PMGR_CUDA(cudaStreamCreateWithFlags(&h.cap_stream, cudaStreamNonBlocking));
        h.graphs.emplace_back();
        g = &h.graphs.back();
        g->v = v;
        g->z = z;
        g->prof = prof;
        cudaGraph_t graph;
        PMGR_CUDA(cudaStreamBeginCapture(h.cap_stream, cudaStreamCaptureModeThreadLocal));
        if (prof) prof_capture_begin(&g->recs);
        g_capture_count = &g->kernels;
        try {
            apply_level(h, 0, v, z, h.cap_stream);
        } catch (...) {
            g_capture_count = nullptr;
            prof_capture_end();
            cudaStreamEndCapture(h.cap_stream, &graph);
            throw;
        }
        g_capture_count = nullptr;
        prof_capture_end();
        PMGR_CUDA(cudaStreamEndCapture(h.cap_stream, &graph));
        PMGR_CUDA(cudaGraphInstantiate(&g->exec, graph, 0));
        PMGR_CUDA(cudaGraphDestroy(graph));
    }
    if (g->pending) {
        prof_collect(g->recs);
        g->pending = false;
    }
    g->last_use = ++h.tick;
    PMGR_CUDA(cudaGraphLaunch(g->exec, s));
    g_launches.fetch_add(g->kernels, std::memory_order_relaxed);
    g->pending = g->prof;
}

void mgr_apply_direct(pmgr_mgr &h, const double *v, double *z, cudaStream_t s) { apply_level(h, 0, v, z, s); }

// algorithmic bytes and kernel count of one application: a dry capture of
// the cycle (nothing executes) with the byte ledger attached
void mgr_apply_bytes(pmgr_mgr &h, double *bytes, int64_t *kernels) {
    DBuf<double> v(h.n), z(h.n);
    cudaStream_t cs;
    PMGR_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t graph = nullptr;
    double b = 0.0;
    int64_t k = 0;
    PMGR_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    g_byte_ledger = &b;
    g_capture_count = &k;
    try {
        apply_level(h, 0, v.p, z.p, cs);
    } catch (...) {
        g_byte_ledger = nullptr;
        g_capture_count = nullptr;
        cudaStreamEndCapture(cs, &graph);
        if (graph) cudaGraphDestroy(graph);
        cudaStreamDestroy(cs);
        throw;
    }
    g_byte_ledger = nullptr;
    g_capture_count = nullptr;
    PMGR_CUDA(cudaStreamEndCapture(cs, &graph));
    PMGR_CUDA(cudaGraphDestroy(graph));
    PMGR_CUDA(cudaStreamDestroy(cs));
    *bytes = b;
    *kernels = k;
}

void mgr_collect(pmgr_mgr &h) {
    for (auto &e : h.graphs)
        if (e.pending) {
            prof_collect(e.recs);
            e.pending = false;
        }
}

}  // namespace pmgr

pmgr_mgr::~pmgr_mgr() {
    for (auto &e : graphs) {
        pmgr::prof_release(e.recs);
        if (e.exec) cudaGraphExecDestroy(e.exec);
    }
    if (cap_stream) cudaStreamDestroy(cap_stream);
}

namespace pmgr {

}  // namespace pmgr
