// capi.cu -- the extern "C" surface declared in include/pmgr.h.
//
// Every entry point catches pmgr::Error and converts it into a status code
// plus a thread-local message / row index that the Python layer turns back
// into the reference's exception (ValueError / RuntimeError / ...).
#include <mutex>
#include <cstring>
#include <string>

#include "dist.cuh"
#include "dsetup.cuh"

namespace {
thread_local std::string g_msg;
thread_local int64_t g_index = -1;

int set_error(const pmgr::Error &e) {
    g_msg = e.msg;
    g_index = e.index;
    return (int)e.code;
}

template <class F>
int guard(F &&f) {
    try {
        f();
        return PMGR_OK;
    } catch (const pmgr::Error &e) {
        return set_error(e);
    } catch (const std::bad_alloc &) {
        g_msg = "host allocation failed";
        g_index = -1;
        return PMGR_ERR_OOM;
    } catch (const std::exception &e) {
        g_msg = e.what();
        g_index = -1;
        return PMGR_ERR_CUDA;
    }
}

cudaStream_t S(void *p) { return (cudaStream_t)p; }

void require(bool ok, const char *msg) {
    if (!ok) pmgr::fail(PMGR_ERR_INVALID, msg);
}

void init_pool() {
    static bool done = false;
    if (done) return;
    int dev = 0;
    PMGR_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    PMGR_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = UINT64_MAX;
    PMGR_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    done = true;
}

pmgr_csr *wrap(std::shared_ptr<pmgr::Csr> m) {
    auto *h = new pmgr_csr;
    h->m = std::move(m);
    return h;
}

const pmgr::AmgLevel &amg_level(const pmgr_amg *h, int32_t level) {
    if (level < 0 || level >= (int32_t)h->levels.size()) pmgr::fail(PMGR_ERR_INVALID, "AMG level out of range");
    return h->levels[level];
}
}  // namespace

namespace {
// per-thread grow-only pinned staging buffer for the host-array GMRES entry
struct PinnedStage {
    void *p = nullptr;
    size_t cap = 0;
    ~PinnedStage() {
        if (p) cudaFreeHost(p);
    }
};
double *pinned_stage(size_t bytes) {
    thread_local PinnedStage st;
    if (st.cap < bytes) {
        if (st.p) cudaFreeHost(st.p);
        st.p = nullptr;
        st.cap = 0;
        PMGR_CUDA(cudaMallocHost(&st.p, bytes));
        st.cap = bytes;
    }
    return static_cast<double *>(st.p);
}
bool is_pinned(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}
}  // namespace

extern "C" {

int pmgr_version(void) { return 1; }
const char *pmgr_last_error(void) { return g_msg.c_str(); }
int64_t pmgr_last_error_index(void) { return g_index; }
int64_t pmgr_launch_count(void) { return pmgr::g_launches.load(); }

int pmgr_csr_create(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t *row_offsets,
                    const int32_t *col_indices, const double *values, int on_device, int validate,
                    void *stream, pmgr_csr **out) {
    return guard([&] {
        require(out != nullptr, "out handle is NULL");
        require(nrows >= 0 && ncols >= 0 && nnz >= 0, "negative dimension");
        require(nnz < (int64_t)2147483647, "nnz exceeds the per-device int32 limit");
        init_pool();
        auto m = std::make_shared<pmgr::Csr>();
        m->alloc(nrows, ncols, nnz);
        cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        PMGR_CUDA(cudaMemcpyAsync(m->ro.p, row_offsets, sizeof(int64_t) * (nrows + 1), k, S(stream)));
        if (nnz) {
            PMGR_CUDA(cudaMemcpyAsync(m->ci.p, col_indices, sizeof(int32_t) * nnz, k, S(stream)));
            PMGR_CUDA(cudaMemcpyAsync(m->v.p, values, sizeof(double) * nnz, k, S(stream)));
        }
        if (validate) pmgr::csr_validate(m->view(), S(stream));
        pmgr::csr_finalize(*m, S(stream), false);  // sliced jagged copy: at first use (ensure_sj)
        PMGR_CUDA(cudaStreamSynchronize(S(stream)));
        *out = wrap(std::move(m));
    });
}

int pmgr_csr_destroy(pmgr_csr *A) {
    return guard([&] {
        pmgr::gmres_forget(A);
        delete A;
    });
}

int pmgr_csr_info(const pmgr_csr *A, int64_t *nrows, int64_t *ncols, int64_t *nnz) {
    return guard([&] {
        require(A != nullptr, "NULL matrix");
        if (nrows) *nrows = A->m->nrows;
        if (ncols) *ncols = A->m->ncols;
        if (nnz) *nnz = A->m->nnz;
    });
}

int pmgr_csr_download(const pmgr_csr *A, int64_t *row_offsets, int32_t *col_indices, double *values,
                      int to_device, void *stream) {
    return guard([&] {
        require(A != nullptr, "NULL matrix");
        const pmgr::Csr &m = *A->m;
        cudaMemcpyKind k = to_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        if (row_offsets)
            PMGR_CUDA(cudaMemcpyAsync(row_offsets, m.ro.p, sizeof(int64_t) * (m.nrows + 1), k, S(stream)));
        if (m.nnz && col_indices)
            PMGR_CUDA(cudaMemcpyAsync(col_indices, m.ci.p, sizeof(int32_t) * m.nnz, k, S(stream)));
        if (m.nnz && values) PMGR_CUDA(cudaMemcpyAsync(values, m.v.p, sizeof(double) * m.nnz, k, S(stream)));
        PMGR_CUDA(cudaStreamSynchronize(S(stream)));
    });
}

// A caller's matrix gets its sliced jagged solve copy when it is first
// applied: MGR setup builds it from the block-prefix copy; a matrix used
// without one (matvec, AMG level 0, unpreconditioned GMRES) builds it here.
static void ensure_sj(const pmgr_csr *A, void *stream) {
    static std::mutex mu;  // two threads may apply the same matrix for the first time
    std::lock_guard<std::mutex> lock(mu);
    pmgr::Csr &m = *A->m;
    if (m.sj_want && !m.sj && !m.sj_tried) {
        pmgr::csr_make_sj(m, S(stream));
        PMGR_CUDA(cudaStreamSynchronize(S(stream)));
        m.sj_tried = true;  // one attempt per layout
    }
}

int pmgr_spmv(const pmgr_csr *A, const double *x_dev, double *y_dev, void *stream) {
    return guard([&] {
        require(A != nullptr, "NULL matrix");
        ensure_sj(A, stream);
        pmgr::spmv(A->m->view(), x_dev, y_dev, S(stream));
    });
}

// ---------------------------------------------------------------- AMG
int pmgr_amg_setup(const pmgr_csr *A, const pmgr_amg_cfg *cfg, void *stream, pmgr_amg **out) {
    return guard([&] {
        require(A && cfg && out, "NULL argument");
        init_pool();
        ensure_sj(A, stream);
        auto h = pmgr::amg_build(A->m, *cfg, S(stream));
        *out = h.release();
    });
}

int pmgr_amg_destroy(pmgr_amg *h) {
    return guard([&] { delete h; });
}

int pmgr_amg_num_levels(const pmgr_amg *h, int32_t *nlevels) {
    return guard([&] { *nlevels = (int32_t)h->levels.size(); });
}

int pmgr_amg_level_sizes(const pmgr_amg *h, int64_t *sizes) {
    return guard([&] {
        size_t i = 0;
        for (; i < h->levels.size(); ++i) sizes[i] = h->levels[i].A->nrows;
        sizes[i] = h->coarse->nrows;
    });
}

int pmgr_amg_flagged_rows(const pmgr_amg *h, int64_t *flagged) {
    return guard([&] { *flagged = h->flagged; });
}

int pmgr_amg_vcycle(pmgr_amg *h, const double *b_dev, const double *x_dev, double *out_dev, void *stream) {
    return guard([&] {
        require(h != nullptr, "NULL hierarchy");
        pmgr::amg_cycle(*h, b_dev, x_dev, out_dev, S(stream));
    });
}

int pmgr_amg_export_csr(const pmgr_amg *h, int32_t level, int32_t what, void *stream, pmgr_csr **out) {
    return guard([&] {
        auto m = std::make_shared<pmgr::Csr>();
        if (what == 2) {
            pmgr::csr_copy(h->coarse->view(), *m, S(stream));
        } else {
            const pmgr::AmgLevel &L = amg_level(h, level);
            pmgr::csr_copy(what == 0 ? L.A->view() : L.P.view(), *m, S(stream));
        }
        pmgr::csr_finalize(*m, S(stream), false);  // an exported operator is a matrix like any other
        PMGR_CUDA(cudaStreamSynchronize(S(stream)));
        *out = wrap(std::move(m));
    });
}

int pmgr_amg_export_vec(const pmgr_amg *h, int32_t level, int32_t what, void *host_out, void *stream) {
    return guard([&] {
        const pmgr::AmgLevel &L = amg_level(h, level);
        const int64_t n = L.A->nrows;
        if (what == 0)
            PMGR_CUDA(cudaMemcpyAsync(host_out, L.is_c.p, n, cudaMemcpyDeviceToHost, S(stream)));
        else
            PMGR_CUDA(cudaMemcpyAsync(host_out, L.dtilde.p, sizeof(double) * n, cudaMemcpyDeviceToHost, S(stream)));
        PMGR_CUDA(cudaStreamSynchronize(S(stream)));
    });
}

// ---------------------------------------------------------------- MGR
int pmgr_mgr_setup(const pmgr_csr *A, const int8_t *field_of, const int32_t *entity_of,
                   const pmgr_level_spec *levels, int32_t nlevels, const pmgr_mgr_cfg *cfg, void *stream,
                   pmgr_mgr **out) {
    return guard([&] {
        require(A && field_of && entity_of && cfg && out, "NULL argument");
        require(nlevels >= 0 && (nlevels == 0 || levels), "bad level list");
        init_pool();
        auto h = pmgr::mgr_build(A->m, field_of, entity_of, levels, nlevels, *cfg, S(stream));
        // solve-phase block copy of A0 for the Krylov SpMV (node-blocked F prefix)
        if (h->block_prefix > 0 && A->m->nbrows == 0) {
            static const bool share = !(getenv("PMGR_NO_BSR_SHARE") && getenv("PMGR_NO_BSR_SHARE")[0] != '0');
            if (share && h->block_src)
                pmgr::csr_make_bsr3_shared(*A->m, h->block_prefix, h->block_src, S(stream));
            else
                pmgr::csr_make_bsr3(*A->m, h->block_prefix, h->block_prefix, S(stream));
            PMGR_CUDA(cudaStreamSynchronize(S(stream)));
        }
        ensure_sj(A, stream);
        pmgr::setup_trace("mgr A0 solve copies", -1, S(stream));
        pmgr::host_trace_report("mgr_setup");
        *out = h.release();
    });
}

int pmgr_mgr_destroy(pmgr_mgr *h) {
    return guard([&] {
        pmgr::gmres_forget(h);
        delete h;
    });
}

int pmgr_mgr_num_levels(const pmgr_mgr *h, int32_t *nlevels) {
    return guard([&] { *nlevels = (int32_t)h->levels.size(); });
}

int pmgr_mgr_apply_bytes(pmgr_mgr *h, double *bytes, int64_t *kernels) {
    return guard([&] { pmgr::mgr_apply_bytes(*h, bytes, kernels); });
}

int pmgr_mgr_level_sizes(const pmgr_mgr *h, int64_t *sizes) {
    return guard([&] {
        size_t i = 0;
        for (; i < h->levels.size(); ++i) sizes[i] = h->levels[i].n;
        sizes[i] = h->terminal_A->nrows;
    });
}

int pmgr_mgr_apply(pmgr_mgr *h, const double *v_dev, double *z_dev, void *stream) {
    return guard([&] {
        require(h != nullptr, "NULL hierarchy");
        pmgr::mgr_apply(*h, v_dev, z_dev, S(stream));
    });
}

int pmgr_mgr_export_csr(const pmgr_mgr *h, int32_t level, int32_t what, void *stream, pmgr_csr **out) {
    return guard([&] {
        require(level >= 0 && level < (int32_t)h->levels.size(), "MGR level out of range");
        auto m = std::make_shared<pmgr::Csr>();
        if (what == 0) {
            pmgr::csr_copy(h->levels[level].P.view(), *m, S(stream));
        } else if (what == 2) {
            const auto &g = h->levels[level].smoother;
            require(g && g->kind == PMGR_SMOOTHER_ILU, "level has no ILU smoother");
            pmgr::csr_copy(g->lu.view(), *m, S(stream));
        } else {
            const pmgr::Csr &nx = (level + 1 < (int32_t)h->levels.size()) ? *h->levels[level + 1].A : *h->terminal_A;
            pmgr::csr_copy(nx.view(), *m, S(stream));
        }
        pmgr::csr_finalize(*m, S(stream), false);
        PMGR_CUDA(cudaStreamSynchronize(S(stream)));
        *out = wrap(std::move(m));
    });
}

int pmgr_mgr_export_vec(const pmgr_mgr *h, int32_t level, int32_t what, void *host_out, void *stream) {
    return guard([&] {
        require(level >= 0 && level < (int32_t)h->levels.size(), "MGR level out of range");
        require(what == 0, "unknown vector");
        const pmgr::MgrLevel &L = h->levels[level];
        PMGR_CUDA(cudaMemcpyAsync(host_out, L.is_c.p, L.n, cudaMemcpyDeviceToHost, S(stream)));
        PMGR_CUDA(cudaStreamSynchronize(S(stream)));
    });
}

int pmgr_mgr_amg(const pmgr_mgr *h, int32_t level, const pmgr_amg **out) {
    return guard([&] {
        if (level < 0) {
            *out = h->terminal.get();
        } else {
            require(level < (int32_t)h->levels.size(), "MGR level out of range");
            *out = h->levels[level].amg.get();
        }
    });
}

// ---------------------------------------------------------------- GMRES
int pmgr_gmres(const pmgr_csr *A, pmgr_mgr *M, const double *b_dev, double *x_dev, int nonzero_x0,
               const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats, double *history_host, int32_t history_cap,
               void *stream) {
    return guard([&] {
        require(A && cfg && stats && b_dev && x_dev, "NULL argument");
        require(cfg->restart <= 1000, "restart above 1000 is not supported");
        ensure_sj(A, stream);
        pmgr::gmres_device(A, M, b_dev, x_dev, nonzero_x0, *cfg, *stats, history_host, history_cap, S(stream));
    });
}

int pmgr_gmres_host(const pmgr_csr *A, pmgr_mgr *M, const double *b_host, double *x_host, int nonzero_x0,
                    const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats, double *history_host,
                    int32_t history_cap, void *stream) {
    return guard([&] {
        require(A && cfg && stats && b_host && x_host, "NULL argument");
        require(cfg->restart <= 1000, "restart above 1000 is not supported");
        ensure_sj(A, stream);
        const int64_t n = A->m->nrows;
        const size_t bytes = sizeof(double) * (size_t)n;
        pmgr::TBuf<double> b(n, S(stream)), x(n, S(stream));
        // pageable caller arrays go through a pinned staging buffer (one host
        // memcpy + a DMA at full link speed instead of the driver's chunked
        // pageable path); pinned ones are copied directly
        double *stage = pinned_stage(bytes);
        auto h2d = [&](double *dst, const double *src) {
            if (is_pinned(src)) {
                PMGR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, S(stream)));
            } else {
                PMGR_CUDA(cudaStreamSynchronize(S(stream)));  // the stage is free
                std::memcpy(stage, src, bytes);
                PMGR_CUDA(cudaMemcpyAsync(dst, stage, bytes, cudaMemcpyHostToDevice, S(stream)));
            }
        };
        h2d(b.p, b_host);
        if (nonzero_x0) h2d(x.p, x_host);
        else PMGR_CUDA(cudaMemsetAsync(x.p, 0, bytes, S(stream)));
        pmgr::gmres_device(A, M, b.p, x.p, nonzero_x0, *cfg, *stats, history_host, history_cap, S(stream));
        if (is_pinned(x_host)) {
            PMGR_CUDA(cudaMemcpyAsync(x_host, x.p, bytes, cudaMemcpyDeviceToHost, S(stream)));
            PMGR_CUDA(cudaStreamSynchronize(S(stream)));
        } else {
            PMGR_CUDA(cudaMemcpyAsync(stage, x.p, bytes, cudaMemcpyDeviceToHost, S(stream)));
            PMGR_CUDA(cudaStreamSynchronize(S(stream)));
            std::memcpy(x_host, stage, bytes);
        }
    });
}

int pmgr_release_cached_memory(void) {
    return guard([&] {
        PMGR_CUDA(cudaDeviceSynchronize());
        pmgr::dbuf_trim();
    });
}

int pmgr_prof_enable(int on) {
    return guard([&] { pmgr::prof_enable(on != 0); });
}

int pmgr_prof_query(int32_t kind, int64_t *count, double *ms, double *bytes) {
    return guard([&] {
        require(kind >= 0 && kind < pmgr::PROF_KINDS, "unknown profile kind");
        pmgr::prof_query(kind, count, ms, bytes);
    });
}

int pmgr_multidot(const double *V_dev, int64_t n, int32_t nvec, const double *w_dev, double *h_dev, void *stream) {
    return guard([&] { pmgr::multidot(V_dev, n, nvec, w_dev, h_dev, S(stream)); });
}

int pmgr_multiaxpy(const double *V_dev, int64_t n, int32_t nvec, const double *h_dev, double *w_dev,
                   void *stream) {
    return guard([&] { pmgr::multiaxpy(V_dev, n, nvec, h_dev, w_dev, S(stream)); });
}

int pmgr_vec_norm2(const double *x_dev, int64_t n, double *out_host, void *stream) {
    return guard([&] { *out_host = pmgr::vec_norm2(x_dev, n, S(stream)); });
}

int pmgr_vec_axpby(double a, const double *x_dev, double b, double *y_dev, int64_t n, void *stream) {
    return guard([&] { pmgr::vec_axpby(a, x_dev, b, y_dev, n, S(stream)); });
}

int pmgr_combine(const double *V_dev, int64_t n, int64_t ldv, int32_t nvec, const double *y_dev, double *u_dev,
                 void *stream) {
    return guard([&] { pmgr::vec_combine(V_dev, n, ldv, nvec, y_dev, u_dev, S(stream)); });
}

}  // extern "C"

// ---------------------------------------------------------------- distribution

struct pmgr_transport {
    std::unique_ptr<pmgr::Transport> t;
};
struct pmgr_dist {
    std::unique_ptr<pmgr::DistSolver> d;
};

int pmgr_nccl_get_id(pmgr_nccl_id *out) {
    return guard([&] {
        require(out, "NULL argument");
        pmgr::nccl_unique_id(out);
    });
}

int pmgr_transport_nccl_create(const pmgr_nccl_id *id, int32_t rank, int32_t nranks, pmgr_transport **out) {
    return guard([&] {
        require(id && out, "NULL argument");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
        auto *t = new pmgr_transport;
        t->t = pmgr::make_nccl_transport(*id, rank, nranks);
        *out = t;
    });
}

int pmgr_transport_host_create(int32_t rank, int32_t nranks, pmgr_alltoallv_fn alltoallv,
                               pmgr_allreduce_fn allreduce, void *ctx, pmgr_transport **out) {
    return guard([&] {
        require(out && alltoallv && allreduce, "NULL argument");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / nranks");
        auto *t = new pmgr_transport;
        t->t = pmgr::make_callback_transport(rank, nranks, alltoallv, allreduce, ctx);
        *out = t;
    });
}

int pmgr_transport_destroy(pmgr_transport *t) {
    return guard([&] { delete t; });
}

int pmgr_dist_create(const pmgr_csr *A, pmgr_mgr *M, const int64_t *bounds, int32_t rank, int32_t nranks,
                     pmgr_transport *t, void *stream, pmgr_dist **out) {
    return guard([&] {
        require(A && M && bounds && out, "NULL argument");
        require(nranks == 1 || t, "a transport is required for more than one rank");
        init_pool();
        auto *d = new pmgr_dist;
        try {
            d->d = pmgr::dist_build(A, M, bounds, rank, nranks, t ? t->t.get() : nullptr, S(stream));
        } catch (...) {
            delete d;
            throw;
        }
        *out = d;
    });
}

int pmgr_dist_info(const pmgr_dist *d, int64_t *lo, int64_t *n_own) {
    return guard([&] {
        require(d && lo && n_own, "NULL argument");
        *lo = d->d->lo;
        *n_own = d->d->n_own;
    });
}

int pmgr_dist_apply(pmgr_dist *d, const double *v_own_dev, double *z_own_dev, void *stream) {
    return guard([&] {
        require(d && (d->d->n_own == 0 || (v_own_dev && z_own_dev)), "NULL argument");
        pmgr::dist_apply(*d->d, v_own_dev, z_own_dev, S(stream));
    });
}

int pmgr_dist_spmv(pmgr_dist *d, const double *x_own_dev, double *y_own_dev, void *stream) {
    return guard([&] {
        require(d && (d->d->n_own == 0 || (x_own_dev && y_own_dev)), "NULL argument");
        pmgr::DistSolver &D = *d->d;
        D.ensure_work();
        if (D.n_own > 0)
            PMGR_CUDA(cudaMemcpyAsync(D.ze.p + D.off, x_own_dev, sizeof(double) * D.n_own, cudaMemcpyDeviceToDevice,
                                      S(stream)));
        pmgr::halo_exchange(D.halo0.get(), D.ze.p, S(stream));
        pmgr::spmv(D.A.view(), D.ze.p, D.we.p, S(stream));
        if (D.n_own > 0)
            PMGR_CUDA(cudaMemcpyAsync(y_own_dev, D.we.p + D.off, sizeof(double) * D.n_own, cudaMemcpyDeviceToDevice,
                                      S(stream)));
    });
}

int pmgr_dist_gmres(pmgr_dist *d, const double *b_own_dev, double *x_own_dev, int nonzero_x0,
                    const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats, double *history_host, int32_t history_cap,
                    void *stream) {
    return guard([&] {
        require(d && cfg && stats, "NULL argument");
        require(d->d->n_own == 0 || (b_own_dev && x_own_dev), "NULL argument");
        pmgr::dist_gmres(*d->d, b_own_dev, x_own_dev, nonzero_x0, *cfg, *stats, history_host, history_cap,
                         S(stream));
    });
}

int pmgr_dist_destroy(pmgr_dist *d) {
    return guard([&] { delete d; });
}

int pmgr_dist_emulate(const pmgr_csr *A, pmgr_mgr *M, const int64_t *bounds, int32_t nranks, int32_t what,
                      const double *in_dev, double *out_dev, const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats,
                      void *stream) {
    return guard([&] {
        require(A && M && bounds && in_dev && out_dev, "NULL argument");
        require(what == 0 || (cfg && stats), "NULL argument");
        require(nranks >= 1, "nranks must be positive");
        init_pool();
        pmgr::dist_emulate(A, M, bounds, nranks, what, in_dev, out_dev, cfg, stats, S(stream));
    });
}

int pmgr_dist_setup(const pmgr_csr *A_rows, const int8_t *field_of, const int32_t *entity_of,
                    const pmgr_level_spec *levels, int32_t nlevels, const pmgr_mgr_cfg *cfg, const int64_t *bounds,
                    int32_t rank, int32_t nranks, pmgr_transport *t, void *stream, pmgr_dist **out) {
    return guard([&] {
        require(A_rows && field_of && entity_of && cfg && bounds && out, "NULL argument");
        require(nlevels >= 0 && (nlevels == 0 || levels), "bad level list");
        require(nranks == 1 || t, "a transport is required for more than one rank");
        init_pool();
        auto *d = new pmgr_dist;
        try {
            d->d = pmgr::dist_setup(A_rows, field_of, entity_of, levels, nlevels, *cfg, bounds, rank, nranks,
                                    t ? t->t.get() : nullptr, S(stream));
        } catch (...) {
            delete d;
            throw;
        }
        *out = d;
    });
}

int pmgr_dist_setup_emulate(const pmgr_csr *A, const int8_t *field_of, const int32_t *entity_of,
                            const pmgr_level_spec *levels, int32_t nlevels, const pmgr_mgr_cfg *mcfg,
                            const int64_t *bounds, int32_t nranks, int32_t what, const double *in_dev, double *out_dev,
                            const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats, void *stream) {
    return guard([&] {
        require(A && field_of && entity_of && mcfg && bounds && in_dev && out_dev, "NULL argument");
        require(nlevels >= 0 && (nlevels == 0 || levels), "bad level list");
        require(what == 0 || (cfg && stats), "NULL argument");
        require(nranks >= 1, "nranks must be positive");
        init_pool();
        pmgr::dist_setup_emulate(A, field_of, entity_of, levels, nlevels, *mcfg, bounds, nranks, what, in_dev, out_dev,
                                 cfg, stats, S(stream));
    });
}

// ---------------------------------------------------------------- assembly

int pmgr_assemble_poromech(const pmgr_assembly *a, void *stream, pmgr_csr **out) {
    return guard([&] {
        require(a && out && a->E && a->kx && a->ky && a->kz && a->pstate && a->K0 && a->bvec, "NULL argument");
        require(a->phases == 1 || a->sats, "NULL saturations");
        init_pool();
        *out = wrap(pmgr::assemble_poromech(*a, S(stream)));
    });
}

int pmgr_csr_rows(const pmgr_csr *A, int64_t lo, int64_t hi, void *stream, pmgr_csr **out) {
    return guard([&] {
        require(A && out, "NULL argument");
        require(lo >= 0 && lo <= hi && hi <= A->m->nrows, "row range out of bounds");
        auto m = std::make_shared<pmgr::Csr>();
        pmgr::ds_partial_rows(*A->m, lo, hi, *m, S(stream));
        pmgr::csr_finalize(*m, S(stream), false);
        *out = wrap(m);
    });
}

int pmgr_csr_permute(const pmgr_csr *A, const int64_t *perm_host, void *stream, pmgr_csr **out) {
    return guard([&] {
        require(A && perm_host && out, "NULL argument");
        *out = wrap(pmgr::csr_permute(*A->m, perm_host, S(stream)));
    });
}
