// krylov.cu -- right-preconditioned restarted GMRES on the device
// (reference krylov.py:39-117).
//
// Same outer semantics as the reference: x0 = 0 unless given; convergence
// on ||b - A x|| <= max(rtol*||r0||, atol); Givens least squares; at each
// restart x += M^{-1}(V y), the true residual is recomputed and replaces the
// last history entry; an Arnoldi breakdown counts as convergence in the
// subspace.  Orthogonalisation is classical Gram-Schmidt with one
// re-orthogonalisation (CGS2) instead of MGS: the projections become two
// fused multi-dot / multi-axpy passes over the Krylov basis (HBM streaming,
// deterministic block partials) -- not bitwise MGS, but at least as
// orthogonal, which keeps iteration counts within +-1.
// The small Hessenberg / Givens work runs in one single-thread kernel; the
// host only reads three status words per iteration.
#include <cmath>

#include "hier.cuh"

namespace pmgr {

namespace {

constexpr int DOT_BLOCK = 256;
constexpr int KC = 8;  // basis vectors per register chunk

int dot_grid(int64_t n) {
    int64_t g = (n + DOT_BLOCK - 1) / DOT_BLOCK;
    int64_t cap = 2LL * num_sms();
    return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}

__device__ __forceinline__ double block_sum(double v, double *sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
    return t;  // valid in thread 0
}

// partial[blk*ld + k] = sum over this block's rows of V_k[i] * w[i], k < nk
__global__ void __launch_bounds__(DOT_BLOCK) k_multidot(const double *__restrict__ V, int64_t n, int nk,
                                                         const double *__restrict__ w, double *partial, int ld) {
    __shared__ double sh[DOT_BLOCK / 32];
    for (int k0 = 0; k0 < nk; k0 += KC) {
        double acc[KC];
#pragma unroll
        for (int t = 0; t < KC; ++t) acc[t] = 0.0;
        for (int64_t i = blockIdx.x * (int64_t)DOT_BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * DOT_BLOCK) {
            const double wi = w[i];
#pragma unroll
            for (int t = 0; t < KC; ++t)
                if (k0 + t < nk) acc[t] = fma(V[(int64_t)(k0 + t) * n + i], wi, acc[t]);
        }
#pragma unroll
        for (int t = 0; t < KC; ++t) {
            if (k0 + t >= nk) break;
            double s = block_sum(acc[t], sh);
            if (threadIdx.x == 0) partial[(int64_t)blockIdx.x * ld + k0 + t] = s;
        }
    }
}

// w -= sum_k h[k] V_k ; then mode 1: partial dots V_k . w (k < nk),
// mode 2: partial ||w||^2 (slot 0).  Each thread re-reads its rows of V
// for the dots (L1-resident tile).
__global__ void __launch_bounds__(DOT_BLOCK) k_update(const double *__restrict__ V, int64_t n, int nk,
                                                       const double *__restrict__ h, double *w, int mode,
                                                       double *partial, int ld) {
    __shared__ double sh[DOT_BLOCK / 32];
    __shared__ double hs[1024];
    for (int k = threadIdx.x; k < nk && k < 1024; k += DOT_BLOCK) hs[k] = h[k];
    __syncthreads();
    double nrm = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)DOT_BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * DOT_BLOCK) {
        double wi = w[i];
        for (int k = 0; k < nk; ++k) wi = fma(-hs[k], V[(int64_t)k * n + i], wi);
        w[i] = wi;
        nrm = fma(wi, wi, nrm);
    }
    if (mode == 2) {
        double s = block_sum(nrm, sh);
        if (threadIdx.x == 0) partial[(int64_t)blockIdx.x * ld] = s;
        return;
    }
    if (mode == 1) {
        for (int k0 = 0; k0 < nk; k0 += KC) {
            double acc[KC];
#pragma unroll
            for (int t = 0; t < KC; ++t) acc[t] = 0.0;
            for (int64_t i = blockIdx.x * (int64_t)DOT_BLOCK + threadIdx.x; i < n;
                 i += (int64_t)gridDim.x * DOT_BLOCK) {
                const double wi = w[i];
#pragma unroll
                for (int t = 0; t < KC; ++t)
                    if (k0 + t < nk) acc[t] = fma(V[(int64_t)(k0 + t) * n + i], wi, acc[t]);
            }
#pragma unroll
            for (int t = 0; t < KC; ++t) {
                if (k0 + t >= nk) break;
                double s = block_sum(acc[t], sh);
                if (threadIdx.x == 0) partial[(int64_t)blockIdx.x * ld + k0 + t] = s;
            }
        }
    }
}

// out[k] (+)= sum over blocks of partial[b*ld + k], one warp per k, fixed order
__global__ void k_reduce_partials(const double *partial, int nblk, int nk, int ld, double *out, int accumulate) {
    int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (k >= nk) return;
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += partial[(int64_t)b * ld + k];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0) out[k] = accumulate ? out[k] + s : s;
}

// u = sum_k y[k] V_k
__global__ void k_combine(const double *__restrict__ V, int64_t n, int nk, const double *__restrict__ y,
                          double *u) {
    __shared__ double ys[1024];
    for (int k = threadIdx.x; k < nk && k < 1024; k += blockDim.x) ys[k] = y[k];
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = 0; k < nk; ++k) s = fma(ys[k], V[(int64_t)k * n + i], s);
        u[i] = s;
    }
}

__global__ void k_scale(const double *x, int64_t n, const double *den, double *y, double *y2) {
    const double d = *den;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double t = x[i] / d;
        y[i] = t;
        if (y2) y2[i] = t;
    }
}

__global__ void k_sqrt(double *x) { *x = sqrt(*x); }

// ---- classical Gram-Schmidt with DGKS re-orthogonalisation ---------------
// Pass 1 (k_mdot): h_k = V_k . w for k < nk and ||w||^2, one block per
// (row range, vector) so every block streams one contiguous slice of V.
// Pass 2 (k_upd): w -= sum_k h_k V_k with ||w'||^2 partials.  A second
// projection runs only when ||w'|| < ||w||/sqrt(2) (device flag; the two
// extra launches exit at once otherwise), which keeps the basis orthogonal
// to working precision like the reference's MGS (krylov.py:75-77).

__device__ __forceinline__ double block_sum_all(double v, double *sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
    return t;
}

__global__ void __launch_bounds__(DOT_BLOCK) k_mdot(const double *__restrict__ V, int64_t n, int nk,
                                                     const double *__restrict__ w, double *partial, int nsplit,
                                                     int64_t chunk, const int *active) {
    if (active && !*active) return;
    __shared__ double sh[DOT_BLOCK / 32];
    const int k = blockIdx.y;
    const double *x = k < nk ? V + (int64_t)k * n : w;
    const int64_t lo = blockIdx.x * chunk;
    const int64_t hi = lo + chunk < n ? lo + chunk : n;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t i = lo + threadIdx.x;
    for (; i + 3 * DOT_BLOCK < hi; i += 4 * DOT_BLOCK) {
        a0 = fma(x[i], w[i], a0);
        a1 = fma(x[i + DOT_BLOCK], w[i + DOT_BLOCK], a1);
        a2 = fma(x[i + 2 * DOT_BLOCK], w[i + 2 * DOT_BLOCK], a2);
        a3 = fma(x[i + 3 * DOT_BLOCK], w[i + 3 * DOT_BLOCK], a3);
    }
    for (; i < hi; i += DOT_BLOCK) a0 = fma(x[i], w[i], a0);
    double t = block_sum_all((a0 + a1) + (a2 + a3), sh);
    if (threadIdx.x == 0) partial[(int64_t)k * nsplit + blockIdx.x] = t;
}

// out[k] = sum_s partial[k*nsplit + s], one warp per k, fixed order
__global__ void k_preduce(const double *partial, int nsplit, int nk1, double *out, const int *active) {
    if (active && !*active) return;
    int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (k >= nk1) return;
    double s = 0.0;
    for (int b = lane; b < nsplit; b += 32) s += partial[(int64_t)k * nsplit + b];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    if (lane == 0) out[k] = s;
}

__global__ void __launch_bounds__(DOT_BLOCK) k_upd(const double *__restrict__ V, int64_t n, int nk,
                                                    const double *__restrict__ h, double *w, double *partial,
                                                    const int *active) {
    if (active && !*active) return;
    __shared__ double sh[DOT_BLOCK / 32];
    __shared__ double hs[1024];
    for (int k = threadIdx.x; k < nk; k += DOT_BLOCK) hs[k] = h[k];
    __syncthreads();
    double nrm = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)DOT_BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * DOT_BLOCK) {
        double a0 = w[i], a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int k = 0;
        for (; k + 3 < nk; k += 4) {
            a0 = fma(-hs[k], V[(int64_t)k * n + i], a0);
            a1 = fma(-hs[k + 1], V[(int64_t)(k + 1) * n + i], a1);
            a2 = fma(-hs[k + 2], V[(int64_t)(k + 2) * n + i], a2);
            a3 = fma(-hs[k + 3], V[(int64_t)(k + 3) * n + i], a3);
        }
        for (; k < nk; ++k) a0 = fma(-hs[k], V[(int64_t)k * n + i], a0);
        const double wi = (a0 + a1) + (a2 + a3);
        w[i] = wi;
        nrm = fma(wi, wi, nrm);
    }
    double t = block_sum_all(nrm, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

// DGKS test: re-orthogonalise when ||w'||^2 < ||w||^2 / 2
__global__ void k_reorth_flag(const double *h1, int nk, const double *nrm1, int *flag, double *h2) {
    const int f = nrm1[0] < 0.5 * h1[nk];
    if (threadIdx.x == 0) *flag = f;
    for (int k = threadIdx.x; k <= nk; k += blockDim.x) h2[k] = 0.0;
}

struct GmresState {
    double *H;     // (m+1) x m, row-major (i, j) at i*m + j
    double *cs, *sn, *g;
    double *h1, *h2;  // dot results (m+1)
    double *hnext;    // ||w|| after orthogonalisation
    double *nrm1, *nrm2;  // ||w'||^2 after the first / second projection
    int *reorth;          // DGKS flag of the current step
    double *y;        // triangular solve result
    int *status;      // [0] breakdown, [1] dead column, [2] converged-by-estimate
    double *hist;     // |g[j+1]| per iteration
};

// Arnoldi column j: h = h1 + h2, Hessenberg update, Givens (krylov.py:75-104)
__global__ void k_arnoldi_tail(GmresState st, int m, int j, double tol) {
    double *H = st.H;
    const double hn = sqrt(*st.reorth ? *st.nrm2 : *st.nrm1);
    double cs2 = 0.0;
    for (int i = 0; i <= j; ++i) {
        double hv = st.h1[i] + st.h2[i];
        H[i * m + j] = hv;
        cs2 += hv * hv;
    }
    H[(j + 1) * m + j] = hn;
    cs2 += hn * hn;
    const double colscale = sqrt(cs2);
    int brk = !(hn > 1e-12 * fmax(colscale, 1e-300));
    *st.hnext = hn;
    for (int i = 0; i < j; ++i) {
        double t = H[i * m + j];
        H[i * m + j] = st.cs[i] * t + st.sn[i] * H[(i + 1) * m + j];
        H[(i + 1) * m + j] = -st.sn[i] * t + st.cs[i] * H[(i + 1) * m + j];
    }
    const double a = H[j * m + j], b = H[(j + 1) * m + j];
    const double rho = hypot(a, b);
    if (rho == 0.0) {
        st.status[0] = 1;
        st.status[1] = 1;
        return;
    }
    st.cs[j] = a / rho;
    st.sn[j] = b / rho;
    H[j * m + j] = rho;
    H[(j + 1) * m + j] = 0.0;
    st.g[j + 1] = -st.sn[j] * st.g[j];
    st.g[j] = st.cs[j] * st.g[j];
    const double est = fabs(st.g[j + 1]);
    st.hist[j] = est;
    st.status[0] = brk;
    st.status[1] = 0;
    st.status[2] = est <= tol;
}

__global__ void k_cycle_init(GmresState st, int m, const double *beta) {
    for (int i = threadIdx.x; i < (m + 1) * m; i += blockDim.x) st.H[i] = 0.0;
    for (int i = threadIdx.x; i <= m; i += blockDim.x) st.g[i] = (i == 0) ? *beta : 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) st.cs[i] = st.sn[i] = 0.0;
    if (threadIdx.x == 0) st.status[0] = st.status[1] = st.status[2] = 0;
}

// back substitution H[:j,:j] y = g[:j]
__global__ void k_trsv(GmresState st, int m, int j) {
    for (int i = j - 1; i >= 0; --i) {
        double s = st.g[i];
        for (int k = i + 1; k < j; ++k) s -= st.H[i * m + k] * st.y[k];
        st.y[i] = s / st.H[i * m + i];
    }
}

struct Reducer {
    TBuf<double> partial;
    int nblk = 0, ld = 0;
    void init(int64_t n, int maxk, cudaStream_t s) {
        nblk = dot_grid(n);
        ld = maxk > 1 ? maxk : 1;
        partial.alloc((int64_t)nblk * ld, s);
    }
};

void norm2(const double *x, int64_t n, Reducer &R, double *out, cudaStream_t s) {
    // ||x||^2 via the update kernel with no basis vectors
    k_update<<<R.nblk, DOT_BLOCK, 0, s>>>(nullptr, n, 0, nullptr, const_cast<double *>(x), 2, R.partial.p, R.ld);
    PMGR_LAUNCHED();
    k_reduce_partials<<<1, 32, 0, s>>>(R.partial.p, R.nblk, 1, R.ld, out, 0);
    PMGR_LAUNCHED();
    k_sqrt<<<1, 1, 0, s>>>(out);
    PMGR_LAUNCHED();
}

}  // namespace

void gmres_device(const pmgr_csr *A, pmgr_mgr *M, const double *b, double *x, int nonzero_x0,
                  const pmgr_gmres_cfg &cfg, pmgr_gmres_stats &stats, double *history, int32_t history_cap,
                  cudaStream_t s) {
    if (cfg.restart < 1) fail(PMGR_ERR_INVALID, "restart must be >= 1");
    if (!(cfg.rtol > 0) || !(cfg.atol > 0)) fail(PMGR_ERR_INVALID, "tolerances must be positive");
    const CsrView Av = A->m->view();
    if (Av.nrows != Av.ncols) fail(PMGR_ERR_INVALID, "gmres requires a square operator");
    if (M && M->n != Av.nrows) fail(PMGR_ERR_INVALID, "preconditioner size does not match the operator");
    const int64_t n = Av.nrows;
    const int m = cfg.restart;
    // vin: fixed input buffer of the preconditioner (its CUDA graph is keyed
    // by buffer addresses); the normalisation writes V_{j+1} and vin at once
    TBuf<double> V((int64_t)(m + 1) * n, s), w(n, s), z(n, s), r(n, s), vin(n, s);
    TBuf<double> small((int64_t)(m + 1) * m + 6 * (m + 1) + 8, s);
    TBuf<int> status(4, s);
    TBuf<double> dhist(m + 1, s);
    GmresState st;
    st.H = small.p;
    st.cs = st.H + (m + 1) * m;
    st.sn = st.cs + (m + 1);
    st.g = st.sn + (m + 1);
    st.h1 = st.g + (m + 1);
    st.h2 = st.h1 + (m + 1);
    st.y = st.h2 + (m + 1);
    st.hnext = st.y + (m + 1);
    double *beta_d = st.hnext + 1;
    st.nrm1 = beta_d + 1;
    st.nrm2 = st.nrm1 + 1;
    st.status = status.p;
    st.reorth = status.p + 3;
    st.hist = dhist.p;
    Reducer R;
    R.init(n, m + 1, s);
    // projection partials: (nk+1) vectors x nsplit row slices
    const int64_t min_chunk = 4096;
    int nsplit_max = (int)((n + min_chunk - 1) / min_chunk);
    if (nsplit_max < 1) nsplit_max = 1;
    TBuf<double> mpart((int64_t)(m + 2) * (nsplit_max > 64 ? 64 : nsplit_max), s);
    const int upd_blocks = 4 * num_sms();
    TBuf<double> upart(upd_blocks, s);
    auto project = [&](int nk, double *h, double *nrm, const int *active) {
        int nsplit = (int)((4 * num_sms() + nk) / (nk + 1));
        if (nsplit > nsplit_max) nsplit = nsplit_max;
        if (nsplit > 64) nsplit = 64;
        if (nsplit < 1) nsplit = 1;
        const int64_t chunk = (n + nsplit - 1) / nsplit;
        k_mdot<<<dim3(nsplit, nk + 1), DOT_BLOCK, 0, s>>>(V.p, n, nk, w.p, mpart.p, nsplit, chunk, active);
        PMGR_LAUNCHED();
        k_preduce<<<((nk + 1) * 32 + 255) / 256, 256, 0, s>>>(mpart.p, nsplit, nk + 1, h, active);
        PMGR_LAUNCHED();
        k_upd<<<upd_blocks, DOT_BLOCK, 0, s>>>(V.p, n, nk, h, w.p, upart.p, active);
        PMGR_LAUNCHED();
        k_preduce<<<1, 32, 0, s>>>(upart.p, upd_blocks, 1, nrm, active);
        PMGR_LAUNCHED();
    };

    std::vector<double> hist;
    int hcount = 0;
    auto push_hist = [&](double v) {
        hist.push_back(v);
        ++hcount;
    };
    auto apply_M = [&](const double *in, double *out) {
        if (M) mgr_apply(*M, in, out, s);
        else vec_copy(in, out, n, s);
    };

    if (nonzero_x0) {
        spmv_residual(Av, x, b, r.p, s);
    } else {
        vec_copy(b, r.p, n, s);
    }
    norm2(r.p, n, R, beta_d, s);
    double beta = read_scalar(beta_d, s);
    push_hist(beta);
    const double tol = std::fmax(cfg.rtol * beta, cfg.atol);
    int total = 0;
    int restarts = 0;
    bool converged = beta <= tol;
    if (!converged) {
        while (total < cfg.max_iters) {
            k_cycle_init<<<1, 256, 0, s>>>(st, m, beta_d);
            PMGR_LAUNCHED();
            k_scale<<<dot_grid(n), DOT_BLOCK, 0, s>>>(r.p, n, beta_d, V.p, vin.p);
            PMGR_LAUNCHED();
            int j = 0;
            bool brk = false;
            while (j < m && total < cfg.max_iters) {
                double *Vj = V.p + (int64_t)j * n;
                {
                    ProfScope ps(PROF_MGR_APPLY, 0.0, s);
                    apply_M(M ? vin.p : Vj, z.p);
                }
                {
                    ProfScope ps(PROF_OUTER_SPMV, csr_pass_bytes(Av.nrows, Av.ncols, Av.nnz), s);
                    spmv(Av, z.p, w.p, s);
                }
                const int nk = j + 1;
                {
                    ProfScope pso(PROF_ORTHO, 8.0 * n * (2.0 * nk + 6.0), s);
                    project(nk, st.h1, st.nrm1, nullptr);
                    k_reorth_flag<<<1, 128, 0, s>>>(st.h1, nk, st.nrm1, st.reorth, st.h2);
                    PMGR_LAUNCHED();
                    project(nk, st.h2, st.nrm2, st.reorth);
                    k_arnoldi_tail<<<1, 1, 0, s>>>(st, m, j, tol);
                    PMGR_LAUNCHED();
                }
                int flags[3];
                PMGR_CUDA(cudaMemcpyAsync(flags, status.p, sizeof(flags), cudaMemcpyDeviceToHost, s));
                PMGR_CUDA(cudaStreamSynchronize(s));
                if (M && prof_on()) mgr_collect(*M);
                if (flags[1]) {  // dead column: discard (krylov.py:88-91)
                    brk = true;
                    break;
                }
                if (!flags[0]) {
                    k_scale<<<dot_grid(n), DOT_BLOCK, 0, s>>>(w.p, n, st.hnext, V.p + (int64_t)(j + 1) * n, vin.p);
                    PMGR_LAUNCHED();
                } else {
                    brk = true;
                }
                ++total;
                ++j;
                double est;
                PMGR_CUDA(cudaMemcpyAsync(&est, dhist.p + (j - 1), sizeof(double), cudaMemcpyDeviceToHost, s));
                PMGR_CUDA(cudaStreamSynchronize(s));
                push_hist(est);
                if (flags[2] || brk) break;
            }
            if (j > 0) {
                k_trsv<<<1, 1, 0, s>>>(st, m, j);
                PMGR_LAUNCHED();
                k_combine<<<dot_grid(n), DOT_BLOCK, 0, s>>>(V.p, n, j, st.y, w.p);
                PMGR_LAUNCHED();
                apply_M(w.p, z.p);
                vec_axpy(1.0, z.p, x, n, s);
                spmv_residual(Av, x, b, r.p, s);
                norm2(r.p, n, R, beta_d, s);
                beta = read_scalar(beta_d, s);
                if (M && prof_on()) mgr_collect(*M);
                hist.back() = beta;
            }
            ++restarts;
            if (beta <= tol) {
                converged = true;
                break;
            }
            if (brk) break;
        }
    }
    stats.iterations = total;
    stats.converged = beta <= tol;
    stats.restarts = restarts;
    int32_t nh = (int32_t)hist.size();
    stats.history_len = nh < history_cap ? nh : history_cap;
    if (history)
        for (int32_t i = 0; i < stats.history_len; ++i) history[i] = hist[i];
    (void)converged;
    (void)hcount;
}

void multidot(const double *V, int64_t n, int32_t nvec, const double *w, double *h, cudaStream_t s) {
    Reducer R;
    R.init(n, nvec, s);
    k_multidot<<<R.nblk, DOT_BLOCK, 0, s>>>(V, n, nvec, w, R.partial.p, R.ld);
    PMGR_LAUNCHED();
    k_reduce_partials<<<(nvec * 32 + 255) / 256, 256, 0, s>>>(R.partial.p, R.nblk, nvec, R.ld, h, 0);
    PMGR_LAUNCHED();
}

void multiaxpy(const double *V, int64_t n, int32_t nvec, const double *h, double *w, cudaStream_t s) {
    Reducer R;
    R.init(n, 1, s);
    k_update<<<R.nblk, DOT_BLOCK, 0, s>>>(V, n, nvec, h, w, 0, R.partial.p, R.ld);
    PMGR_LAUNCHED();
}

}  // namespace pmgr
