// amg.cu -- classical AMG setup and V(1,1) cycle on the device.
//
// Setup follows reference amg.py:184-211 level by level, bit-exact:
//   strength   (amg.py:72-101)   warp per row; rowmax via warp max (order
//                                free), threshold fl(theta*rowmax)
//   coarsening (amg.py:104-119, greedy_mis_kernel _kernels.py:240-256)
//              the sequential greedy MIS in (-measure, index) order equals
//              the lexicographically-first MIS, computed here in parallel
//              rounds: a vertex turns F once an earlier neighbour is C and
//              C once every earlier neighbour is F (SURVEY §0 finding 3)
//   direct interpolation (amg.py:122-168) with the two per-row sums in
//              stored order (warp_seq_sum) and w = ((-alpha)*a)/d
//   Galerkin   (P^T A) P with scipy's zero dropping (amg.py:200-202)
//   l1 diagonal (smoothers.py:90-106) a_ii + seq sum |a_ij| off-partition
//   coarsest   dense Gauss-Jordan inverse (replaces LAPACK getrf/getrs;
//              values only, 1e-10)
// The cycle uses the fused kernels of spmv.cu; with one row per partition
// the hybrid l1-GS sweep is exactly l1-Jacobi.
#include <cmath>
#include <cstdlib>

#include "dsetup.cuh"
#include "hier.cuh"

namespace pmgr {

namespace {

constexpr int64_t DENSE_SOLVE_CAP = 20000;  // reference amg.py:32

__global__ void k_funcs_init(int32_t *f, int64_t n, int nf) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) f[i] = (int32_t)(i % nf);
}

// strength mask per stored entry and strong count per row (warp per row)
__global__ void k_strength(int64_t n, const int64_t *__restrict__ ro, const int32_t *__restrict__ ci,
                           const double *__restrict__ v, const int32_t *__restrict__ funcs, double theta,
                           uint8_t *mask, int64_t *cnt) {
    int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int32_t fi = funcs[i];
    const int64_t b = ro[i], e = ro[i + 1];
    double m = 0.0;
    for (int64_t q = b + lane; q < e; q += 32) {
        int32_t j = ci[q];
        if (j != i && funcs[j] == fi) m = fmax(m, -v[q]);
    }
    const double rowmax = warp_max(m);
    const double thr = __dmul_rn(theta, rowmax);
    int64_t c = 0;
    for (int64_t q = b + lane; q < e; q += 32) {
        int32_t j = ci[q];
        double a = v[q];
        bool cand = (j != i) && (funcs[j] == fi);
        bool st = cand && a < 0.0 && rowmax > 0.0 && -a >= thr;
        mask[q] = st;
        c += st;
    }
    c = warp_sum_i64(c);
    if (lane == 0) cnt[i] = c;
}

// S pattern (column indices of strong entries, stored order)
__global__ void k_mask_compact(int64_t n, const int64_t *ro, const int32_t *ci, const uint8_t *mask,
                               const int64_t *sro, int32_t *sci) {
    int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    int64_t w = sro[i];
    for (int64_t q0 = ro[i]; q0 < ro[i + 1]; q0 += 32) {
        int64_t q = q0 + lane;
        bool keep = q < ro[i + 1] && mask[q];
        unsigned m = __ballot_sync(FULL, keep);
        if (keep) sci[w + __popc(m & ((1u << lane) - 1u))] = ci[q];
        w += __popc(m);
    }
}

__global__ void k_measure(const int32_t *sci, int64_t nnz, int32_t *meas) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < nnz) atomicAdd(meas + sci[q], 1);
}

__global__ void k_transpose_pattern(int64_t n, const int64_t *sro, const int32_t *sci, int64_t *cursor,
                                    int32_t *tci) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int64_t q = sro[i]; q < sro[i + 1]; ++q) {
        int64_t p = atomicAdd((unsigned long long *)(cursor + sci[q]), 1ull);
        tci[p] = (int32_t)i;
    }
}

__device__ __forceinline__ bool earlier(int32_t mu, int64_t u, int32_t mv, int64_t v) {
    return mu > mv || (mu == mv && u < v);
}

// one round of lexicographically-first MIS; status 0 undecided, 1 C, 2 F
__global__ void k_mis_round(int64_t lo, int64_t n, const int64_t *__restrict__ sro, const int32_t *__restrict__ sci,
                            const int64_t *__restrict__ tro, const int32_t *__restrict__ tci,
                            const int32_t *__restrict__ meas, int8_t *status, int *undecided) {
    int64_t v = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    volatile int8_t *st = status;
    if (st[v] != 0) return;
    const int32_t mv = meas[v];
    bool pending = false;
    for (int pass = 0; pass < 2; ++pass) {
        const int64_t *ro = pass ? tro : sro;
        const int32_t *ci = pass ? tci : sci;
        for (int64_t q = ro[v]; q < ro[v + 1]; ++q) {
            int64_t u = ci[q];
            if (!earlier(meas[u], u, mv, v)) continue;
            int8_t su = st[u];
            if (su == 1) {
                st[v] = 2;
                return;
            }
            if (su == 0) pending = true;
        }
    }
    if (!pending) {
        st[v] = 1;
    } else {
        atomicAdd(undecided, 1);
    }
}

__global__ void k_status_to_isc(int64_t n, const int8_t *status, int8_t *is_c, int64_t *isc64) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int8_t c = status[i] == 1;
    is_c[i] = c;
    isc64[i] = c;
}

// c_index from the exclusive scan of is_c
__global__ void k_cindex(int64_t n, const int8_t *is_c, const int64_t *scan, int64_t *cidx) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) cidx[i] = is_c[i] ? scan[i] : -1;
}

// direct interpolation pass 1: per-row alpha and entry count (warp per row)
__global__ void k_interp_count(int64_t lo, int64_t n, const int64_t *__restrict__ ro, const int32_t *__restrict__ ci,
                               const double *__restrict__ v, const uint8_t *__restrict__ strong,
                               const int8_t *__restrict__ is_c, const int32_t *__restrict__ funcs,
                               double *alpha, double *diag, int64_t *cnt, int *zero_diag, int *flagged) {
    int64_t i = lo + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    const int64_t b = ro[i], e = ro[i + 1];
    const int32_t fi = funcs[i];
    double sn = 0.0, sc = 0.0, dv = 0.0;
    bool found = false;
    int64_t nsc = 0;
    for (int64_t q0 = b; q0 < e; q0 += 32) {
        int64_t q = q0 + lane;
        int cntc = (int)((e - q0) < 32 ? (e - q0) : 32);
        double xn = 0.0, xc = 0.0;
        bool in_n = false, in_c = false;
        if (q < e) {
            int32_t j = ci[q];
            double a = v[q];
            if (j == i) {
                dv = a;
                found = true;
            }
            in_n = (j != i) && (funcs[j] == fi);
            in_c = strong[q] && is_c[j];
            xn = a;
            xc = a;
        }
        // sequential sums restricted to the selected entries, in stored order
        unsigned mn = __ballot_sync(FULL, in_n);
        unsigned mc = __ballot_sync(FULL, in_c);
        nsc += __popc(mc);
        for (int k = 0; k < cntc; ++k) {
            double yn = __shfl_sync(FULL, xn, k);
            double yc = __shfl_sync(FULL, xc, k);
            if (mn >> k & 1u) sn = __dadd_rn(sn, yn);
            if (mc >> k & 1u) sc = __dadd_rn(sc, yc);
        }
    }
    unsigned mf = __ballot_sync(FULL, found);
    double d = mf ? __shfl_sync(FULL, dv, __ffs(mf) - 1) : 0.0;
    if (lane != 0) return;
    diag[i] = d;
    if (d == 0.0) atomicAdd(zero_diag, 1);
    if (is_c[i]) {
        cnt[i] = 1;
        alpha[i] = 0.0;
    } else if (sc != 0.0) {
        cnt[i] = nsc;
        alpha[i] = __ddiv_rn(sn, sc);
    } else {
        cnt[i] = 0;
        alpha[i] = 0.0;
        atomicAdd(flagged, 1);
    }
}

// direct interpolation pass 2: fill P (warp per row)
__global__ void k_interp_fill(int64_t lo, int64_t n, const int64_t *__restrict__ ro, const int32_t *__restrict__ ci,
                              const double *__restrict__ v, const uint8_t *__restrict__ strong,
                              const int8_t *__restrict__ is_c, const int64_t *__restrict__ cidx,
                              const double *__restrict__ alpha, const double *__restrict__ diag,
                              const int64_t *__restrict__ pro, int32_t *pci, double *pv) {
    int64_t i = lo + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    int64_t w = pro[i];
    if (is_c[i]) {
        if (lane == 0) {
            pci[w] = (int32_t)cidx[i];
            pv[w] = 1.0;
        }
        return;
    }
    if (pro[i + 1] == w) return;
    const double na = -alpha[i];
    const double d = diag[i];
    for (int64_t q0 = ro[i]; q0 < ro[i + 1]; q0 += 32) {
        int64_t q = q0 + lane;
        bool keep = false;
        int32_t j = 0;
        if (q < ro[i + 1]) {
            j = ci[q];
            keep = strong[q] && is_c[j];
        }
        unsigned m = __ballot_sync(FULL, keep);
        if (keep) {
            int pos = __popc(m & ((1u << lane) - 1u));
            pci[w + pos] = (int32_t)cidx[j];
            pv[w + pos] = __ddiv_rn(__dmul_rn(na, v[q]), d);
        }
        w += __popc(m);
    }
}

// l1 diagonal: a_ii + seq sum over off-partition |a_ij| (warp per row)
__global__ void k_l1diag(int64_t lo0, int64_t n, const int64_t *__restrict__ ro, const int32_t *__restrict__ ci,
                         const double *__restrict__ v, int64_t nparts, const int64_t *__restrict__ starts,
                         int jacobi, double *dt, unsigned long long *bad) {
    int64_t i = lo0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    int64_t lo = i, hi = i + 1;
    if (!jacobi) {
        int64_t a = 0, b = nparts;  // find p with starts[p] <= i < starts[p+1]
        while (b - a > 1) {
            int64_t m = (a + b) / 2;
            if (starts[m] <= i) a = m;
            else b = m;
        }
        lo = starts[a];
        hi = starts[a + 1];
    }
    const int64_t b0 = ro[i], e = ro[i + 1];
    double s = 0.0, dv = 0.0;
    bool found = false;
    for (int64_t q0 = b0; q0 < e; q0 += 32) {
        int64_t q = q0 + lane;
        int cntc = (int)((e - q0) < 32 ? (e - q0) : 32);
        bool off = false;
        double x = 0.0;
        if (q < e) {
            int32_t j = ci[q];
            if (j == i) {
                dv = v[q];
                found = true;
            }
            off = (j < lo || j >= hi);
            x = fabs(v[q]);
        }
        unsigned m = __ballot_sync(FULL, off);
        for (int k = 0; k < cntc; ++k) {
            double y = __shfl_sync(FULL, x, k);
            if (m >> k & 1u) s = __dadd_rn(s, y);
        }
    }
    unsigned mf = __ballot_sync(FULL, found);
    double d = mf ? __shfl_sync(FULL, dv, __ffs(mf) - 1) : 0.0;
    if (lane == 0) {
        double r = __dadd_rn(d, s);
        dt[i] = r;
        if (r == 0.0) atomicMin(bad, (unsigned long long)i);
    }
}

__global__ void k_meas_from_ro(int64_t lo, int64_t hi, const int64_t *ro, int32_t *meas) {
    const int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < hi) meas[i] = (int32_t)(ro[i + 1] - ro[i]);
}

__global__ void k_gather_i32(const int32_t *src, const int64_t *cidx, int64_t n, int32_t *dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && cidx[i] >= 0) dst[cidx[i]] = src[i];
}

__global__ void k_to_dense(int64_t n, const int64_t *ro, const int32_t *ci, const double *v, double *M) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q) M[i * n + ci[q]] = v[q];
}

__global__ void k_identity(int64_t n, double *M) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n * n) M[t] = (t / n == t % n) ? 1.0 : 0.0;
}

// Gauss-Jordan with partial pivoting, one CTA: A (n x n) is destroyed,
// X (n x n, identity on entry) becomes A^{-1}.
__global__ void __launch_bounds__(1024) k_gauss_jordan(int64_t n, double *A, double *X, double *colk,
                                                        int *singular) {
    __shared__ double sval[32];
    __shared__ int64_t sidx[32];
    __shared__ int64_t piv;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int64_t k = 0; k < n; ++k) {
        // pivot: first row of maximal |A[i][k]| over i >= k
        double best = -1.0;
        int64_t bi = n;
        for (int64_t i = k + tid; i < n; i += nt) {
            double a = fabs(A[i * n + k]);
            if (a > best || (a == best && i < bi)) {
                best = a;
                bi = i;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            double ob = __shfl_xor_sync(FULL, best, o);
            int64_t oi = __shfl_xor_sync(FULL, bi, o);
            if (ob > best || (ob == best && oi < bi)) {
                best = ob;
                bi = oi;
            }
        }
        if ((tid & 31) == 0) {
            sval[tid >> 5] = best;
            sidx[tid >> 5] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            double b = -1.0;
            int64_t p = n;
            for (int w = 0; w < (nt + 31) / 32; ++w)
                if (sval[w] > b || (sval[w] == b && sidx[w] < p)) {
                    b = sval[w];
                    p = sidx[w];
                }
            piv = p;
            if (b == 0.0) *singular = 1;
        }
        __syncthreads();
        const int64_t p = piv;
        if (p != k) {
            for (int64_t j = tid; j < n; j += nt) {
                double t = A[k * n + j];
                A[k * n + j] = A[p * n + j];
                A[p * n + j] = t;
                t = X[k * n + j];
                X[k * n + j] = X[p * n + j];
                X[p * n + j] = t;
            }
        }
        __syncthreads();
        const double inv = 1.0 / A[k * n + k];
        __syncthreads();
        for (int64_t j = tid; j < n; j += nt) {
            A[k * n + j] *= inv;
            X[k * n + j] *= inv;
        }
        for (int64_t i = tid; i < n; i += nt) colk[i] = A[i * n + k];
        __syncthreads();
        for (int64_t t = tid; t < n * n; t += nt) {
            int64_t i = t / n, j = t % n;
            if (i == k) continue;
            double f = colk[i];
            if (f != 0.0) {
                A[i * n + j] -= f * A[k * n + j];
                X[i * n + j] -= f * X[k * n + j];
            }
        }
        __syncthreads();
    }
}

// Gauss-Jordan for larger coarsest grids: five small launches per pivot
__global__ void k_gj_pivot(int64_t n, int64_t k, const double *A, int64_t *piv, int *singular) {
    __shared__ double sval[32];
    __shared__ int64_t sidx[32];
    double best = -1.0;
    int64_t bi = n;
    for (int64_t i = k + threadIdx.x; i < n; i += blockDim.x) {
        double a = fabs(A[i * n + k]);
        if (a > best) {
            best = a;
            bi = i;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        double ob = __shfl_xor_sync(FULL, best, o);
        int64_t oi = __shfl_xor_sync(FULL, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        sval[threadIdx.x >> 5] = best;
        sidx[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = -1.0;
        int64_t p = n;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            if (sval[w] > b || (sval[w] == b && sidx[w] < p)) {
                b = sval[w];
                p = sidx[w];
            }
        *piv = p;
        if (b == 0.0) *singular = 1;
    }
}

__global__ void k_gj_swap(int64_t n, int64_t k, const int64_t *piv, double *A, double *X) {
    const int64_t p = *piv;
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p == k || j >= n) return;
    double t = A[k * n + j];
    A[k * n + j] = A[p * n + j];
    A[p * n + j] = t;
    t = X[k * n + j];
    X[k * n + j] = X[p * n + j];
    X[p * n + j] = t;
}

__global__ void k_gj_col(int64_t n, int64_t k, const double *A, double *colk) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) colk[i] = A[i * n + k];
}

__global__ void k_gj_scale(int64_t n, int64_t k, const double *colk, double *A, double *X) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double inv = 1.0 / colk[k];
    A[k * n + j] *= inv;
    X[k * n + j] *= inv;
}

__global__ void k_gj_elim(int64_t n, int64_t k, const double *colk, double *A, double *X) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t i = blockIdx.y;
    if (j >= n || i == k) return;
    const double f = colk[i];
    if (f == 0.0) return;
    A[i * n + j] -= f * A[k * n + j];
    X[i * n + j] -= f * X[k * n + j];
}

std::vector<int64_t> partition_starts(int64_t n, int64_t nparts) {
    // reference PartitionSet.contiguous (smoothers.py:67-75), align = 1
    int64_t np_ = nparts < n ? nparts : n;
    if (np_ < 1) np_ = 1;
    std::vector<int64_t> b(np_ + 1);
    const double step = (double)n / (double)np_;
    for (int64_t k = 0; k <= np_; ++k) b[k] = (int64_t)std::nearbyint((double)k * step);
    b[0] = 0;
    b[np_] = n;
    std::vector<int64_t> u;
    for (int64_t x : b)
        if (u.empty() || x != u.back()) u.push_back(x);
    return u;
}

}  // namespace

std::unique_ptr<pmgr_amg> amg_build(std::shared_ptr<const Csr> A0, const pmgr_amg_cfg &cfg, cudaStream_t s,
                                    const DistSetup *dist) {
    if (A0->nrows != A0->ncols) fail(PMGR_ERR_INVALID, "amg_setup requires a square matrix");
    if (!(cfg.strength_threshold >= 0.0 && cfg.strength_threshold < 1.0))
        fail(PMGR_ERR_INVALID, "strength_threshold must be in [0, 1)");
    if (cfg.coarse_size_cutoff < 1) fail(PMGR_ERR_INVALID, "coarse_size_cutoff must be >= 1");
    auto h = std::make_unique<pmgr_amg>();
    h->cfg = cfg;
    const int nfun = cfg.num_functions > 0 ? cfg.num_functions : 1;
    std::shared_ptr<const Csr> cur = A0;
    // distributed setup (dsetup.cuh): operators hold the owned rows of their
    // global row space; small levels are gathered and built on every rank
    std::unique_ptr<DistSetup> dd;
    if (dist && dist->nranks > 1) dd.reset(new DistSetup(*dist));
    auto replicate = [&](bool force) {
        if (dd && (force || cur->nrows <= dd->replicate_below)) {
            // a pure block operator (the node-blocked displacement block) keeps
            // its 3x3 block copy when gathered: the block kernels sum in another
            // order than the CSR ones, and the gathered level must apply exactly
            // like the single-GPU hierarchy's
            const bool blocks = cur->nbrows > 0 && cur->nbrows * 3 == cur->nrows && cur->nrem == 0;
            auto full = std::make_shared<Csr>();
            ds_gather_rows(*dd, *cur, *full, s);
            csr_finalize(*full, s, !blocks);
            if (blocks) {
                csr_make_bsr3(*full, full->nrows, full->ncols, s, true);
                if (!full->sj) csr_make_sj(*full, s);
            }
            cur = full;
            dd.reset();
        }
    };
    replicate(false);
    TBuf<int32_t> funcs(cur->nrows, s);
    if (cur->nrows) {
        k_funcs_init<<<grid_for(cur->nrows, 256), 256, 0, s>>>(funcs.p, cur->nrows, nfun);
        PMGR_LAUNCHED();
    }
    while (cur->nrows > cfg.coarse_size_cutoff && (int64_t)h->levels.size() < (int64_t)cfg.max_levels - 1) {
        const CsrView Av = cur->view();
        const int64_t n = Av.nrows;
        const int64_t rlo = dd ? dd->lo() : 0, rhi = dd ? dd->hi() : n, nown = rhi - rlo;
        // ---- strength
        TBuf<uint8_t> mask(Av.nnz, s);
        TBuf<int64_t> scnt(n, s), sro(n + 1, s);
        k_strength<<<grid_for(n * 32, 256), 256, 0, s>>>(n, Av.ro, Av.ci, Av.v, funcs.p, cfg.strength_threshold,
                                                         mask.p, scnt.p);
        PMGR_LAUNCHED();
        const int64_t snnz = exclusive_scan_total(scnt.p, sro.p, n, s);
        TBuf<int32_t> sci(snnz, s);
        k_mask_compact<<<grid_for(n * 32, 256), 256, 0, s>>>(n, Av.ro, Av.ci, mask.p, sro.p, sci.p);
        PMGR_LAUNCHED();
        setup_trace("amg strength", (int64_t)h->levels.size(), s);
        // ---- measures and S^T
        TBuf<int32_t> meas(n, s);
        PMGR_CUDA(cudaMemsetAsync(meas.p, 0, sizeof(int32_t) * n, s));
        if (snnz) {
            k_measure<<<grid_for(snnz, 256), 256, 0, s>>>(sci.p, snnz, meas.p);
            PMGR_LAUNCHED();
        }
        TBuf<int64_t> tro(n + 1, s), cursor(n + 1, s);
        exclusive_scan_total_i32(meas.p, tro.p, n, s);
        PMGR_CUDA(cudaMemcpyAsync(cursor.p, tro.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
        TBuf<int32_t> tci(snnz, s);
        k_transpose_pattern<<<grid_for(n, 256), 256, 0, s>>>(n, sro.p, sci.p, cursor.p, tci.p);
        PMGR_LAUNCHED();
        const int64_t *trop = tro.p;
        const int32_t *tcip = tci.p;
        Csr ST;
        if (dd) {
            // my rows' strong entries, by column, assembled at the columns'
            // owners: every owned point gets its full in-neighbourhood
            Csr STl;
            STl.nrows = STl.ncols = n;
            STl.nnz = snnz;
            STl.ro.alloc(n + 1);
            STl.ci.alloc(snnz);
            PMGR_CUDA(cudaMemcpyAsync(STl.ro.p, tro.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
            if (snnz) PMGR_CUDA(cudaMemcpyAsync(STl.ci.p, tci.p, sizeof(int32_t) * snnz, cudaMemcpyDeviceToDevice, s));
            ds_rows_to_owners(*dd, STl, ST, s);
            PMGR_CUDA(cudaMemsetAsync(meas.p, 0, sizeof(int32_t) * n, s));
            if (nown > 0) {
                k_meas_from_ro<<<grid_for(nown, 256), 256, 0, s>>>(rlo, rhi, ST.ro.p, meas.p);
                PMGR_LAUNCHED();
            }
            ds_gather_segment(*dd, meas.p, sizeof(int32_t), s);
            trop = ST.ro.p;
            tcip = ST.ci.p;
        }
        setup_trace("amg measure+transpose", (int64_t)h->levels.size(), s);
        // ---- lexicographically-first MIS rounds
        TBuf<int8_t> status(n, s);
        TBuf<int> undec(1, s);
        PMGR_CUDA(cudaMemsetAsync(status.p, 0, n, s));
        for (int round = 0;; ++round) {
            PMGR_CUDA(cudaMemsetAsync(undec.p, 0, sizeof(int), s));
            if (nown > 0) {
                k_mis_round<<<grid_for(nown, 256), 256, 0, s>>>(rlo, rhi, sro.p, sci.p, trop, tcip, meas.p,
                                                                 status.p, undec.p);
                PMGR_LAUNCHED();
            }
            int64_t left = read_scalar(undec.p, s);
            if (dd) {
                ds_gather_segment(*dd, status.p, 1, s);
                left = ds_allsum(*dd, left, s);
            }
            if (left == 0) break;
            if (round > 100000) fail(PMGR_ERR_CUDA, "MIS rounds did not terminate");
        }
        AmgLevel lev;
        lev.is_c.alloc(n);
        TBuf<int64_t> isc64(n, s), cscan(n + 1, s), cidx(n, s);
        k_status_to_isc<<<grid_for(n, 256), 256, 0, s>>>(n, status.p, lev.is_c.p, isc64.p);
        PMGR_LAUNCHED();
        const int64_t nc = exclusive_scan_total(isc64.p, cscan.p, n, s);
        if (nc == n) break;  // coarsening stagnated (amg.py:196-198)
        k_cindex<<<grid_for(n, 256), 256, 0, s>>>(n, lev.is_c.p, cscan.p, cidx.p);
        PMGR_LAUNCHED();
        setup_trace("amg MIS", (int64_t)h->levels.size(), s);
        // ---- direct interpolation
        TBuf<double> alpha(n, s), diag(n, s);
        TBuf<int64_t> pcnt(n, s);
        TBuf<int> flags(2, s);
        PMGR_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * 2, s));
        PMGR_CUDA(cudaMemsetAsync(pcnt.p, 0, sizeof(int64_t) * n, s));
        if (nown > 0) {
            k_interp_count<<<grid_for(nown * 32, 256), 256, 0, s>>>(rlo, rhi, Av.ro, Av.ci, Av.v, mask.p,
                                                                    lev.is_c.p, funcs.p, alpha.p, diag.p, pcnt.p,
                                                                    flags.p, flags.p + 1);
            PMGR_LAUNCHED();
        }
        int hflags[2];
        PMGR_CUDA(cudaMemcpyAsync(hflags, flags.p, sizeof(hflags), cudaMemcpyDeviceToHost, s));
        PMGR_CUDA(cudaStreamSynchronize(s));
        if (dd) {
            hflags[0] = (int)ds_allsum(*dd, hflags[0], s);
            hflags[1] = (int)ds_allsum(*dd, hflags[1], s);
        }
        if (hflags[0]) fail(PMGR_ERR_INTERP_DIAG, "direct interpolation requires nonzero diagonals");
        h->flagged += hflags[1];
        lev.P.nrows = n;
        lev.P.ncols = nc;
        lev.P.ro.alloc(n + 1);
        lev.P.nnz = exclusive_scan_total(pcnt.p, lev.P.ro.p, n, s);
        lev.P.ci.alloc(lev.P.nnz);
        lev.P.v.alloc(lev.P.nnz);
        if (nown > 0) {
            k_interp_fill<<<grid_for(nown * 32, 256), 256, 0, s>>>(rlo, rhi, Av.ro, Av.ci, Av.v, mask.p, lev.is_c.p,
                                                                   cidx.p, alpha.p, diag.p, lev.P.ro.p, lev.P.ci.p,
                                                                   lev.P.v.p);
            PMGR_LAUNCHED();
        }
        setup_trace("amg interpolation", (int64_t)h->levels.size(), s);
        // ---- Galerkin (P^T A) P, zero dropping after each product
        ds_finalize(dd.get(), lev.P, s);
        auto next = std::make_shared<Csr>();
        std::vector<int64_t> cstart;
        if (!dd) {
            csr_transpose(lev.P.view(), lev.R, s);
            csr_finalize(lev.R, s);
            setup_trace("  amg R = P^T", (int64_t)h->levels.size(), s);
            {
                Csr T1;
                spgemm(lev.R.view(), Av, 0, T1, s);
                spgemm(T1.view(), lev.P.view(), 0, *next, s);
                setup_trace("  amg R A P", (int64_t)h->levels.size(), s);
            }
            setup_trace("  amg free R A", (int64_t)h->levels.size(), s);
            csr_finalize(*next, s);
            setup_trace("  amg finalize", (int64_t)h->levels.size(), s);
        } else {
            // R = P^T: my fine rows' entries assembled at the coarse owners
            // (pieces in rank order = ascending fine index, as csr_transpose
            // orders them); rows of A and P behind the products' middle
            // indices fetched from their owners
            cstart = ds_sub_bounds(dd->start, lev.is_c.p, n, true, s);
            const DistSetup dc = dd->with(cstart);
            Csr Rp;
            csr_transpose(lev.P.view(), Rp, s);
            ds_rows_to_owners(dc, Rp, lev.R, s);
            ds_finalize(&dc, lev.R, s);
            Csr Aext, T1, Pext;
            ds_fetch_rows(*dd, *cur, ds_cols_outside(lev.R, dc.lo(), dc.hi(), rlo, rhi, s), Aext, s);
            spgemm(lev.R.view(), Aext.view(), 0, T1, s);
            ds_fetch_rows(*dd, lev.P, ds_cols_outside(T1, dc.lo(), dc.hi(), rlo, rhi, s), Pext, s);
            spgemm(T1.view(), Pext.view(), 0, *next, s);
            ds_finalize(&dc, *next, s);
        }
        setup_trace("amg Galerkin", (int64_t)h->levels.size(), s);
        static const bool dstats = getenv("PMGR_HIER_STATS") && getenv("PMGR_HIER_STATS")[0] != '0';
        if (dd && dstats)
            fprintf(stderr, "[pmgr] rank %d distributed AMG level %d: %lld rows (own %lld) -> %lld\n", dd->rank,
                    (int)h->levels.size(), (long long)n, (long long)nown, (long long)nc);
        // ---- l1 diagonal with the contiguous partitions
        lev.jacobi = cfg.npartitions >= n;
        lev.dtilde.alloc(n);
        std::vector<int64_t> st;
        if (!lev.jacobi) {
            if (dd) fail(PMGR_ERR_NOT_SUPPORTED, "distributed setup needs l1-Jacobi AMG levels (npartitions >= n)");
            st = partition_starts(n, cfg.npartitions);
            lev.nparts = (int64_t)st.size() - 1;
            lev.jacobi = lev.nparts == n;  // one row per partition anyway
            lev.starts.alloc((int64_t)st.size());
            PMGR_CUDA(cudaMemcpyAsync(lev.starts.p, st.data(), sizeof(int64_t) * st.size(), cudaMemcpyHostToDevice, s));
        } else {
            lev.nparts = n;
        }
        TBuf<unsigned long long> bad(1, s);
        PMGR_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), s));
        if (nown > 0) {
            k_l1diag<<<grid_for(nown * 32, 256), 256, 0, s>>>(rlo, rhi, Av.ro, Av.ci, Av.v, lev.nparts,
                                                              lev.jacobi ? nullptr : lev.starts.p, lev.jacobi ? 1 : 0,
                                                              lev.dtilde.p, bad.p);
            PMGR_LAUNCHED();
        }
        const unsigned long long b = read_scalar(bad.p, s);
        int64_t bi = b == ~0ull ? -1 : (int64_t)b;
        if (dd) {  // the first vanishing row over all ranks
            const int64_t g = ds_allmax(*dd, bi < 0 ? INT64_MIN : -bi, s);
            bi = g == INT64_MIN ? -1 : -g;
        }
        if (bi >= 0) fail(PMGR_ERR_L1_VANISHES, "l1 diagonal vanishes at row " + std::to_string(bi), bi);
        setup_trace("amg l1 diagonal", (int64_t)h->levels.size(), s);
        // ---- next level functions
        TBuf<int32_t> nfuncs(nc, s);
        k_gather_i32<<<grid_for(n, 256), 256, 0, s>>>(funcs.p, cidx.p, n, nfuncs.p);
        PMGR_LAUNCHED();
        funcs = std::move(nfuncs);
        // ---- workspace
        lev.A = cur;
        lev.b.alloc(n);
        lev.x.alloc(n);
        lev.r.alloc(n);
        lev.xo.alloc(n);
        if (!lev.jacobi) lev.xpre.alloc(n);
        h->levels.push_back(std::move(lev));
        cur = next;
        if (dd) {
            dd->start = cstart;
            replicate(false);
        }
    }
    replicate(true);
    const int64_t nc = cur->nrows;
    if (nc > DENSE_SOLVE_CAP)
        fail(PMGR_ERR_DENSE_CAP, "coarsest AMG level of size " + std::to_string(nc) + " is too large for a dense solve");
    h->coarse = cur;
    h->coarse_inv.alloc(nc * nc);
    h->cb.alloc(nc);
    h->cx.alloc(nc);
    h->ctmp.alloc(nc);
    if (nc > 0) {
        TBuf<double> M(nc * nc, s), colk(nc, s);
        TBuf<int> sing(1, s);
        PMGR_CUDA(cudaMemsetAsync(M.p, 0, sizeof(double) * nc * nc, s));
        PMGR_CUDA(cudaMemsetAsync(sing.p, 0, sizeof(int), s));
        k_to_dense<<<grid_for(nc, 128), 128, 0, s>>>(nc, cur->ro.p, cur->ci.p, cur->v.p, M.p);
        PMGR_LAUNCHED();
        k_identity<<<grid_for(nc * nc, 256), 256, 0, s>>>(nc, h->coarse_inv.p);
        PMGR_LAUNCHED();
        if (nc <= 512) {
            k_gauss_jordan<<<1, 1024, 0, s>>>(nc, M.p, h->coarse_inv.p, colk.p, sing.p);
            PMGR_LAUNCHED();
        } else {
            TBuf<int64_t> piv(1, s);
            const unsigned gx = grid_for(nc, 256);
            // five dependent launches per pivot, straight on the stream: the
            // kernels of one pivot take ~30 us, more than their launches cost,
            // so a recorded CUDA graph bought nothing (70 ms either way at
            // nc = 2,034) and its capture broke when several ranks' host
            // threads set up at once (the emulated-rank harness)
            for (int64_t k = 0; k < nc; ++k) {
                k_gj_pivot<<<1, 1024, 0, s>>>(nc, k, M.p, piv.p, sing.p);
                k_gj_swap<<<gx, 256, 0, s>>>(nc, k, piv.p, M.p, h->coarse_inv.p);
                k_gj_col<<<gx, 256, 0, s>>>(nc, k, M.p, colk.p);
                k_gj_scale<<<gx, 256, 0, s>>>(nc, k, colk.p, M.p, h->coarse_inv.p);
                k_gj_elim<<<dim3(gx, (unsigned)nc), 256, 0, s>>>(nc, k, colk.p, M.p, h->coarse_inv.p);
            }
            PMGR_CUDA(cudaPeekAtLastError());
            g_launches.fetch_add(5 * nc, std::memory_order_relaxed);
        }
        PMGR_CUDA(cudaStreamSynchronize(s));
    }
    setup_trace("amg coarsest inverse", (int64_t)h->levels.size(), s);
    collapse_tail(*h, s);
    setup_trace("amg collapse", h->collapse_from, s);
    return h;
}

namespace {

// V(1,1) from level l with right-hand side lev.b (already in place), zero
// initial guess; the result is left in lev.xo (or h.cx at the coarsest).
void cycle_from_zero(pmgr_amg &h, size_t l, cudaStream_t s, double *out = nullptr);

const double *coarse_solve(pmgr_amg &h, cudaStream_t s) {
    dense_matvec(h.coarse_inv.p, h.coarse->nrows, h.coarse->nrows, h.cb.p, h.cx.p, s);
    return h.cx.p;
}

void cycle_from_zero(pmgr_amg &h, size_t l, cudaStream_t s, double *out) {
    // precondition: L.b holds the right-hand side and, on l1-Jacobi levels,
    // L.x = L.b / dtilde (the first sweep from zero), written by the producer.
    // Row-distributed hierarchies: owned rows only, ghosts exchanged before
    // every operator that reads them (halo_exchange is a no-op otherwise).
    AmgLevel &L = h.levels[l];
    double *y = out ? out : L.xo.p;
    if ((int)l == h.collapse_from) {
        if (h.gather) {
            gather_full(h.gather.get(), L.b.p + L.off, h.full.p, s);
            dense_matvec_rows(h.collapsed.p, L.A->nrows, h.gather->n_full, h.collapsed_ld, h.full.p, y + L.off, s);
        } else {
            dense_matvec(h.collapsed.p, L.A->nrows, h.collapsed_ld, L.b.p, y, s);
        }
        return;
    }
    const CsrView A = L.A->view();
    const bool has_next = l + 1 < h.levels.size();
    const bool tag = h.prof_tag && l == 0;
    const double pass = csr_pass_bytes(A) + 16.0 * A.nrows;
    if (L.jacobi) {
        ProfScope ps(tag ? PROF_FRELAX_SWEEP0 : PROF_KINDS, pass, s);
        with_halo(*L.A, L.halo.get(), L.x.p, s, [&](const CsrView &V) { spmv_residual(V, L.x.p, L.b.p, L.r.p, s); });
    } else {
        vec_zero(L.x.p, A.nrows, s);
        hybrid_gs(A, L.nparts, L.starts.p, L.dtilde.p, L.b.p, L.x.p, L.xpre.p, true, s);
        spmv_residual(A, L.x.p, L.b.p, L.r.p, s);
    }
    const double *e;
    if (has_next) {
        AmgLevel &N = h.levels[l + 1];
        with_halo(L.R, L.halo.get(), L.r.p, s, [&](const CsrView &V) {
            if (N.jacobi) spmv_restrict_div(V, L.r.p, N.dtilde.p, N.b.p, N.x.p, s);
            else spmv(V, L.r.p, N.b.p, s);
        });
        cycle_from_zero(h, l + 1, s);
        with_halo(L.P, N.halo.get(), N.xo.p, s, [&](const CsrView &V) { spmv_add_pre(V, N.xo.p, L.x.p, s); });
    } else {
        halo_exchange(L.halo.get(), L.r.p, s);
        spmv(L.R.view(), L.r.p, h.cb.p, s);
        e = coarse_solve(h, s);
        spmv_add_pre(L.P.view(), e, L.x.p, s);
    }
    if (L.jacobi) {
        ProfScope ps(tag ? PROF_FRELAX_JACOBI : PROF_KINDS, pass, s);
        with_halo(*L.A, L.halo.get(), L.x.p, s,
                  [&](const CsrView &V) { spmv_jacobi_bpre(V, L.x.p, L.b.p, L.dtilde.p, y, s); });
    } else {
        hybrid_gs(A, L.nparts, L.starts.p, L.dtilde.p, L.b.p, L.x.p, L.xpre.p, false, s);
        vec_copy(L.x.p, y, A.nrows, s);
    }
}

}  // namespace

bool amg_cycle_rows(pmgr_amg &h, const double *v, const int64_t *rows, double *out, cudaStream_t s) {
    if (h.levels.empty() || !h.levels[0].jacobi) return false;
    AmgLevel &L = h.levels[0];
    const int64_t o = L.off;
    vec_gather_div(v, rows + o, L.dtilde.p + o, L.A->nrows, L.b.p + o, L.x.p + o, s);
    cycle_from_zero(h, 0, s, out);
    return true;
}

bool amg_entry(pmgr_amg &h, double **b, double **x, const double **dtilde) {
    if (h.levels.empty() || !h.levels[0].jacobi) return false;
    AmgLevel &L = h.levels[0];
    *b = L.b.p;
    *x = L.x.p;
    *dtilde = L.dtilde.p;
    return true;
}

void amg_cycle_prefilled(pmgr_amg &h, double *out, cudaStream_t s) { cycle_from_zero(h, 0, s, out); }

void amg_cycle(pmgr_amg &h, const double *b, const double *x, double *out, cudaStream_t s) {
    if (h.levels.empty()) {
        const int64_t n = h.coarse->nrows;
        if (x) {
            // x + inv * (b - A x)
            spmv_residual(h.coarse->view(), x, b, h.cb.p, s);
            dense_matvec(h.coarse_inv.p, n, n, h.cb.p, h.cx.p, s);
            vec_copy(x, out, n, s);
            vec_axpy(1.0, h.cx.p, out, n, s);
        } else {
            vec_copy(b, h.cb.p, n, s);
            dense_matvec(h.coarse_inv.p, n, n, h.cb.p, out, s);
        }
        return;
    }
    AmgLevel &L = h.levels[0];
    const int64_t n = L.A->nrows;
    if (x && h.collapse_from == 0) {
        // the whole hierarchy is the collapsed operator M_t (the cycle from a
        // zero guess is the linear map b -> M_t b), so the cycle from x is
        // x + M_t (b - A x): one residual pass, the dense product, an axpy
        const int64_t o = L.off;
        halo_exchange(L.halo.get(), const_cast<double *>(x), s);
        spmv_residual(L.A->view(), x, b, L.r.p, s);
        if (h.gather) {
            gather_full(h.gather.get(), L.r.p + o, h.full.p, s);
            dense_matvec_rows(h.collapsed.p, n, h.gather->n_full, h.collapsed_ld, h.full.p, L.xo.p + o, s);
        } else {
            dense_matvec(h.collapsed.p, n, h.collapsed_ld, L.r.p, L.xo.p, s);
        }
        vec_copy(x + o, out + o, n, s);
        vec_axpy(1.0, L.xo.p + o, out + o, n, s);
        return;
    }
    if (!x) {
        const int64_t o = L.off;
        if (L.jacobi) vec_copy_div(b + o, L.dtilde.p + o, n, L.b.p + o, L.x.p + o, s);
        else vec_copy(b, L.b.p, n, s);
        cycle_from_zero(h, 0, s, out);
        return;
    }
    // nonzero initial guess at the top level: pre-sweep from x.  Vectors are
    // in the level's ext layout (row-distributed hierarchies: owned range at
    // L.off plus ghosts, exchanged before every operator that reads them; x
    // must be an ext buffer of the level-0 space; offsets are 0 and the
    // exchanges no-ops on one GPU)
    const int64_t o = L.off;
    vec_copy(b + o, L.b.p + o, n, s);
    const CsrView A = L.A->view();
    if (L.jacobi) {
        with_halo(*L.A, L.halo.get(), const_cast<double *>(x), s,
                  [&](const CsrView &V) { spmv_jacobi(V, x, L.b.p, L.dtilde.p, L.x.p, s); });
    } else {
        vec_copy(x, L.x.p, n, s);
        hybrid_gs(A, L.nparts, L.starts.p, L.dtilde.p, L.b.p, L.x.p, L.xpre.p, true, s);
    }
    with_halo(*L.A, L.halo.get(), L.x.p, s, [&](const CsrView &V) { spmv_residual(V, L.x.p, L.b.p, L.r.p, s); });
    if (h.levels.size() > 1) {
        AmgLevel &N = h.levels[1];
        with_halo(L.R, L.halo.get(), L.r.p, s, [&](const CsrView &V) {
            if (N.jacobi) spmv_restrict_div(V, L.r.p, N.dtilde.p, N.b.p, N.x.p, s);
            else spmv(V, L.r.p, N.b.p, s);
        });
        cycle_from_zero(h, 1, s);
        with_halo(L.P, N.halo.get(), N.xo.p, s, [&](const CsrView &V) { spmv_add(V, N.xo.p, L.x.p, s); });
    } else {
        halo_exchange(L.halo.get(), L.r.p, s);
        spmv(L.R.view(), L.r.p, h.cb.p, s);
        const double *e = coarse_solve(h, s);
        spmv_add(L.P.view(), e, L.x.p, s);
    }
    if (L.jacobi) {
        with_halo(*L.A, L.halo.get(), L.x.p, s,
                  [&](const CsrView &V) { spmv_jacobi(V, L.x.p, L.b.p, L.dtilde.p, out, s); });
    } else {
        hybrid_gs(A, L.nparts, L.starts.p, L.dtilde.p, L.b.p, L.x.p, L.xpre.p, false, s);
        vec_copy(L.x.p, out, n, s);
    }
}

}  // namespace pmgr
