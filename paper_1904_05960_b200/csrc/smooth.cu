// smooth.cu -- level-2 global smoothers of MGR (reference mgr.py:275-292,
// smoothers.py:127-224, _kernels.py:47-237): ILU(k) over partition-local
// couplings and hybrid block Gauss-Seidel over per-cell (s, p) 2x2 blocks.
//
// Both are sequential inside a partition and independent across partitions
// (PartitionSet.contiguous, align 2), so the device runs one thread per
// partition and reproduces the reference's arithmetic order exactly: the
// ILU factors are bitwise equal to iluk_symbolic / iluk_numeric, the
// substitutions and sweeps to ilu_solve_kernel / hbgs_kernel.
#include <algorithm>
#include <cmath>

#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/extrema.h>
#include <thrust/sequence.h>
#include <thrust/sort.h>

#include "hier.cuh"

namespace pmgr {

std::vector<int64_t> partition_starts_aligned(int64_t n, int64_t nparts, int64_t align) {
    // PartitionSet.contiguous (smoothers.py:67-75): np.round(linspace / align) * align
    int64_t lim = n / (align > 0 ? align : 1);
    if (lim < 1) lim = 1;
    int64_t np_ = nparts < lim ? nparts : lim;
    if (np_ < 1) np_ = 1;
    std::vector<int64_t> b(np_ + 1);
    const double step = (double)n / (double)np_;
    for (int64_t k = 0; k <= np_; ++k) {
        const double y = k == np_ ? (double)n : (double)k * step;
        b[k] = (int64_t)std::nearbyint(y / (double)align) * align;
    }
    b[0] = 0;
    b[np_] = n;
    std::vector<int64_t> u;
    for (int64_t x : b)
        if (u.empty() || x != u.back()) u.push_back(x);
    return u;
}

namespace {

constexpr int INT_BIG = 0x3fffffff;

__device__ __forceinline__ int64_t part_of(const int64_t *starts, int64_t np_, int64_t i) {
    int64_t a = 0, b = np_;  // last p with starts[p] <= i
    while (b - a > 1) {
        const int64_t m = (a + b) >> 1;
        if (starts[m] <= i) a = m;
        else b = m;
    }
    return a;
}

// restrict_to_partitions (smoothers.py:215-224): keep columns inside the row's partition
__global__ void k_restrict_count(int64_t n, const int64_t *ro, const int32_t *ci, const int64_t *starts, int64_t np_,
                                 int64_t *cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p = part_of(starts, np_, i), lo = starts[p], hi = starts[p + 1];
    int64_t c = 0;
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q) c += (ci[q] >= lo && ci[q] < hi);
    cnt[i] = c;
}
__global__ void k_restrict_fill(int64_t n, const int64_t *ro, const int32_t *ci, const double *v, const int64_t *starts,
                                int64_t np_, const int64_t *oro, int32_t *oci, double *ov) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p = part_of(starts, np_, i), lo = starts[p], hi = starts[p + 1];
    int64_t w = oro[i];
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q)
        if (ci[q] >= lo && ci[q] < hi) {
            oci[w] = ci[q];
            ov[w] = v[q];
            ++w;
        }
}

// A + shift I with scipy's csr_plus_csr semantics (exact zeros dropped)
__global__ void k_shift_count(int64_t n, const int64_t *ro, const int32_t *ci, const double *v, double shift,
                              int64_t *cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t c = 0;
    bool diag = false;
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q) {
        double x = v[q];
        if (ci[q] == i) {
            x += shift;
            diag = true;
        }
        c += (x != 0.0);
    }
    if (!diag) c += (shift != 0.0);
    cnt[i] = c;
}
__global__ void k_shift_fill(int64_t n, const int64_t *ro, const int32_t *ci, const double *v, double shift,
                             const int64_t *oro, int32_t *oci, double *ov) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t w = oro[i];
    bool diag = false;
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q) {
        const int32_t c = ci[q];
        if (!diag && c > i) {
            if (shift != 0.0) {
                oci[w] = (int32_t)i;
                ov[w++] = shift;
            }
            diag = true;
        }
        double x = v[q];
        if (c == i) {
            x += shift;
            diag = true;
        }
        if (x != 0.0) {
            oci[w] = c;
            ov[w++] = x;
        }
    }
    if (!diag && shift != 0.0) {
        oci[w] = (int32_t)i;
        ov[w] = shift;
    }
}

__global__ void k_max_abs_diag(int64_t n, const int64_t *ro, const int32_t *ci, const double *v,
                               unsigned long long *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double d = 0.0;
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q)
        if (ci[q] == i) d = fabs(v[q]);
    atomicMax(out, (unsigned long long)__double_as_longlong(d));  // non-negative doubles order as integers
}

// iluk_symbolic (_kernels.py:96-161) for the rows of one partition, written
// into a private region [rbase, rbase + rcap) of (col, level) pairs
__global__ void k_iluk_symbolic(const int64_t *ro, const int32_t *ci, const int64_t *starts, int64_t np_, int k,
                                const int64_t *rbase, const int64_t *rcap, int32_t *rind, int32_t *rlev,
                                int64_t *rstart, int64_t *rcnt, int64_t *dposr, int32_t *lev_ws, int32_t *cols,
                                int64_t *fail_row, int *overflow) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np_) return;
    const int64_t lo = starts[p], hi = starts[p + 1];
    int32_t *lw = lev_ws + lo;  // indexed by column - lo
    int32_t *cl = cols + lo;
    for (int64_t t = 0; t < hi - lo; ++t) lw[t] = INT_BIG;
    int64_t count = 0;
    const int64_t cap = rcap[p];
    int32_t *ind = rind + rbase[p];
    int32_t *lev = rlev + rbase[p];
    fail_row[p] = -1;
    for (int64_t i = lo; i < hi; ++i) {
        int64_t nact = 0;
        for (int64_t q = ro[i]; q < ro[i + 1]; ++q) {
            const int32_t j = ci[q];
            lw[j - lo] = 0;
            cl[nact++] = j;
        }
        int64_t ptr = 0;
        while (ptr < nact) {
            const int32_t m = cl[ptr];
            if (m >= i) break;
            const int32_t lev_im = lw[m - lo];
            const int64_t mb = rstart[m];
            for (int64_t q = mb + dposr[m] + 1; q < mb + rcnt[m]; ++q) {
                const int32_t j = ind[q];
                const int32_t newlev = lev_im + lev[q] + 1;
                if (newlev <= k) {
                    if (lw[j - lo] == INT_BIG) {
                        int64_t a = ptr + 1, b = nact;
                        while (a < b) {
                            const int64_t mid = (a + b) >> 1;
                            if (cl[mid] < j) a = mid + 1;
                            else b = mid;
                        }
                        for (int64_t t = nact; t > a; --t) cl[t] = cl[t - 1];
                        cl[a] = j;
                        ++nact;
                        lw[j - lo] = newlev;
                    } else if (newlev < lw[j - lo]) {
                        lw[j - lo] = newlev;
                    }
                }
            }
            ++ptr;
        }
        if (count + nact > cap) {
            *overflow = 1;
            return;
        }
        rstart[i] = count;
        dposr[i] = -1;
        for (int64_t t = 0; t < nact; ++t) {
            const int32_t j = cl[t];
            ind[count + t] = j;
            lev[count + t] = lw[j - lo];
            if (j == i) dposr[i] = t;
            lw[j - lo] = INT_BIG;
        }
        rcnt[i] = nact;
        count += nact;
        if (dposr[i] < 0) {  // structurally missing pivot: the reference stops here
            fail_row[p] = i;
            for (int64_t r = i + 1; r < hi; ++r) {
                rstart[r] = count;
                rcnt[r] = 0;
                dposr[r] = -1;
            }
            return;
        }
    }
}

__global__ void k_ilu_compact(int64_t n, const int64_t *starts, int64_t np_, const int64_t *rbase,
                              const int64_t *rstart, const int64_t *rcnt, const int32_t *rind, const int64_t *lptr,
                              int32_t *lind) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p = part_of(starts, np_, i);
    const int32_t *src = rind + rbase[p] + rstart[i];
    for (int64_t t = 0; t < rcnt[i]; ++t) lind[lptr[i] + t] = src[t];
}

__global__ void k_dpos_abs(int64_t n, const int64_t *lptr, const int64_t *dposr, int64_t *dpos) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dpos[i] = dposr[i] >= 0 ? lptr[i] + dposr[i] : -1;
}

// iluk_numeric (_kernels.py:164-197), one thread per partition
__global__ void k_iluk_numeric(const int64_t *aptr, const int32_t *aind, const double *adata, const int64_t *starts,
                               int64_t np_, const int64_t *luptr, const int32_t *luind, const int64_t *dpos,
                               double *ludata, double *w, int64_t *posof, int64_t *fail_row) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np_) return;
    const int64_t lo = starts[p], hi = starts[p + 1];
    for (int64_t j = lo; j < hi; ++j) {
        posof[j] = -1;
        w[j] = 0.0;
    }
    fail_row[p] = -1;
    for (int64_t i = lo; i < hi; ++i) {
        if (dpos[i] < 0) {
            fail_row[p] = i;
            return;
        }
        for (int64_t q = luptr[i]; q < luptr[i + 1]; ++q) {
            posof[luind[q]] = q;
            w[luind[q]] = 0.0;
        }
        for (int64_t q = aptr[i]; q < aptr[i + 1]; ++q) w[aind[q]] = adata[q];
        for (int64_t q = luptr[i]; q < dpos[i]; ++q) {
            const int32_t m = luind[q];
            const double um = ludata[dpos[m]];
            if (um == 0.0) {
                fail_row[p] = m;
                return;
            }
            const double lam = w[m] / um;
            w[m] = lam;
            for (int64_t t = dpos[m] + 1; t < luptr[m + 1]; ++t) {
                const int32_t j = luind[t];
                if (posof[j] >= luptr[i]) w[j] = __dsub_rn(w[j], __dmul_rn(lam, ludata[t]));  // no FMA: bitwise
            }
        }
        for (int64_t q = luptr[i]; q < luptr[i + 1]; ++q) {
            ludata[q] = w[luind[q]];
            posof[luind[q]] = -1;
        }
        if (ludata[dpos[i]] == 0.0) {
            fail_row[p] = i;
            return;
        }
    }
}

// ilu_solve_kernel (_kernels.py:200-214) per partition: the factors of the
// restricted matrix couple nothing across partitions
__global__ void k_ilu_solve(const int64_t *starts, int64_t np_, const int64_t *luptr, const int32_t *luind,
                            const double *ludata, const int64_t *dpos, const double *r, double *z) {
    pdl_wait();
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np_) return;
    const int64_t lo = starts[p], hi = starts[p + 1];
    for (int64_t i = lo; i < hi; ++i) {
        double s = r[i];
        for (int64_t q = luptr[i]; q < dpos[i]; ++q) s = __dsub_rn(s, __dmul_rn(ludata[q], z[luind[q]]));
        z[i] = s;
    }
    for (int64_t i = hi - 1; i >= lo; --i) {
        double s = z[i];
        for (int64_t q = dpos[i] + 1; q < luptr[i + 1]; ++q) s = __dsub_rn(s, __dmul_rn(ludata[q], z[luind[q]]));
        z[i] = s / ludata[dpos[i]];
    }
}

// level schedule of the substitutions: a row's forward level is one past its
// L-part columns' (backward: U-part), computed per partition in row order
__global__ void k_ilu_levels(const int64_t *starts, int64_t np_, const int64_t *luptr, const int32_t *luind,
                             const int64_t *dpos, int32_t *lf, int32_t *lb) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np_) return;
    const int64_t lo = starts[p], hi = starts[p + 1];
    for (int64_t i = lo; i < hi; ++i) {
        int32_t l = 0;
        for (int64_t q = luptr[i]; q < dpos[i]; ++q) l = max(l, lf[luind[q]] + 1);
        lf[i] = l;
    }
    for (int64_t i = hi - 1; i >= lo; --i) {
        int32_t l = 0;
        for (int64_t q = dpos[i] + 1; q < luptr[i + 1]; ++q) l = max(l, lb[luind[q]] + 1);
        lb[i] = l;
    }
}

__global__ void k_count_levels(int64_t n, const int32_t *lev, int64_t *cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) atomicAdd((unsigned long long *)(cnt + lev[i]), 1ull);
}

// one level of the substitutions: every row of the level at once, each row
// summed in its stored order exactly as ilu_solve_kernel does
__global__ void k_ilu_fwd_level(const int32_t *rows, int64_t cnt, const int64_t *luptr, const int32_t *luind,
                                const double *ludata, const int64_t *dpos, const double *r, double *z) {
    pdl_wait();
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    const int64_t i = rows[t];
    double s = r[i];
    for (int64_t q = luptr[i]; q < dpos[i]; ++q) s = __dsub_rn(s, __dmul_rn(ludata[q], z[luind[q]]));
    z[i] = s;
}
__global__ void k_ilu_bwd_level(const int32_t *rows, int64_t cnt, const int64_t *luptr, const int32_t *luind,
                                const double *ludata, const int64_t *dpos, double *z) {
    pdl_wait();
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    const int64_t i = rows[t];
    double s = z[i];
    for (int64_t q = dpos[i] + 1; q < luptr[i + 1]; ++q) s = __dsub_rn(s, __dmul_rn(ludata[q], z[luind[q]]));
    z[i] = s / ludata[dpos[i]];
}

// offpart_abs_rowsum (smoothers.py:90-96): sequential sum in entry order
__global__ void k_offpart_abs(int64_t n, const int64_t *ro, const int32_t *ci, const double *v, const int64_t *starts,
                              int64_t np_, double *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p = part_of(starts, np_, i), lo = starts[p], hi = starts[p + 1];
    double s = 0.0;
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q)
        if (ci[q] < lo || ci[q] >= hi) s += fabs(v[q]);
    out[i] = s;
}

// the static 2x2 blocks: first singular one per partition (hbgs_kernel's test)
__global__ void k_hbgs_check(const int64_t *ro, const int32_t *ci, const double *v, const double *add,
                             const int64_t *cstart, const int64_t *cs, const int64_t *cp, int64_t np_,
                             int64_t *bad) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np_) return;
    bad[p] = -1;
    for (int64_t t = cstart[p]; t < cstart[p + 1]; ++t) {
        const int64_t i0 = cs[t], i1 = cp[t];
        double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
        for (int64_t q = ro[i0]; q < ro[i0 + 1]; ++q) {
            if (ci[q] == i0) a00 = v[q];
            else if (ci[q] == i1) a01 = v[q];
        }
        for (int64_t q = ro[i1]; q < ro[i1 + 1]; ++q) {
            if (ci[q] == i0) a10 = v[q];
            else if (ci[q] == i1) a11 = v[q];
        }
        a00 += add[i0];
        a11 += add[i1];
        if (__dsub_rn(__dmul_rn(a00, a11), __dmul_rn(a01, a10)) == 0.0) {
            bad[p] = t;
            return;
        }
    }
}

// one hbgs_kernel sweep (_kernels.py:47-93), one thread per partition, cells
// of the partition in entity order; xpre = x before the sweep
__global__ void k_hbgs_sweep(const int64_t *ro, const int32_t *ci, const double *v, const int64_t *starts,
                             const double *add, const int64_t *cstart, const int64_t *cs, const int64_t *cp,
                             int64_t np_, const double *b, double *x, const double *xpre) {
    pdl_wait();
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np_) return;
    const int64_t lo = starts[p], hi = starts[p + 1];
    for (int64_t t = cstart[p]; t < cstart[p + 1]; ++t) {
        const int64_t i0 = cs[t], i1 = cp[t];
        double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
        double r0 = b[i0], r1 = b[i1];
        for (int64_t q = ro[i0]; q < ro[i0 + 1]; ++q) {
            const int64_t j = ci[q];
            const double vv = v[q];
            if (j == i0) a00 = vv;
            else if (j == i1) a01 = vv;
            r0 = __dsub_rn(r0, __dmul_rn(vv, (lo <= j && j < hi) ? x[j] : xpre[j]));
        }
        for (int64_t q = ro[i1]; q < ro[i1 + 1]; ++q) {
            const int64_t j = ci[q];
            const double vv = v[q];
            if (j == i0) a10 = vv;
            else if (j == i1) a11 = vv;
            r1 = __dsub_rn(r1, __dmul_rn(vv, (lo <= j && j < hi) ? x[j] : xpre[j]));
        }
        a00 += add[i0];
        a11 += add[i1];
        const double det = __dsub_rn(__dmul_rn(a00, a11), __dmul_rn(a01, a10));
        x[i0] += __dsub_rn(__dmul_rn(a11, r0), __dmul_rn(a01, r1)) / det;
        x[i1] += __dadd_rn(__dmul_rn(-a10, r0), __dmul_rn(a00, r1)) / det;
    }
}

void upload(DBuf<int64_t> &d, const std::vector<int64_t> &h, cudaStream_t s) {
    d.alloc((int64_t)h.size());
    if (!h.empty())
        PMGR_CUDA(cudaMemcpyAsync(d.p, h.data(), sizeof(int64_t) * h.size(), cudaMemcpyHostToDevice, s));
}

int64_t min_fail(const int64_t *dev, int64_t np_, cudaStream_t s) {
    std::vector<int64_t> h(np_);
    PMGR_CUDA(cudaMemcpyAsync(h.data(), dev, sizeof(int64_t) * np_, cudaMemcpyDeviceToHost, s));
    PMGR_CUDA(cudaStreamSynchronize(s));
    int64_t f = -1;
    for (int64_t x : h)
        if (x >= 0 && (f < 0 || x < f)) f = x;
    return f;
}

// one ILU(k) attempt on M: -1 on success, else the reference's failing row
int64_t iluk(const Csr &M, int k, const std::vector<int64_t> &st, const DBuf<int64_t> &starts, Csr &lu,
             DBuf<int64_t> &dpos, cudaStream_t s) {
    const int64_t n = M.nrows, np_ = (int64_t)st.size() - 1;
    std::vector<int64_t> ro_h(n + 1);
    PMGR_CUDA(cudaMemcpyAsync(ro_h.data(), M.ro.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    PMGR_CUDA(cudaStreamSynchronize(s));
    TBuf<int32_t> lev_ws(n > 0 ? n : 1, s), cols(n > 0 ? n : 1, s);
    TBuf<int64_t> rstart(n > 0 ? n : 1, s), rcnt(n > 0 ? n : 1, s), dposr(n > 0 ? n : 1, s), fail(np_, s);
    TBuf<int> ovf(1, s);
    int64_t factor = 4;
    for (;;) {
        std::vector<int64_t> base(np_), cap(np_);
        int64_t tot = 0;
        for (int64_t p = 0; p < np_; ++p) {
            cap[p] = factor * (ro_h[st[p + 1]] - ro_h[st[p]]) + 2 * (st[p + 1] - st[p]) + 16;
            base[p] = tot;
            tot += cap[p];
        }
        DBuf<int64_t> rbase, rcap;
        upload(rbase, base, s);
        upload(rcap, cap, s);
        TBuf<int32_t> rind(tot, s), rlev(tot, s);
        PMGR_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(int), s));
        PMGR_CUDA(cudaMemsetAsync(rcnt.p, 0, sizeof(int64_t) * (n > 0 ? n : 1), s));
        k_iluk_symbolic<<<grid_for(np_, 32), 32, 0, s>>>(M.ro.p, M.ci.p, starts.p, np_, k, rbase.p, rcap.p, rind.p,
                                                          rlev.p, rstart.p, rcnt.p, dposr.p, lev_ws.p, cols.p,
                                                          fail.p, ovf.p);
        PMGR_LAUNCHED();
        if (read_scalar(ovf.p, s)) {
            factor *= 2;
            continue;
        }
        lu.nrows = lu.ncols = n;
        lu.ro.alloc(n + 1);
        lu.nnz = exclusive_scan_total(rcnt.p, lu.ro.p, n, s);
        lu.ci.alloc(lu.nnz);
        lu.v.alloc(lu.nnz);
        k_ilu_compact<<<grid_for(n, 128), 128, 0, s>>>(n, starts.p, np_, rbase.p, rstart.p, rcnt.p, rind.p, lu.ro.p,
                                                       lu.ci.p);
        PMGR_LAUNCHED();
        dpos.alloc(n > 0 ? n : 1);
        k_dpos_abs<<<grid_for(n, 128), 128, 0, s>>>(n, lu.ro.p, dposr.p, dpos.p);
        PMGR_LAUNCHED();
        break;
    }
    const int64_t sym_fail = min_fail(fail.p, np_, s);
    TBuf<double> w(n > 0 ? n : 1, s);
    TBuf<int64_t> posof(n > 0 ? n : 1, s);
    k_iluk_numeric<<<grid_for(np_, 32), 32, 0, s>>>(M.ro.p, M.ci.p, M.v.p, starts.p, np_, lu.ro.p, lu.ci.p, dpos.p,
                                                     lu.v.p, w.p, posof.p, fail.p);
    PMGR_LAUNCHED();
    const int64_t num_fail = min_fail(fail.p, np_, s);
    if (sym_fail >= 0 && (num_fail < 0 || sym_fail < num_fail)) return sym_fail;
    return num_fail;
}

}  // namespace

std::unique_ptr<GlobalSmoother> smoother_build(std::shared_ptr<const Csr> A, int kind, int ilu_fill, int hbgs_sweeps,
                                               int64_t npartitions, bool interleaved, const int8_t *field_of,
                                               const int32_t *entity_of, cudaStream_t s) {
    auto g = std::make_unique<GlobalSmoother>();
    g->kind = kind;
    g->A = A;
    const int64_t n = A->nrows;
    g->n = n;
    const std::vector<int64_t> st = partition_starts_aligned(n, npartitions, 2);
    g->nparts = (int64_t)st.size() - 1;
    upload(g->starts, st, s);
    if (kind == PMGR_SMOOTHER_ILU) {
        if (ilu_fill < 0) fail(PMGR_ERR_INVALID, "fill level must be >= 0");
        // _IluGlobal (mgr.py:275-281): partition-local couplings only
        const Csr *M = A.get();
        Csr local;
        if (g->nparts > 1) {
            TBuf<int64_t> cnt(n, s);
            k_restrict_count<<<grid_for(n, 128), 128, 0, s>>>(n, A->ro.p, A->ci.p, g->starts.p, g->nparts, cnt.p);
            PMGR_LAUNCHED();
            local.nrows = local.ncols = n;
            local.ro.alloc(n + 1);
            local.nnz = exclusive_scan_total(cnt.p, local.ro.p, n, s);
            local.ci.alloc(local.nnz);
            local.v.alloc(local.nnz);
            k_restrict_fill<<<grid_for(n, 128), 128, 0, s>>>(n, A->ro.p, A->ci.p, A->v.p, g->starts.p, g->nparts,
                                                             local.ro.p, local.ci.p, local.v.p);
            PMGR_LAUNCHED();
            M = &local;
        }
        int64_t bad = iluk(*M, ilu_fill, st, g->starts, g->lu, g->dpos, s);
        if (bad >= 0) {
            // ilu_factor's zero_pivot_shift retry (smoothers.py:176-187)
            TBuf<unsigned long long> mx(1, s);
            PMGR_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long), s));
            if (n > 0) {
                k_max_abs_diag<<<grid_for(n, 256), 256, 0, s>>>(n, M->ro.p, M->ci.p, M->v.p, mx.p);
                PMGR_LAUNCHED();
            }
            const unsigned long long bits = read_scalar(mx.p, s);
            double dmax;
            memcpy(&dmax, &bits, sizeof(double));
            const double shift = 1e-8 * std::max(dmax, 1.0);
            Csr sh;
            TBuf<int64_t> cnt(n, s);
            k_shift_count<<<grid_for(n, 128), 128, 0, s>>>(n, M->ro.p, M->ci.p, M->v.p, shift, cnt.p);
            PMGR_LAUNCHED();
            sh.nrows = sh.ncols = n;
            sh.ro.alloc(n + 1);
            sh.nnz = exclusive_scan_total(cnt.p, sh.ro.p, n, s);
            sh.ci.alloc(sh.nnz);
            sh.v.alloc(sh.nnz);
            k_shift_fill<<<grid_for(n, 128), 128, 0, s>>>(n, M->ro.p, M->ci.p, M->v.p, shift, sh.ro.p, sh.ci.p,
                                                          sh.v.p);
            PMGR_LAUNCHED();
            bad = iluk(sh, ilu_fill, st, g->starts, g->lu, g->dpos, s);
            if (bad >= 0) fail(PMGR_ERR_ZERO_PIVOT, "zero pivot at row " + std::to_string(bad), bad);
        }
        // level-scheduled substitutions when partitions are long: one launch
        // per level instead of one thread walking a whole partition
        int64_t maxrows = 0;
        for (size_t p = 0; p + 1 < st.size(); ++p) maxrows = std::max(maxrows, st[p + 1] - st[p]);
        TBuf<int32_t> lf(n, s), lb(n, s);
        k_ilu_levels<<<grid_for(g->nparts, 32), 32, 0, s>>>(g->starts.p, g->nparts, g->lu.ro.p, g->lu.ci.p,
                                                            g->dpos.p, lf.p, lb.p);
        PMGR_LAUNCHED();
        auto schedule = [&](TBuf<int32_t> &lev, DBuf<int32_t> &rows, std::vector<int64_t> &ptr) {
            thrust::device_ptr<int32_t> lp(lev.p);
            const int32_t top = *thrust::max_element(thrust::cuda::par.on(s), lp, lp + n);
            TBuf<int64_t> cnt(top + 1, s);
            PMGR_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t) * (top + 1), s));
            k_count_levels<<<grid_for(n, 256), 256, 0, s>>>(n, lev.p, cnt.p);
            PMGR_LAUNCHED();
            std::vector<int64_t> c(top + 1);
            PMGR_CUDA(cudaMemcpyAsync(c.data(), cnt.p, sizeof(int64_t) * (top + 1), cudaMemcpyDeviceToHost, s));
            rows.alloc(n);
            thrust::device_ptr<int32_t> rp(rows.p);
            thrust::sequence(thrust::cuda::par.on(s), rp, rp + n);
            thrust::stable_sort_by_key(thrust::cuda::par.on(s), lp, lp + n, rp);
            PMGR_CUDA(cudaStreamSynchronize(s));
            ptr.assign(1, 0);
            for (int64_t x : c) ptr.push_back(ptr.back() + x);
        };
        static const int force = [] {
            const char *e = getenv("PMGR_ILU_LEVELS");
            return e ? atoi(e) : -1;
        }();
        if (n > 0) {
            schedule(lf, g->frows, g->fptr);
            schedule(lb, g->brows, g->bptr);
            const int64_t nlev = (int64_t)g->fptr.size() + (int64_t)g->bptr.size() - 2;
            g->leveled = force >= 0 ? force != 0 : nlev < maxrows;  // ~5 us per level vs ~2 us per row
            if (getenv("PMGR_SETUP_TRACE"))
                fprintf(stderr, "[pmgr setup] ILU(%d) n=%lld nnz=%lld parts=%lld levels fwd=%zu bwd=%zu leveled=%d\n",
                        ilu_fill, (long long)n, (long long)g->lu.nnz, (long long)g->nparts, g->fptr.size() - 1,
                        g->bptr.size() - 1, (int)g->leveled);
        }
        return g;
    }
    // _HbgsGlobal (mgr.py:284-292): per-cell (s, p) blocks, S / P dofs paired by entity
    if (!interleaved) fail(PMGR_ERR_INVALID, "hbgs_sweeps requires an interleaved flow layout");
    g->nsweeps = hbgs_sweeps;
    std::vector<int64_t> sv, pv;
    for (int64_t i = 0; i < n; ++i) {
        if (field_of[i] == 1) sv.push_back(i);
        else if (field_of[i] == 2) pv.push_back(i);
    }
    auto by_entity = [&](std::vector<int64_t> &v) {
        std::stable_sort(v.begin(), v.end(), [&](int64_t a, int64_t b) { return entity_of[a] < entity_of[b]; });
    };
    by_entity(sv);
    by_entity(pv);
    if (sv.size() != pv.size()) fail(PMGR_ERR_INVALID, "hbgs_sweeps requires an interleaved flow layout");
    // cells grouped by the partition of their s row, entity order inside
    const int64_t nc = (int64_t)sv.size();
    std::vector<int64_t> cstart(g->nparts + 1, 0), cs, cp;
    std::vector<int64_t> partc(nc);
    for (int64_t c = 0; c < nc; ++c) {
        partc[c] = (int64_t)(std::upper_bound(st.begin(), st.end(), sv[c]) - st.begin()) - 1;
        ++cstart[partc[c] + 1];
    }
    for (int64_t p = 0; p < g->nparts; ++p) cstart[p + 1] += cstart[p];
    cs.resize(nc);
    cp.resize(nc);
    std::vector<int64_t> fill(cstart.begin(), cstart.end() - 1);
    std::vector<int32_t> ent(nc);
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t t = fill[partc[c]]++;
        cs[t] = sv[c];
        cp[t] = pv[c];
        ent[t] = entity_of[sv[c]];
    }
    upload(g->cstart, cstart, s);
    upload(g->cs, cs, s);
    upload(g->cp, cp, s);
    g->add.alloc(n > 0 ? n : 1);
    if (n > 0) {
        k_offpart_abs<<<grid_for(n, 128), 128, 0, s>>>(n, A->ro.p, A->ci.p, A->v.p, g->starts.p, g->nparts,
                                                       g->add.p);
        PMGR_LAUNCHED();
    }
    TBuf<int64_t> bad(g->nparts, s);
    k_hbgs_check<<<grid_for(g->nparts, 32), 32, 0, s>>>(A->ro.p, A->ci.p, A->v.p, g->add.p, g->cstart.p, g->cs.p,
                                                         g->cp.p, g->nparts, bad.p);
    PMGR_LAUNCHED();
    std::vector<int64_t> hb(g->nparts);
    PMGR_CUDA(cudaMemcpyAsync(hb.data(), bad.p, sizeof(int64_t) * g->nparts, cudaMemcpyDeviceToHost, s));
    PMGR_CUDA(cudaStreamSynchronize(s));
    for (int64_t p = 0; p < g->nparts; ++p)
        if (hb[p] >= 0)
            fail(PMGR_ERR_INVALID, "singular 2x2 diagonal block at cell " + std::to_string(ent[hb[p]]));
    g->xpre.alloc(n > 0 ? n : 1);
    return g;
}

// z = S v (x0 = 0); z may not alias v
namespace {
__global__ void k_lu_slice(int64_t n, int64_t lo, int64_t e0, const int64_t *ro, const int32_t *ci, const double *v,
                           const int64_t *dpos, int64_t *oro, int32_t *oci, double *ov, int64_t *odpos) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    oro[i] = ro[lo + i] - e0;
    if (i == n) return;
    odpos[i] = dpos[lo + i] - e0;
    for (int64_t q = ro[lo + i]; q < ro[lo + i + 1]; ++q) {
        oci[q - e0] = ci[q] - (int32_t)lo;
        ov[q - e0] = v[q];
    }
}
}  // namespace

std::unique_ptr<GlobalSmoother> smoother_slice(const GlobalSmoother &g, int64_t lo, int64_t hi, cudaStream_t s) {
    if (g.kind != PMGR_SMOOTHER_ILU || g.leveled)
        fail(PMGR_ERR_NOT_SUPPORTED,
             "row distribution of a global smoother supports ILU(k) over short partitions (one thread per partition)");
    std::vector<int64_t> st((size_t)g.nparts + 1);
    PMGR_CUDA(cudaMemcpyAsync(st.data(), g.starts.p, sizeof(int64_t) * st.size(), cudaMemcpyDeviceToHost, s));
    PMGR_CUDA(cudaStreamSynchronize(s));
    const auto a = std::lower_bound(st.begin(), st.end(), lo), b = std::lower_bound(st.begin(), st.end(), hi);
    if (a == st.end() || *a != lo || b == st.end() || *b != hi)
        fail(PMGR_ERR_NOT_SUPPORTED,
             "row distribution of an ILU smoother needs its partition boundaries on the rank boundaries");
    auto out = std::make_unique<GlobalSmoother>();
    out->kind = PMGR_SMOOTHER_ILU;
    out->n = hi - lo;
    std::vector<int64_t> ls(a, b + 1);
    for (int64_t &x : ls) x -= lo;
    out->nparts = (int64_t)ls.size() - 1;
    upload(out->starts, ls, s);
    const int64_t n = hi - lo;
    int64_t e0 = 0, e1 = 0;
    PMGR_CUDA(cudaMemcpyAsync(&e0, g.lu.ro.p + lo, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PMGR_CUDA(cudaMemcpyAsync(&e1, g.lu.ro.p + hi, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PMGR_CUDA(cudaStreamSynchronize(s));
    out->lu.alloc(n, n, e1 - e0);
    out->dpos.alloc(n);
    k_lu_slice<<<grid_for(n + 1, 128), 128, 0, s>>>(n, lo, e0, g.lu.ro.p, g.lu.ci.p, g.lu.v.p, g.dpos.p, out->lu.ro.p,
                                                    out->lu.ci.p, out->lu.v.p, out->dpos.p);
    PMGR_LAUNCHED();
    return out;
}

void smoother_apply(GlobalSmoother &g, const double *v, double *z, cudaStream_t s) {
    const int64_t n = g.n;
    if (n == 0) return;
    const unsigned grid = grid_for(g.nparts, 32);
    if (g.kind == PMGR_SMOOTHER_ILU)  // one pass over L\U (+ diagonal positions), v read, z written and re-read
        ledger(csr_pass_bytes(g.lu.nrows, g.lu.ncols, g.lu.nnz) + 8.0 * n + 16.0 * n);
    else if (g.A)
        ledger(g.nsweeps * (csr_pass_bytes(g.A->nrows, g.A->ncols, g.A->nnz) + 40.0 * n));
    if (g.kind == PMGR_SMOOTHER_ILU && g.leveled) {
        for (size_t l = 0; l + 1 < g.fptr.size(); ++l) {
            const int64_t c = g.fptr[l + 1] - g.fptr[l];
            launch_pdl(k_ilu_fwd_level, dim3(grid_for(c, 128)), dim3(128), 0, s, (const int32_t *)g.frows.p + g.fptr[l],
                       c, (const int64_t *)g.lu.ro.p, (const int32_t *)g.lu.ci.p, (const double *)g.lu.v.p,
                       (const int64_t *)g.dpos.p, v, z);
            PMGR_LAUNCHED();
        }
        for (size_t l = 0; l + 1 < g.bptr.size(); ++l) {
            const int64_t c = g.bptr[l + 1] - g.bptr[l];
            launch_pdl(k_ilu_bwd_level, dim3(grid_for(c, 128)), dim3(128), 0, s, (const int32_t *)g.brows.p + g.bptr[l],
                       c, (const int64_t *)g.lu.ro.p, (const int32_t *)g.lu.ci.p, (const double *)g.lu.v.p,
                       (const int64_t *)g.dpos.p, z);
            PMGR_LAUNCHED();
        }
        return;
    }
    if (g.kind == PMGR_SMOOTHER_ILU) {
        launch_pdl(k_ilu_solve, dim3(grid), dim3(32), 0, s, (const int64_t *)g.starts.p, g.nparts,
                   (const int64_t *)g.lu.ro.p, (const int32_t *)g.lu.ci.p, (const double *)g.lu.v.p,
                   (const int64_t *)g.dpos.p, v, z);
        PMGR_LAUNCHED();
        return;
    }
    vec_zero(z, n, s);
    const CsrView A = g.A->view();
    for (int k = 0; k < g.nsweeps; ++k) {
        vec_copy(z, g.xpre.p, n, s);
        launch_pdl(k_hbgs_sweep, dim3(grid), dim3(32), 0, s, A.ro, A.ci, A.v, (const int64_t *)g.starts.p,
                   (const double *)g.add.p, (const int64_t *)g.cstart.p, (const int64_t *)g.cs.p,
                   (const int64_t *)g.cp.p, g.nparts, v, z, (const double *)g.xpre.p);
        PMGR_LAUNCHED();
    }
}

}  // namespace pmgr
