// dsetup.cu -- distributed setup primitives (see dsetup.cuh).
#include <algorithm>

#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sort.h>
#include <thrust/unique.h>

#include "dist.cuh"
#include "dsetup.cuh"

namespace pmgr {

namespace {

__global__ void k_sel(int64_t n, const int8_t *is_c, int want, int64_t *o) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) o[i] = (is_c[i] != 0) == (want != 0) ? 1 : 0;
}

__global__ void k_row_len(int64_t n, const int64_t *ro, int64_t *len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) len[i] = ro[i + 1] - ro[i];
}

__global__ void k_clamp_ro(int64_t n, const int64_t *ro, int64_t lo, int64_t hi, int64_t *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    const int64_t a = ro[lo], b = ro[hi];
    int64_t v = ro[i];
    v = v < a ? a : (v > b ? b : v);
    out[i] = v - a;
}

// owned row t: total length over the nr received pieces
__global__ void k_sum_pieces(int64_t m, int nr, const int64_t *rlen, int64_t lo, int64_t *tot) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= m) return;
    int64_t s = 0;
    for (int p = 0; p < nr; ++p) s += rlen[(int64_t)p * m + t];
    tot[lo + t] = s;
}

// owned row t: the pieces of ranks 0..nr-1 in order
__global__ void k_merge_pieces(int64_t m, int nr, const int64_t *rlen, const int64_t *soff, const int64_t *poff,
                               const int32_t *rci, const double *rv, int64_t lo, const int64_t *ro, int32_t *ci,
                               double *v) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= m) return;
    int64_t dst = ro[lo + t];
    for (int p = 0; p < nr; ++p) {
        const int64_t len = rlen[(int64_t)p * m + t];
        const int64_t src = poff[p] + soff[(int64_t)p * (m + 1) + t];
        for (int64_t k = 0; k < len; ++k) {
            ci[dst + k] = rci[src + k];
            if (v) v[dst + k] = rv[src + k];
        }
        dst += len;
    }
}

__global__ void k_gather_len(int64_t k, const int64_t *ids, const int64_t *ro, int64_t *len) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < k) len[t] = ro[ids[t] + 1] - ro[ids[t]];
}

__global__ void k_pack_rows(int64_t k, const int64_t *ids, const int64_t *ro, const int32_t *ci, const double *v,
                            const int64_t *off, int32_t *oci, double *ov) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= k) return;
    const int64_t b = ro[ids[t]], e = ro[ids[t] + 1], o = off[t];
    for (int64_t q = b; q < e; ++q) {
        oci[o + q - b] = ci[q];
        ov[o + q - b] = v[q];
    }
}

__global__ void k_scatter_len(int64_t k, const int64_t *ids, const int64_t *len, int64_t *tot) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < k) tot[ids[t]] += len[t];
}

__global__ void k_copy_rows(int64_t n, const int64_t *ro, const int32_t *ci, const double *v, const int64_t *nro,
                            int32_t *nci, double *nv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t b = ro[i], e = ro[i + 1], o = nro[i];
    for (int64_t q = b; q < e; ++q) {
        nci[o + q - b] = ci[q];
        nv[o + q - b] = v[q];
    }
}

// fetched row t (global id ids[t]) appended after the row's own entries
__global__ void k_place_rows(int64_t k, const int64_t *ids, const int64_t *len, const int64_t *soff,
                             const int32_t *rci, const double *rv, const int64_t *yro, const int64_t *nro,
                             int32_t *nci, double *nv) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= k) return;
    const int64_t g = ids[t];
    const int64_t o = nro[g] + (yro[g + 1] - yro[g]);
    for (int64_t q = 0; q < len[t]; ++q) {
        nci[o + q] = rci[soff[t] + q];
        nv[o + q] = rv[soff[t] + q];
    }
}

__global__ void k_outside(int64_t rlo, int64_t rhi, const int64_t *ro, const int32_t *ci, int64_t clo, int64_t chi,
                          int64_t *out, unsigned long long *cnt) {
    const int64_t i = rlo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= rhi) return;
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q) {
        const int64_t c = ci[q];
        if (c < clo || c >= chi) out[atomicAdd(cnt, 1ull)] = c;
    }
}

__global__ void k_maxrow_range(int64_t lo, int64_t hi, const int64_t *ro, unsigned long long *out) {
    unsigned long long m = 0;
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long l = (unsigned long long)(ro[i + 1] - ro[i]);
        m = l > m ? l : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(FULL, m, o);
        m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_diag_inv_range(int64_t lo, int64_t hi, const int64_t *ro, const int32_t *ci, const double *v,
                                 double *dinv, unsigned long long *bad) {
    const int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= hi) return;
    double d = 0.0;
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q)
        if (ci[q] == i) {
            d = v[q];
            break;
        }
    if (d == 0.0) atomicMin(bad, (unsigned long long)i);
    dinv[i] = __ddiv_rn(1.0, d);
}

std::vector<int64_t> host_at(const int64_t *dev, const std::vector<int64_t> &idx, cudaStream_t s) {
    std::vector<int64_t> out(idx.size());
    for (size_t k = 0; k < idx.size(); ++k)
        PMGR_CUDA(cudaMemcpyAsync(&out[k], dev + idx[k], sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PMGR_CUDA(cudaStreamSynchronize(s));
    return out;
}

}  // namespace

std::vector<int64_t> ds_sub_bounds(const std::vector<int64_t> &start, const int8_t *is_c, int64_t n, bool want,
                                   cudaStream_t s) {
    TBuf<int64_t> sel(n > 0 ? n : 1, s), sc(n + 1, s);
    if (n > 0) {
        k_sel<<<grid_for(n, 256), 256, 0, s>>>(n, is_c, want ? 1 : 0, sel.p);
        PMGR_LAUNCHED();
    }
    exclusive_scan_total(sel.p, sc.p, n, s);
    return host_at(sc.p, start, s);
}

int64_t ds_allsum(const DistSetup &d, int64_t v, cudaStream_t s) {
    std::vector<int64_t> snd(d.nranks, v), rcv;
    d.tr->alltoall_counts(snd, rcv, s);
    int64_t t = 0;
    for (int64_t x : rcv) t += x;
    return t;
}

int64_t ds_allmax(const DistSetup &d, int64_t v, cudaStream_t s) {
    std::vector<int64_t> snd(d.nranks, v), rcv;
    d.tr->alltoall_counts(snd, rcv, s);
    int64_t t = rcv.empty() ? v : rcv[0];
    for (int64_t x : rcv) t = std::max(t, x);
    return t;
}

void ds_partial_rows(const Csr &A, int64_t lo, int64_t hi, Csr &out, cudaStream_t s) {
    const int64_t n = A.nrows;
    const std::vector<int64_t> e = host_at(A.ro.p, {lo, hi}, s);
    out.alloc(n, A.ncols, e[1] - e[0]);
    k_clamp_ro<<<grid_for(n + 1, 256), 256, 0, s>>>(n, A.ro.p, lo, hi, out.ro.p);
    PMGR_LAUNCHED();
    if (out.nnz > 0) {
        PMGR_CUDA(cudaMemcpyAsync(out.ci.p, A.ci.p + e[0], sizeof(int32_t) * out.nnz, cudaMemcpyDeviceToDevice, s));
        PMGR_CUDA(cudaMemcpyAsync(out.v.p, A.v.p + e[0], sizeof(double) * out.nnz, cudaMemcpyDeviceToDevice, s));
    }
}

void ds_rows_to_owners(const DistSetup &d, const Csr &X, Csr &out, cudaStream_t s) {
    const int nr = d.nranks;
    const int64_t n = X.nrows, lo = d.lo(), m = d.hi() - d.lo();
    TBuf<int64_t> len(n > 0 ? n : 1, s);
    if (n > 0) {
        k_row_len<<<grid_for(n, 256), 256, 0, s>>>(n, X.ro.p, len.p);
        PMGR_LAUNCHED();
    }
    const std::vector<int64_t> eq = host_at(X.ro.p, d.start, s);
    std::vector<int64_t> scnt(nr), rcnt;
    for (int q = 0; q < nr; ++q) scnt[q] = eq[q + 1] - eq[q];
    d.tr->alltoall_counts(scnt, rcnt, s);
    std::vector<int64_t> poff(nr + 1, 0);
    for (int p = 0; p < nr; ++p) poff[p + 1] = poff[p] + rcnt[p];
    TBuf<int64_t> rlen((int64_t)nr * m > 0 ? (int64_t)nr * m : 1, s);
    TBuf<int32_t> rci(poff[nr] > 0 ? poff[nr] : 1, s);
    TBuf<double> rv(X.v.p && poff[nr] > 0 ? poff[nr] : 1, s);
    std::vector<const void *> sp(nr);
    std::vector<void *> rp(nr);
    std::vector<int64_t> sb(nr), rb(nr);
    for (int q = 0; q < nr; ++q) {
        sp[q] = len.p + d.start[q];
        sb[q] = 8 * (d.start[q + 1] - d.start[q]);
        rp[q] = rlen.p + (int64_t)q * m;
        rb[q] = 8 * m;
    }
    d.tr->alltoallv(sp, sb, rp, rb, s);
    for (int q = 0; q < nr; ++q) {
        sp[q] = X.ci.p + eq[q];
        sb[q] = 4 * scnt[q];
        rp[q] = rci.p + poff[q];
        rb[q] = 4 * rcnt[q];
    }
    d.tr->alltoallv(sp, sb, rp, rb, s);
    if (X.v.p) {
        for (int q = 0; q < nr; ++q) {
            sp[q] = X.v.p + eq[q];
            sb[q] = 8 * scnt[q];
            rp[q] = rv.p + poff[q];
            rb[q] = 8 * rcnt[q];
        }
        d.tr->alltoallv(sp, sb, rp, rb, s);
    }
    // per piece: offsets of its rows inside the piece
    TBuf<int64_t> soff((int64_t)nr * (m + 1), s);
    for (int p = 0; p < nr; ++p) exclusive_scan_total(rlen.p + (int64_t)p * m, soff.p + (int64_t)p * (m + 1), m, s);
    TBuf<int64_t> tot(n > 0 ? n : 1, s);
    PMGR_CUDA(cudaMemsetAsync(tot.p, 0, sizeof(int64_t) * (size_t)(n > 0 ? n : 1), s));
    if (m > 0) {
        k_sum_pieces<<<grid_for(m, 256), 256, 0, s>>>(m, nr, rlen.p, lo, tot.p);
        PMGR_LAUNCHED();
    }
    out.nrows = n;
    out.ncols = X.ncols;
    out.ro.alloc(n + 1);
    out.nnz = exclusive_scan_total(tot.p, out.ro.p, n, s);
    out.ci.alloc(out.nnz);
    if (X.v.p) out.v.alloc(out.nnz);
    else out.v.release();
    TBuf<int64_t> poff_d(nr + 1, s);
    PMGR_CUDA(cudaMemcpyAsync(poff_d.p, poff.data(), sizeof(int64_t) * (nr + 1), cudaMemcpyHostToDevice, s));
    if (m > 0) {
        k_merge_pieces<<<grid_for(m, 128), 128, 0, s>>>(m, nr, rlen.p, soff.p, poff_d.p, rci.p,
                                                       X.v.p ? rv.p : nullptr, lo, out.ro.p, out.ci.p,
                                                       X.v.p ? out.v.p : nullptr);
        PMGR_LAUNCHED();
    }
    PMGR_CUDA(cudaStreamSynchronize(s));
}

void ds_fetch_rows(const DistSetup &d, const Csr &Y, const std::vector<int64_t> &want, Csr &Yext, cudaStream_t s) {
    const int nr = d.nranks;
    const int64_t n = Y.nrows;
    // requests: my wanted ids per owner
    std::vector<int64_t> wcnt(nr, 0), woff(nr + 1, 0);
    for (int q = 0; q < nr; ++q) {
        const auto a = std::lower_bound(want.begin(), want.end(), d.start[q]);
        const auto b = std::lower_bound(want.begin(), want.end(), d.start[q + 1]);
        wcnt[q] = b - a;
        woff[q] = a - want.begin();
        if (q == d.rank && wcnt[q] > 0) fail(PMGR_ERR_INVALID, "fetch of an owned row");
    }
    woff[nr] = (int64_t)want.size();
    std::vector<int64_t> qcnt;  // ids each peer asks me for
    d.tr->alltoall_counts(wcnt, qcnt, s);
    std::vector<int64_t> qoff(nr + 1, 0);
    for (int p = 0; p < nr; ++p) qoff[p + 1] = qoff[p] + qcnt[p];
    const int64_t nw = (int64_t)want.size(), nq = qoff[nr];
    TBuf<int64_t> wdev(nw > 0 ? nw : 1, s), qdev(nq > 0 ? nq : 1, s);
    if (nw > 0) PMGR_CUDA(cudaMemcpyAsync(wdev.p, want.data(), sizeof(int64_t) * nw, cudaMemcpyHostToDevice, s));
    std::vector<const void *> sp(nr);
    std::vector<void *> rp(nr);
    std::vector<int64_t> sb(nr), rb(nr);
    for (int q = 0; q < nr; ++q) {
        sp[q] = wdev.p + woff[q];
        sb[q] = 8 * wcnt[q];
        rp[q] = qdev.p + qoff[q];
        rb[q] = 8 * qcnt[q];
    }
    d.tr->alltoallv(sp, sb, rp, rb, s);
    // answers: lengths, then the packed rows
    TBuf<int64_t> qlen(nq > 0 ? nq : 1, s), qpos(nq + 1, s);
    if (nq > 0) {
        k_gather_len<<<grid_for(nq, 256), 256, 0, s>>>(nq, qdev.p, Y.ro.p, qlen.p);
        PMGR_LAUNCHED();
    }
    const int64_t qtot = exclusive_scan_total(qlen.p, qpos.p, nq, s);
    TBuf<int32_t> qci(qtot > 0 ? qtot : 1, s);
    TBuf<double> qv(qtot > 0 ? qtot : 1, s);
    if (nq > 0) {
        k_pack_rows<<<grid_for(nq, 128), 128, 0, s>>>(nq, qdev.p, Y.ro.p, Y.ci.p, Y.v.p, qpos.p, qci.p, qv.p);
        PMGR_LAUNCHED();
    }
    std::vector<int64_t> qe = host_at(qpos.p, qoff, s);  // entry offsets per peer
    std::vector<int64_t> ecnt(nr), rcnt;
    for (int p = 0; p < nr; ++p) ecnt[p] = qe[p + 1] - qe[p];
    d.tr->alltoall_counts(ecnt, rcnt, s);
    std::vector<int64_t> roff(nr + 1, 0);
    for (int q = 0; q < nr; ++q) roff[q + 1] = roff[q] + rcnt[q];
    TBuf<int64_t> wlen(nw > 0 ? nw : 1, s), wpos(nw + 1, s);
    TBuf<int32_t> wci(roff[nr] > 0 ? roff[nr] : 1, s);
    TBuf<double> wv(roff[nr] > 0 ? roff[nr] : 1, s);
    for (int q = 0; q < nr; ++q) {
        sp[q] = qlen.p + qoff[q];
        sb[q] = 8 * qcnt[q];
        rp[q] = wlen.p + woff[q];
        rb[q] = 8 * wcnt[q];
    }
    d.tr->alltoallv(sp, sb, rp, rb, s);
    for (int q = 0; q < nr; ++q) {
        sp[q] = qci.p + qe[q];
        sb[q] = 4 * ecnt[q];
        rp[q] = wci.p + roff[q];
        rb[q] = 4 * rcnt[q];
    }
    d.tr->alltoallv(sp, sb, rp, rb, s);
    for (int q = 0; q < nr; ++q) {
        sp[q] = qv.p + qe[q];
        sb[q] = 8 * ecnt[q];
        rp[q] = wv.p + roff[q];
        rb[q] = 8 * rcnt[q];
    }
    d.tr->alltoallv(sp, sb, rp, rb, s);
    exclusive_scan_total(wlen.p, wpos.p, nw, s);
    // Yext: Y's rows plus the fetched ones
    TBuf<int64_t> tot(n > 0 ? n : 1, s);
    if (n > 0) {
        k_row_len<<<grid_for(n, 256), 256, 0, s>>>(n, Y.ro.p, tot.p);
        PMGR_LAUNCHED();
    }
    if (nw > 0) {
        k_scatter_len<<<grid_for(nw, 256), 256, 0, s>>>(nw, wdev.p, wlen.p, tot.p);
        PMGR_LAUNCHED();
    }
    Yext.nrows = n;
    Yext.ncols = Y.ncols;
    Yext.ro.alloc(n + 1);
    Yext.nnz = exclusive_scan_total(tot.p, Yext.ro.p, n, s);
    Yext.ci.alloc(Yext.nnz);
    Yext.v.alloc(Yext.nnz);
    if (n > 0) {
        k_copy_rows<<<grid_for(n, 128), 128, 0, s>>>(n, Y.ro.p, Y.ci.p, Y.v.p, Yext.ro.p, Yext.ci.p, Yext.v.p);
        PMGR_LAUNCHED();
    }
    if (nw > 0) {
        k_place_rows<<<grid_for(nw, 128), 128, 0, s>>>(nw, wdev.p, wlen.p, wpos.p, wci.p, wv.p, Y.ro.p, Yext.ro.p,
                                                       Yext.ci.p, Yext.v.p);
        PMGR_LAUNCHED();
    }
    PMGR_CUDA(cudaStreamSynchronize(s));
}

void ds_gather_rows(const DistSetup &d, const Csr &X, Csr &full, cudaStream_t s) {
    const int nr = d.nranks;
    const int64_t n = X.nrows, lo = d.lo(), hi = d.hi();
    const std::vector<int64_t> e = host_at(X.ro.p, {lo, hi}, s);
    std::vector<int64_t> mine(nr, e[1] - e[0]), ecnt;
    d.tr->alltoall_counts(mine, ecnt, s);
    TBuf<int64_t> len(n > 0 ? n : 1, s), flen(n > 0 ? n : 1, s);
    if (n > 0) {
        k_row_len<<<grid_for(n, 256), 256, 0, s>>>(n, X.ro.p, len.p);
        PMGR_LAUNCHED();
    }
    std::vector<const void *> sp(nr);
    std::vector<void *> rp(nr);
    std::vector<int64_t> sb(nr), rb(nr);
    for (int q = 0; q < nr; ++q) {
        sp[q] = len.p + lo;
        sb[q] = 8 * (hi - lo);
        rp[q] = flen.p + d.start[q];
        rb[q] = 8 * (d.start[q + 1] - d.start[q]);
    }
    d.tr->alltoallv(sp, sb, rp, rb, s);
    full.nrows = n;
    full.ncols = X.ncols;
    full.ro.alloc(n + 1);
    full.nnz = exclusive_scan_total(flen.p, full.ro.p, n, s);
    full.ci.alloc(full.nnz);
    full.v.alloc(full.nnz);
    const std::vector<int64_t> fo = host_at(full.ro.p, d.start, s);
    for (int q = 0; q < nr; ++q) {
        sp[q] = X.ci.p + e[0];
        sb[q] = 4 * (e[1] - e[0]);
        rp[q] = full.ci.p + fo[q];
        rb[q] = 4 * ecnt[q];
    }
    d.tr->alltoallv(sp, sb, rp, rb, s);
    for (int q = 0; q < nr; ++q) {
        sp[q] = X.v.p + e[0];
        sb[q] = 8 * (e[1] - e[0]);
        rp[q] = full.v.p + fo[q];
        rb[q] = 8 * ecnt[q];
    }
    d.tr->alltoallv(sp, sb, rp, rb, s);
}

void ds_gather_segment(const DistSetup &d, void *arr, size_t elem, cudaStream_t s) {
    const int nr = d.nranks;
    char *a = static_cast<char *>(arr);
    std::vector<const void *> sp(nr);
    std::vector<void *> rp(nr);
    std::vector<int64_t> sb(nr), rb(nr);
    for (int q = 0; q < nr; ++q) {
        const bool self = q == d.rank;
        sp[q] = a + elem * d.lo();
        sb[q] = self ? 0 : (int64_t)elem * (d.hi() - d.lo());
        rp[q] = a + elem * d.start[q];
        rb[q] = self ? 0 : (int64_t)elem * (d.start[q + 1] - d.start[q]);
    }
    d.tr->alltoallv(sp, sb, rp, rb, s);
}

std::vector<int64_t> ds_cols_outside(const Csr &X, int64_t rlo, int64_t rhi, int64_t clo, int64_t chi,
                                     cudaStream_t s) {
    std::vector<int64_t> out;
    if (rhi <= rlo) return out;
    const std::vector<int64_t> e = host_at(X.ro.p, {rlo, rhi}, s);
    if (e[1] <= e[0]) return out;
    TBuf<int64_t> buf(e[1] - e[0], s);
    TBuf<unsigned long long> cnt(1, s);
    PMGR_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), s));
    k_outside<<<grid_for(rhi - rlo, 128), 128, 0, s>>>(rlo, rhi, X.ro.p, X.ci.p, clo, chi, buf.p, cnt.p);
    PMGR_LAUNCHED();
    const int64_t c = (int64_t)read_scalar(cnt.p, s);
    if (c == 0) return out;
    thrust::device_ptr<int64_t> b(buf.p);
    thrust::sort(thrust::cuda::par.on(s), b, b + c);
    const int64_t u = thrust::unique(thrust::cuda::par.on(s), b, b + c) - b;
    out.resize(u);
    PMGR_CUDA(cudaMemcpyAsync(out.data(), buf.p, sizeof(int64_t) * u, cudaMemcpyDeviceToHost, s));
    PMGR_CUDA(cudaStreamSynchronize(s));
    return out;
}

void ds_finalize(const DistSetup *d, Csr &A, cudaStream_t s, bool build_sj) {
    // a partial (owned-rows) operator is never applied: its rank-local slices
    // are (dist.cu), and they take the sliced jagged copy when the GLOBAL
    // operator is large enough
    csr_finalize(A, s, build_sj && d == nullptr);
    if (!d) return;
    // the global operator's statistics decide the lane group and long rows
    TBuf<unsigned long long> m(1, s);
    PMGR_CUDA(cudaMemsetAsync(m.p, 0, sizeof(unsigned long long), s));
    if (d->hi() > d->lo()) {
        const unsigned g = grid_for(d->hi() - d->lo(), 256);
        k_maxrow_range<<<g < 1024 ? g : 1024, 256, 0, s>>>(d->lo(), d->hi(), A.ro.p, m.p);
        PMGR_LAUNCHED();
    }
    const int64_t gmax = ds_allmax(*d, (int64_t)read_scalar(m.p, s), s);
    const int64_t gnnz = ds_allsum(*d, A.nnz, s);
    A.maxrow = gmax;
    const double mean = A.nrows ? (double)gnnz / (double)A.nrows : 0.0;
    const int gm = spmv_lanes_mean(mean);
    static const bool no_long = getenv("PMGR_NO_LONG_ROWS") && getenv("PMGR_NO_LONG_ROWS")[0] != '0';
    A.long_len = (!no_long && gmax > 16 * gm) ? 16 * gm : 0;
    csr_long_rows(A, s);
    A.lanes = (A.long_len > 0 || gmax <= 16 * gm) ? gm : 32;
    A.lanes_u = spmv_u_for(gnnz, A.nrows, A.lanes);
    A.sj_want = sj_wanted(A.nrows, gnnz);
    A.g_rows = A.nrows;
    A.g_nnz = gnnz;
}

int64_t ds_diag_inverse(const Csr &A, int64_t lo, int64_t hi, double *dinv, cudaStream_t s) {
    if (hi <= lo) return -1;
    TBuf<unsigned long long> bad(1, s);
    PMGR_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), s));
    k_diag_inv_range<<<grid_for(hi - lo, 256), 256, 0, s>>>(lo, hi, A.ro.p, A.ci.p, A.v.p, dinv, bad.p);
    PMGR_LAUNCHED();
    const unsigned long long b = read_scalar(bad.p, s);
    return b == ~0ull ? -1 : (int64_t)b;
}

}  // namespace pmgr
