// sj.cu -- builder of the sliced jagged solve copy (SjView, common.cuh).
//
// The large, HBM-streamed operators of the solve phase (A0, the level-0
// displacement block and the fine AMG levels at C3-C5 sizes) are re-laid out
// once at setup so that ONE LANE owns ONE ROW (or one row triple of 3x3
// blocks): rows are grouped in slices of 32; within a slice, position t of
// every row that has a t-th entry is stored contiguously, lane order kept
// (rows shorter than t drop out of the group, so nothing is padded).  A warp
// then streams its slice with fully coalesced loads, every lane summing its
// own row sequentially in stored (ascending column) order: no shuffles, no
// per-row prologue, ~20x fewer instructions per byte than a warp per row.
// The entries themselves are the CSR's (or the block-prefix copy's), only
// permuted inside each slice.
#include <cstdlib>

#include "common.cuh"

namespace pmgr {

namespace {

// lengths of the scalar slices' lane rows and the slice totals
// triple mode (gs < ntslice): slice gs = 3 S + g holds rows 3 (32 S + lane) + g
// consecutive slices hold 32 >> lg rows, 2^lg lanes each: lane gl of a row
// owns its entries g t + gl, so its length is the number of such entries
__global__ void k_sj_slen(int64_t nslice, int64_t ntslice, int64_t prow, int64_t row0, int64_t n, int lg,
                          const int64_t *__restrict__ ro, int32_t *__restrict__ slen, int64_t *__restrict__ tot) {
    const int64_t gs = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gs >= nslice) return;
    int64_t row;
    bool ok;
    if (gs < ntslice) {
        const int64_t S = gs / 3;
        const int g = (int)(gs - 3 * S);
        row = 3 * (32 * S + lane) + g;
        ok = row < prow;
    } else {
        row = row0 + (32 >> lg) * (gs - ntslice) + (lane >> lg);
        ok = row < n;
    }
    int len = ok ? (int)(ro[row + 1] - ro[row]) : 0;
    if (gs >= ntslice && lg > 0) {
        const int g = 1 << lg, gl = lane & (g - 1);
        len = len > gl ? (len - gl + g - 1) >> lg : 0;
    }
    slen[gs * 32 + lane] = len;
    int64_t t = len;
    t = warp_sum_i64(t);
    if (lane == 0) tot[gs] = t;
}

__global__ void k_sj_sfill(int64_t nslice, int64_t ntslice, int64_t row0, int lg, const int64_t *__restrict__ ro,
                           const int32_t *__restrict__ ci, const double *__restrict__ v,
                           const int64_t *__restrict__ sptr, const int32_t *__restrict__ slen,
                           int32_t *__restrict__ sci, double *__restrict__ sv) {
    const int64_t gs = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (gs >= nslice) return;
    int64_t row;
    if (gs < ntslice) {
        const int64_t S = gs / 3;
        row = 3 * (32 * S + lane) + (gs - 3 * S);
    } else {
        row = row0 + (32 >> lg) * (gs - ntslice) + (lane >> lg);
    }
    const int len = slen[gs * 32 + lane];
    const int sh = gs < ntslice ? 0 : lg;
    const int gl = lane & ((1 << sh) - 1);
    const int64_t q0 = len > 0 ? ro[row] + gl : 0;
    int maxlen = len;
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(FULL, maxlen, o));
    const unsigned lt = (1u << lane) - 1u;
    int64_t off = sptr[gs];
    for (int t = 0; t < maxlen; ++t) {
        const bool a = t < len;
        const unsigned m = __ballot_sync(FULL, a);
        if (a) {
            const int64_t w = off + __popc(m & lt);
            sci[w] = ci[q0 + ((int64_t)t << sh)];
            sv[w] = v[q0 + ((int64_t)t << sh)];
        }
        off += __popc(m);
    }
}

__global__ void k_sj_blen(int64_t nbslice, int64_t nb, const int64_t *__restrict__ bro, int32_t *__restrict__ blen,
                          int64_t *__restrict__ tot) {
    const int64_t S = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (S >= nbslice) return;
    const int64_t I = 32 * S + lane;
    const int len = I < nb ? (int)(bro[I + 1] - bro[I]) : 0;
    blen[S * 32 + lane] = len;
    int64_t t = len;
    t = warp_sum_i64(t);
    if (lane == 0) tot[S] = t;
}

__global__ void k_sj_bfill(int64_t nbslice, const int64_t *__restrict__ bro, const int32_t *__restrict__ bci,
                           const double *__restrict__ bval, const int64_t *__restrict__ bptr,
                           const int32_t *__restrict__ blen, int32_t *__restrict__ oci, double *__restrict__ oval) {
    const int64_t S = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (S >= nbslice) return;
    const int len = blen[S * 32 + lane];
    const int64_t b0 = len > 0 ? bro[32 * S + lane] : 0;
    int maxlen = len;
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(FULL, maxlen, o));
    const unsigned lt = (1u << lane) - 1u;
    int64_t off = bptr[S];
    for (int t = 0; t < maxlen; ++t) {
        const bool a = t < len;
        const unsigned m = __ballot_sync(FULL, a);
        const int k = __popc(m);
        if (a) {
            const int r = __popc(m & lt);
            oci[off + r] = bci[b0 + t];
            const double *src = bval + 9 * (b0 + t);
            double *dst = oval + 9 * off + r;
#pragma unroll
            for (int e = 0; e < 9; ++e) dst[(int64_t)e * k] = src[e];
        }
        off += k;
    }
}

}  // namespace

// One lane per row needs rows to fill the machine: operators below
// PMGR_SJ_MIN_ROWS rows (one wave of 148 SMs x 48 warps is ~227k lanes) or
// PMGR_SJ_MIN_NNZ entries keep the lane-group kernels (measured at C4: the
// 146k-row AMG level 83 vs 70 us, a 5k-row level with 1400 entries per row
// 600 vs 18 us; from 570k rows up the copy wins).
int64_t sj_min_nnz() {
    static const int64_t v = [] {
        const char *e = getenv("PMGR_SJ_MIN_NNZ");
        return e ? atoll(e) : (int64_t)1 << 22;
    }();
    return v;
}
int64_t sj_min_rows() {
    static const int64_t v = [] {
        const char *e = getenv("PMGR_SJ_MIN_ROWS");
        return e ? atoll(e) : (int64_t)200000;
    }();
    return v;
}
bool sj_wanted(int64_t nrows, int64_t nnz) { return nnz >= sj_min_nnz() && nrows >= sj_min_rows(); }

void csr_make_sj(Csr &A, cudaStream_t s, bool force) {
    static const bool off = getenv("PMGR_NO_SJ") && getenv("PMGR_NO_SJ")[0] != '0';
    A.sj.reset();
    A.sj_tried = false;
    if (off || A.nrows == 0 || A.nnz == 0 || !(force || A.sj_want)) return;
    auto J = std::make_shared<Sj>();
    const bool has_blocks = A.nbrows > 0;
    // ---- block piece (own blocks, or borrowed from the operator that owns them)
    if (has_blocks) {
        if (A.blk_src) {
            const Csr *src = A.blk_src.get();
            if (!src->sj || src->sj->nbrows != A.nbrows || src->sj->blk_src) return;  // the owner has no copy
            J->blk_src = src->sj;
        } else {
            const int64_t nb = A.nbrows, nbs = (nb + 31) / 32;
            J->nbslice = nbs;
            J->nbrows = nb;
            J->nblocks = A.nblocks;
            J->blen.alloc(nbs * 32);
            J->bptr.alloc(nbs + 1);
            TBuf<int64_t> tot(nbs, s);
            k_sj_blen<<<grid_for(nbs * 32, 256), 256, 0, s>>>(nbs, nb, A.bro.p, J->blen.p, tot.p);
            PMGR_LAUNCHED();
            exclusive_scan_total(tot.p, J->bptr.p, nbs, s);
            J->bci.alloc(A.nblocks);
            J->bval.alloc(9 * A.nblocks);
            k_sj_bfill<<<grid_for(nbs * 32, 256), 256, 0, s>>>(nbs, A.bro.p, A.bci.p, A.bval.p, J->bptr.p, J->blen.p,
                                                               J->bci.p, J->bval.p);
            PMGR_LAUNCHED();
        }
    }
    // ---- scalar piece: the remainder CSR of a block-prefix operator, else the CSR
    const int64_t *ro = has_blocks ? A.rro.p : A.ro.p;
    const int32_t *ci = has_blocks ? A.rci.p : A.ci.p;
    const double *v = has_blocks ? A.rv.p : A.v.p;
    const int64_t nent = has_blocks ? A.nrem : A.nnz;
    if (ro != nullptr && nent > 0) {
        const int64_t prow = has_blocks ? 3 * A.nbrows : 0;
        const int64_t nbs = has_blocks ? (A.nbrows + 31) / 32 : 0;
        J->ntslice = 3 * nbs;
        J->row0 = prow;
        const double mean = (double)nent / (double)(A.nrows > 0 ? A.nrows : 1);
        // lanes per row of the consecutive slices (PMGR_SJ_G): four for long-row
        // operators of fewer than PMGR_SJ_G_ROWS rows, which one lane per row
        // leaves short of warps (C4 AMG level 2, 573k rows x 164: 270 -> 252 us;
        // level 1, 2.4M rows: 737 us with one lane, 741 with four), decided on
        // the global operator's statistics
        const int64_t grows = A.g_rows > 0 ? A.g_rows : A.nrows;
        const double gmean_rows = (double)(A.g_nnz > 0 ? A.g_nnz : A.nnz) / (double)(grows > 0 ? grows : 1);
        static const int gforce = [] {
            const char *e = getenv("PMGR_SJ_G");
            return e ? atoi(e) : 0;
        }();
        static const double gmean = [] {
            const char *e = getenv("PMGR_SJ_G_MEAN");
            return e ? atof(e) : 64.0;
        }();
        static const int64_t grows_max = [] {
            const char *e = getenv("PMGR_SJ_G_ROWS");
            return e ? atoll(e) : (int64_t)1000000;
        }();
        static const int gbig = [] {
            const char *e = getenv("PMGR_SJ_GBIG");
            return e ? atoi(e) : 4;
        }();
        int g = gforce > 0 ? gforce : (!has_blocks && gmean_rows >= gmean && grows < grows_max ? gbig : 1);
        J->lg = g >= 32 ? 5 : g >= 16 ? 4 : g >= 8 ? 3 : g >= 4 ? 2 : g >= 2 ? 1 : 0;
        const int64_t R = 32 >> J->lg;
        J->ncslice = (A.nrows - prow + R - 1) / R;
        const int64_t ns = J->ntslice + J->ncslice;
        J->nent = nent;
        J->slen.alloc(ns * 32);
        J->sptr.alloc(ns + 1);
        TBuf<int64_t> tot(ns, s);
        k_sj_slen<<<grid_for(ns * 32, 256), 256, 0, s>>>(ns, J->ntslice, prow, J->row0, A.nrows, J->lg, ro,
                                                         J->slen.p, tot.p);
        PMGR_LAUNCHED();
        exclusive_scan_total(tot.p, J->sptr.p, ns, s);
        J->sci.alloc(nent);
        J->sv.alloc(nent);
        k_sj_sfill<<<grid_for(ns * 32, 256), 256, 0, s>>>(ns, J->ntslice, J->row0, J->lg, ro, ci, v, J->sptr.p,
                                                          J->slen.p, J->sci.p, J->sv.p);
        PMGR_LAUNCHED();
        const double lmean = mean / (double)(1 << J->lg);  // positions per lane
        J->u = lmean <= 6.0 ? 2 : lmean <= 24.0 ? 4 : 8;
    }
    A.sj = J;
}

}  // namespace pmgr
