// csr.cu -- setup-phase sparse kernels with the reference's exact arithmetic.
//
//  * csr_transpose     scipy .T.tocsr(): rows of the result in ascending
//                      source-row order (stable counting scatter).
//  * spgemm            scipy csr_matmat order: C_ik = seq sum over j ascending
//                      in row i of X of X_ij*Y_jk from 0.0.
//                      Two passes (symbolic count, numeric fill) with a hash
//                      accumulator per warp in shared memory; rows whose
//                      candidate set cannot fit fall back to a per-row hash
//                      table in global memory.  Each j is processed by the
//                      whole warp (lanes over the distinct k of row j), so
//                      every output entry is accumulated in ascending j --
//                      bit-identical to the sequential product.  Rows are
//                      then key-sorted (CUB segmented sort) and, in mode 0,
//                      compacted without exact zeros (scipy's zero drop).
//  * csr_subtract      scipy csr_binop_csr_canonical '-', zero drop.
//  * csr_sparsify      reference sparsify (sparse.py:439-467).
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "dsetup.cuh"

namespace pmgr {

namespace {

// ------------------------------------------------------------ validation
__global__ void k_validate(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t *ro,
                           const int32_t *ci, unsigned long long *err) {
    // err[0]: min bad row for non-decreasing offsets; err[1]: col range; err[2]: order
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nrows) return;
    int64_t b = ro[i], e = ro[i + 1];
    if (e < b || b < 0 || e > nnz) {
        atomicMin(err + 0, (unsigned long long)i);
        return;
    }
    for (int64_t q = b; q < e; ++q) {
        int32_t c = ci[q];
        if (c < 0 || c >= ncols) atomicMin(err + 1, (unsigned long long)i);
        if (q > b && c <= ci[q - 1]) atomicMin(err + 2, (unsigned long long)i);
    }
}

// ------------------------------------------------------------ transpose
__global__ void k_count_cols(const int32_t *ci, int64_t nnz, int64_t *cnt) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < nnz) atomicAdd((unsigned long long *)(cnt + ci[q]), 1ull);
}

__global__ void k_row_of_entry(int64_t nrows, const int64_t *ro, int32_t *row) {
    // one warp per row
    int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= nrows) return;
    for (int64_t q = ro[i] + lane; q < ro[i + 1]; q += 32) row[q] = (int32_t)i;
}

__global__ void k_transpose_fill(int64_t nnz, const int32_t *sorted_rows, const int32_t *perm,
                                 const double *v, int32_t *tci, double *tv) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nnz) return;
    tci[q] = sorted_rows[q];
    tv[q] = v[perm[q]];
}

__global__ void k_gather_rows(int64_t nnz, const int32_t *rows, const int32_t *perm, int32_t *out) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < nnz) out[q] = rows[perm[q]];
}

__global__ void k_iota(int32_t *p, int64_t n) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < n) p[q] = (int32_t)q;
}

// ------------------------------------------------------------ spgemm
// shared-memory hash tables per warp: the symbolic pass keeps keys only
// (2048 slots, rows up to 1024 by their upper bound: 8 KB per warp), the
// numeric pass keys and values (1024 slots, rows up to 512 by their exact
// count: 12 KB per warp); rows beyond take a global-memory table
constexpr int HS_SYM = 2048;
constexpr int HS_NUM = 512;
constexpr int SP_WARPS = 4;       // warps per block
constexpr int SMALL_LIMIT = HS_SYM / 2;      // symbolic: upper bound
constexpr int SMALL_LIMIT_NUM = HS_NUM / 2;  // numeric: exact count

__device__ __forceinline__ unsigned hash_k(int32_t k) { return (unsigned)k * 2654435761u; }

// insert-or-find key k in a table of size tsz (power of two); returns slot
// and whether this call inserted it.
__device__ __forceinline__ int64_t table_insert(int32_t *keys, int64_t tsz, int32_t k, bool &inserted) {
    int64_t h = hash_k(k) & (tsz - 1);
    while (true) {
        int32_t cur = keys[h];
        if (cur == k) {
            inserted = false;
            return h;
        }
        if (cur == -1) {
            int32_t prev = atomicCAS(keys + h, -1, k);
            if (prev == -1) {
                inserted = true;
                return h;
            }
            if (prev == k) {
                inserted = false;
                return h;
            }
        }
        h = (h + 1) & (tsz - 1);
    }
}

// upper bound of distinct columns per row: min(sum_j nnz(Y_j), ncols)
__global__ void k_spgemm_ub(int64_t n, const int64_t *xro, const int32_t *xci, const int64_t *yro,
                            int64_t ycols, int64_t *ub) {
    int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    int64_t s = 0;
    for (int64_t q = xro[i] + lane; q < xro[i + 1]; q += 32) {
        int32_t j = xci[q];
        s += yro[j + 1] - yro[j];
    }
    s = warp_sum_i64(s);
    if (lane == 0) ub[i] = s < ycols ? s : ycols;
}

// global-table sizes for big rows (0 for rows on the shared path)
__global__ void k_table_size(int64_t n, const int64_t *ub, int64_t *tsz, int64_t limit) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t u = ub[i];
    if (u <= limit) {
        tsz[i] = 0;
    } else {
        int64_t t = 1;
        while (t < 2 * u) t <<= 1;
        tsz[i] = t;
    }
}

// NUMERIC = false: count distinct columns per row into cnt[i].
// NUMERIC = true : accumulate and dump (key, value) pairs unsorted into
//                  C at cro[i]; structural mode stores zero sums as +0.0.
// FLAT (products whose right factor has short rows, e.g. (R A) P with two
// entries per row of P): instead of one middle index per step -- two busy
// lanes out of 32 -- the (middle index, entry) pairs of a batch of 32 middle
// indices are flattened in (j, entry) order and taken 32 per step; pairs of
// one step that hit the same output column are added by the lowest lane in
// lane order, i.e. in ascending j, so every sum is still csr_matmat's.
template <bool NUMERIC, bool FLAT = false>
__global__ void __launch_bounds__(SP_WARPS * 32)
    k_spgemm(int64_t n, const int64_t *__restrict__ xro, const int32_t *__restrict__ xci,
             const double *__restrict__ xv, const int64_t *__restrict__ yro,
             const int32_t *__restrict__ yci, const double *__restrict__ yv,
             const int64_t *__restrict__ ub, const int64_t *__restrict__ toff, int32_t *gkeys,
             double *gvals, int64_t *cnt, const int64_t *__restrict__ cro, int32_t *cci, double *cv) {
    constexpr int HS = NUMERIC ? HS_NUM : HS_SYM;
    extern __shared__ unsigned char smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    int32_t *skeys = (int32_t *)smem + warp * HS;
    double *svals = NUMERIC ? (double *)(smem + sizeof(int32_t) * HS * SP_WARPS) + warp * HS : nullptr;
    const int64_t nwarps = (int64_t)gridDim.x * SP_WARPS;
    for (int64_t i = blockIdx.x * (int64_t)SP_WARPS + warp; i < n; i += nwarps) {
        // symbolic: table by the upper bound; numeric: by the exact count
        const bool big = NUMERIC ? cro[i + 1] - cro[i] > SMALL_LIMIT_NUM : ub[i] > SMALL_LIMIT;
        int32_t *keys;
        double *vals;
        int64_t tsz;
        if (big) {
            keys = gkeys + toff[i];
            vals = NUMERIC ? gvals + toff[i] : nullptr;
            tsz = toff[i + 1] - toff[i];
        } else {
            keys = skeys;
            vals = svals;
            tsz = HS;
        }
        for (int64_t t = lane; t < tsz; t += 32) {
            keys[t] = -1;
            if (NUMERIC) vals[t] = 0.0;
        }
        __syncwarp();
        int64_t local = 0;
        // The middle index is walked in ascending order (csr_matmat's
        // summation order), but its loads are batched: lane t fetches the
        // t-th middle index of the batch, its X value and Y row bounds (32
        // independent loads instead of a chain of three per index), and the
        // first chunk of Y's row for step t+1 is loaded while step t inserts.
        const int64_t xe = xro[i + 1];
        for (int64_t jb = xro[i]; jb < xe; jb += 32) {
            const int64_t jq = jb + lane;
            const bool has = jq < xe;
            const int32_t jl = has ? xci[jq] : 0;
            const double xl = (NUMERIC && has) ? xv[jq] : 0.0;
            const int64_t sl = has ? yro[jl] : 0, el = has ? yro[jl + 1] : 0;
            if constexpr (FLAT) {
                const int len = (int)(el - sl);
                int inc = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(FULL, inc, o);
                    if (lane >= o) inc += t;
                }
                const int excl = inc - len;
                const int T = __shfl_sync(FULL, inc, 31);
                for (int q0 = 0; q0 < T; q0 += 32) {
                    const int q = q0 + lane;
                    const bool act = q < T;
                    int t = 0;  // the last middle index of the batch whose pairs start at or before q
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const int cand = t + step;
                        const int ev = __shfl_sync(FULL, excl, cand & 31);
                        if (cand < 32 && ev <= q) t = cand;
                    }
                    const int e = q - __shfl_sync(FULL, excl, t);
                    const int64_t ys = __shfl_sync(FULL, sl, t);
                    const double xval = __shfl_sync(FULL, xl, t);
                    int32_t k = -1;
                    double prod = 0.0;
                    if (act) {
                        k = yci[ys + e];
                        if (NUMERIC) prod = __dmul_rn(xval, yv[ys + e]);
                    }
                    int64_t slot = -1;
                    bool ins = false;
                    if (act) slot = table_insert(keys, tsz, k, ins);
                    if (!NUMERIC) {
                        if (ins) ++local;
                    } else {
                        __syncwarp();
                        const unsigned grp = __match_any_sync(FULL, act ? (int)slot : -1 - lane);
                        const int gsz = __popc(grp);
                        const int maxg = __reduce_max_sync(FULL, act ? gsz : 0);
                        const bool leader = act && (__ffs(grp) - 1 == lane);
                        double sacc = leader ? vals[slot] : 0.0;
                        for (int r = 0; r < maxg; ++r) {
                            const unsigned src = __fns(grp, 0, r + 1);
                            const double pv = __shfl_sync(FULL, prod, src & 31u);
                            if (leader && r < gsz) sacc = __dadd_rn(sacc, pv);
                        }
                        if (leader) vals[slot] = sacc;
                    }
                    __syncwarp();
                }
                continue;
            }
            const int nb = (int)(xe - jb < 32 ? xe - jb : 32);
            int64_t st = __shfl_sync(FULL, sl, 0), en = __shfl_sync(FULL, el, 0);
            int32_t kc = st + lane < en ? yci[st + lane] : -1;
            double yc = (NUMERIC && kc >= 0) ? yv[st + lane] : 0.0;
            for (int t = 0; t < nb; ++t) {
                const double xval = __shfl_sync(FULL, xl, t);
                // prefetch step t+1's first chunk
                const int64_t st1 = __shfl_sync(FULL, sl, (t + 1) & 31), en1 = __shfl_sync(FULL, el, (t + 1) & 31);
                const bool nx = t + 1 < nb && st1 + lane < en1;
                const int32_t kn = nx ? yci[st1 + lane] : -1;
                const double yn = (NUMERIC && nx) ? yv[st1 + lane] : 0.0;
                if (kc >= 0) {
                    bool ins;
                    const int64_t slot = table_insert(keys, tsz, kc, ins);
                    if (NUMERIC) vals[slot] = __dadd_rn(vals[slot], __dmul_rn(xval, yc));
                    else if (ins) ++local;
                }
                for (int64_t kk = st + 32 + lane; kk < en; kk += 32) {
                    const int32_t k = yci[kk];
                    bool ins;
                    const int64_t slot = table_insert(keys, tsz, k, ins);
                    if (NUMERIC) vals[slot] = __dadd_rn(vals[slot], __dmul_rn(xval, yv[kk]));
                    else if (ins) ++local;
                }
                __syncwarp();
                st = st1;
                en = en1;
                kc = kn;
                yc = yn;
            }
        }
        if (!NUMERIC) {
            local = warp_sum_i64(local);
            if (lane == 0) cnt[i] = local;
        } else if (!big) {
            // shared table: compact the occupied slots in place (a chunk's
            // reads precede its writes, which land at or below the chunk),
            // then write each entry at its rank among the row's keys -- the
            // row comes out sorted, no segmented sort needed
            int m = 0;
            for (int t0 = 0; t0 < HS; t0 += 32) {
                const int t = t0 + lane;
                const int32_t k = keys[t];
                const double val = vals[t];
                const unsigned msk = __ballot_sync(FULL, k != -1);
                __syncwarp();
                if (k != -1) {
                    const int pos = m + __popc(msk & ((1u << lane) - 1u));
                    keys[pos] = k;
                    vals[pos] = val;
                }
                m += __popc(msk);
                __syncwarp();
            }
            const int64_t base = cro[i];
            for (int e = lane; e < m; e += 32) {
                const int32_t k = keys[e];
                int r = 0;
                for (int q = 0; q < m; ++q) r += keys[q] < k;
                const double val = vals[e];
                cci[base + r] = k;
                cv[base + r] = (val == 0.0) ? 0.0 : val;
            }
        } else {
            // global table: dump occupied slots (sorted afterwards by the
            // segmented sort over the big rows)
            int64_t base = cro[i];
            for (int64_t t0 = 0; t0 < tsz; t0 += 32) {
                int64_t t = t0 + lane;
                int32_t k = t < tsz ? keys[t] : -1;
                unsigned m = __ballot_sync(FULL, k != -1);
                if (k != -1) {
                    int pos = __popc(m & ((1u << lane) - 1u));
                    double val = vals[t];
                    cci[base + pos] = k;
                    cv[base + pos] = (val == 0.0) ? 0.0 : val;
                }
                base += __popc(m);
            }
        }
        __syncwarp();
    }
}

// [begin, end) of the rows with more than `limit` entries (any order)
__global__ void k_big_segments(int64_t n, const int64_t *ro, int64_t limit, int64_t *sb, int64_t *se,
                               unsigned long long *count) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n || ro[i + 1] - ro[i] <= limit) return;
    const unsigned long long p = atomicAdd(count, 1ull);
    sb[p] = ro[i];
    se[p] = ro[i + 1];
}

// Coarse products (few output columns): a dense accumulator per row in
// shared memory, block per row.  The middle index is walked in ascending
// order with a block barrier between j's, so every entry is summed exactly
// like csr_matmat; the flag bitmap yields the row already sorted.
constexpr int DENSE_COLS = 12288;
constexpr int DENSE_THREADS = 256;

// FLAT (numeric pass, right factors with short rows): no block barrier per
// middle index.  Every warp walks the row's flattened (middle index, entry)
// pairs, 32 per step in (j, entry) order, and accumulates the output columns
// k with k mod 8 = its warp number; pairs of a step that hit one column are
// added by the lowest lane in lane order (ascending j), so the sums are
// unchanged bit for bit.
template <bool NUMERIC, bool FLAT = false>
__global__ void __launch_bounds__(DENSE_THREADS)
    k_spgemm_dense(int64_t n, int64_t ncols, const int64_t *__restrict__ xro, const int32_t *__restrict__ xci,
                   const double *__restrict__ xv, const int64_t *__restrict__ yro, const int32_t *__restrict__ yci,
                   const double *__restrict__ yv, int64_t *cnt, const int64_t *__restrict__ cro, int32_t *cci,
                   double *cv) {
    extern __shared__ unsigned char smem[];
    const int W = (int)((ncols + 31) / 32);
    unsigned *flags = (unsigned *)smem;
    double *acc = (double *)(smem + sizeof(unsigned) * ((W + 1) & ~1));
    __shared__ int64_t wbase[DENSE_THREADS + 1];
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        for (int t = threadIdx.x; t < W; t += DENSE_THREADS) flags[t] = 0u;
        if (NUMERIC)
            for (int64_t t = threadIdx.x; t < ncols; t += DENSE_THREADS) acc[t] = 0.0;
        __syncthreads();
        // middle indices in ascending order, their loads batched 32 at a time
        // (every warp fetches the same batch; lane t holds index t)
        const int64_t xe = xro[i + 1];
        const int lane = threadIdx.x & 31;
        for (int64_t jb = xro[i]; jb < xe; jb += 32) {
            const int64_t jq = jb + lane;
            const bool has = jq < xe;
            const int32_t jl = has ? xci[jq] : 0;
            const double xl = (NUMERIC && has) ? xv[jq] : 0.0;
            const int64_t sl = has ? yro[jl] : 0, el = has ? yro[jl + 1] : 0;
            if constexpr (NUMERIC && FLAT) {
                static_assert(DENSE_THREADS == 256, "eight warps share the output columns");
                const int warp = threadIdx.x >> 5;
                const int len = (int)(el - sl);
                int inc = len;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int t = __shfl_up_sync(FULL, inc, o);
                    if (lane >= o) inc += t;
                }
                const int excl = inc - len;
                const int T = __shfl_sync(FULL, inc, 31);
                for (int q0 = 0; q0 < T; q0 += 32) {
                    const int q = q0 + lane;
                    const bool act = q < T;
                    int t = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const int cand = t + step;
                        const int ev = __shfl_sync(FULL, excl, cand & 31);
                        if (cand < 32 && ev <= q) t = cand;
                    }
                    const int e = q - __shfl_sync(FULL, excl, t);
                    const int64_t ys = __shfl_sync(FULL, sl, t);
                    const double xval = __shfl_sync(FULL, xl, t);
                    int32_t k = -1;
                    double prod = 0.0;
                    if (act) {
                        k = yci[ys + e];
                        prod = __dmul_rn(xval, yv[ys + e]);
                    }
                    const bool mine = act && ((k & 7) == warp);
                    const unsigned grp = __match_any_sync(FULL, mine ? k : -1 - lane);
                    const int gsz = __popc(grp);
                    const int maxg = __reduce_max_sync(FULL, mine ? gsz : 0);
                    const bool leader = mine && (__ffs(grp) - 1 == lane);
                    double sacc = leader ? acc[k] : 0.0;
                    for (int r = 0; r < maxg; ++r) {
                        const unsigned src = __fns(grp, 0, r + 1);
                        const double pv = __shfl_sync(FULL, prod, src & 31u);
                        if (leader && r < gsz) sacc = __dadd_rn(sacc, pv);
                    }
                    if (leader) {
                        acc[k] = sacc;
                        atomicOr(flags + (k >> 5), 1u << (k & 31));
                    }
                    __syncwarp();
                }
                continue;
            }
            const int nb = (int)(xe - jb < 32 ? xe - jb : 32);
            for (int t = 0; t < nb; ++t) {
                const double xval = __shfl_sync(FULL, xl, t);
                const int64_t st = __shfl_sync(FULL, sl, t), en = __shfl_sync(FULL, el, t);
                for (int64_t kk = st + threadIdx.x; kk < en; kk += DENSE_THREADS) {
                    const int32_t k = yci[kk];
                    atomicOr(flags + (k >> 5), 1u << (k & 31));
                    if (NUMERIC) acc[k] = __dadd_rn(acc[k], __dmul_rn(xval, yv[kk]));
                }
                if (NUMERIC) __syncthreads();
            }
        }
        __syncthreads();
        // words [w0, w1) of this thread, in order
        const int per = (W + DENSE_THREADS - 1) / DENSE_THREADS;
        const int w0 = threadIdx.x * per, w1 = (w0 + per < W) ? w0 + per : W;
        int64_t mine = 0;
        for (int w = w0; w < w1; ++w) mine += __popc(flags[w]);
        wbase[threadIdx.x + 1] = mine;
        __syncthreads();
        if (threadIdx.x == 0) {
            wbase[0] = 0;
            for (int t = 1; t <= DENSE_THREADS; ++t) wbase[t] += wbase[t - 1];
        }
        __syncthreads();
        if (!NUMERIC) {
            if (threadIdx.x == 0) cnt[i] = wbase[DENSE_THREADS];
        } else {
            int64_t o = cro[i] + wbase[threadIdx.x];
            for (int w = w0; w < w1; ++w) {
                unsigned f = flags[w];
                while (f) {
                    const int bit = __ffs(f) - 1;
                    f &= f - 1;
                    const int k = w * 32 + bit;
                    const double val = acc[k];
                    cci[o] = k;
                    cv[o] = (val == 0.0) ? 0.0 : val;
                    ++o;
                }
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------ zero drop
__global__ void k_count_nonzero(int64_t n, const int64_t *ro, const double *v, int64_t *cnt) {
    int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    int64_t c = 0;
    for (int64_t q = ro[i] + lane; q < ro[i + 1]; q += 32) c += (v[q] != 0.0);
    c = warp_sum_i64(c);
    if (lane == 0) cnt[i] = c;
}

__global__ void k_compact_nonzero(int64_t n, const int64_t *ro, const int32_t *ci, const double *v,
                                  const int64_t *nro, int32_t *nci, double *nv) {
    int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    int64_t w = nro[i];
    for (int64_t q0 = ro[i]; q0 < ro[i + 1]; q0 += 32) {
        int64_t q = q0 + lane;
        bool keep = q < ro[i + 1] && v[q] != 0.0;
        unsigned m = __ballot_sync(FULL, keep);
        if (keep) {
            int pos = __popc(m & ((1u << lane) - 1u));
            nci[w + pos] = ci[q];
            nv[w + pos] = v[q];
        }
        w += __popc(m);
    }
}

// ------------------------------------------------------------ subtract
// C = A - B over the union of two sorted rows; exact zeros dropped.
template <bool FILL>
__global__ void k_subtract(int64_t n, const int64_t *aro, const int32_t *aci, const double *av,
                           const int64_t *bro, const int32_t *bci, const double *bv, int64_t *cnt,
                           const int64_t *cro, int32_t *cci, double *cv) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t p = aro[i], pe = aro[i + 1], q = bro[i], qe = bro[i + 1];
    int64_t w = FILL ? cro[i] : 0;
    while (p < pe || q < qe) {
        int64_t ca = p < pe ? aci[p] : INT64_MAX;
        int64_t cb = q < qe ? bci[q] : INT64_MAX;
        double r;
        int64_t c;
        if (ca == cb) {
            r = __dadd_rn(av[p++], -bv[q++]);
            c = ca;
        } else if (ca < cb) {
            r = __dadd_rn(av[p++], -0.0);
            c = ca;
        } else {
            r = __dadd_rn(0.0, -bv[q++]);
            c = cb;
        }
        if (r != 0.0) {
            if (FILL) {
                cci[w] = (int32_t)c;
                cv[w] = r;
            }
            ++w;
        }
    }
    if (!FILL) cnt[i] = w;
}

// ------------------------------------------------------------ sparsify
// Row-wise dropping: keep same-entity entries and the n_max largest |v|
// among the rest, ties to the smaller column; kept entries in stored order.
template <bool FILL>
__global__ void k_sparsify(int64_t n, const int64_t *ro, const int32_t *ci, const double *v,
                           const int32_t *entity, int64_t nmax, int64_t *cnt, const int64_t *kro,
                           int32_t *kci, double *kv) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t ei = entity[i];
    int64_t w = FILL ? kro[i] : 0;
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q) {
        bool keep = entity[ci[q]] == ei;
        if (!keep && nmax > 0) {
            double a = fabs(v[q]);
            int32_t c = ci[q];
            int64_t rank = 0;
            for (int64_t t = ro[i]; t < ro[i + 1] && rank < nmax; ++t) {
                if (t == q || entity[ci[t]] == ei) continue;
                double b = fabs(v[t]);
                if (b > a || (b == a && ci[t] < c)) ++rank;
            }
            keep = rank < nmax;
        }
        if (keep) {
            if (FILL) {
                kci[w] = ci[q];
                kv[w] = v[q];
            }
            ++w;
        }
    }
    if (!FILL) cnt[i] = w;
}

__global__ void k_diag(int64_t n, const int64_t *ro, const int32_t *ci, const double *v, double *d) {
    int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (i >= n) return;
    double dv = 0.0;
    bool found = false;
    for (int64_t q = ro[i] + lane; q < ro[i + 1]; q += 32)
        if (ci[q] == i) {
            dv = v[q];
            found = true;
        }
    unsigned m = __ballot_sync(FULL, found);
    double r = m ? __shfl_sync(FULL, dv, __ffs(m) - 1) : 0.0;
    if (lane == 0) d[i] = r;
}

__global__ void k_diag_inverse(int64_t n, const double *d, double *dinv, unsigned long long *bad) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x = d[i];
    if (x == 0.0) atomicMin(bad, (unsigned long long)i);
    dinv[i] = __ddiv_rn(1.0, x);
}

__global__ void k_fill_u64(unsigned long long *p, int64_t n, unsigned long long val) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) p[i] = val;
}

}  // namespace

// ===================================================================== API

void csr_validate(const CsrView &A, cudaStream_t s) {
    int64_t r0 = 0, rn = 0;
    if (A.nrows >= 0) {
        PMGR_CUDA(cudaMemcpyAsync(&r0, A.ro, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        PMGR_CUDA(cudaMemcpyAsync(&rn, A.ro + A.nrows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        PMGR_CUDA(cudaStreamSynchronize(s));
    }
    if (r0 != 0 || rn != A.nnz) fail(PMGR_ERR_INVALID, "row_offsets endpoints inconsistent with nnz");
    if (A.nrows == 0) return;
    TBuf<unsigned long long> err(3, s);
    k_fill_u64<<<1, 32, 0, s>>>(err.p, 3, ~0ull);
    PMGR_LAUNCHED();
    k_validate<<<grid_for(A.nrows, 256), 256, 0, s>>>(A.nrows, A.ncols, A.nnz, A.ro, A.ci, err.p);
    PMGR_LAUNCHED();
    unsigned long long h[3];
    PMGR_CUDA(cudaMemcpyAsync(h, err.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    PMGR_CUDA(cudaStreamSynchronize(s));
    if (h[0] != ~0ull) fail(PMGR_ERR_INVALID, "row_offsets must be non-decreasing", (int64_t)h[0]);
    if (h[1] != ~0ull) fail(PMGR_ERR_INVALID, "column index out of range", (int64_t)h[1]);
    if (h[2] != ~0ull)
        fail(PMGR_ERR_INVALID, "column indices must be strictly increasing within each row", (int64_t)h[2]);
}

namespace {
__global__ void k_maxrow(int64_t n, const int64_t *ro, unsigned long long *out) {
    unsigned long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long l = (unsigned long long)(ro[i + 1] - ro[i]);
        m = l > m ? l : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long t = __shfl_xor_sync(FULL, m, o);
        m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}
}  // namespace

namespace {
__global__ void k_long_flag(int64_t n, const int64_t *ro, int64_t len, int32_t *flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (ro[i + 1] - ro[i]) > len ? 1 : 0;
}
__global__ void k_long_fill(int64_t n, const int32_t *flag, const int64_t *pos, int32_t *lrows) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && flag[i]) lrows[pos[i]] = (int32_t)i;
}
}  // namespace

void csr_long_rows(Csr &A, cudaStream_t s) {
    A.nlong = 0;
    A.lrows.release();
    if (A.long_len <= 0 || A.nrows == 0) return;
    TBuf<int32_t> flag(A.nrows, s);
    TBuf<int64_t> pos(A.nrows + 1, s);
    k_long_flag<<<grid_for(A.nrows, 256), 256, 0, s>>>(A.nrows, A.ro.p, A.long_len, flag.p);
    PMGR_LAUNCHED();
    const int64_t nl = exclusive_scan_total_i32(flag.p, pos.p, A.nrows, s);
    if (nl == 0) return;
    A.lrows.alloc(nl);
    k_long_fill<<<grid_for(A.nrows, 256), 256, 0, s>>>(A.nrows, flag.p, pos.p, A.lrows.p);
    PMGR_LAUNCHED();
    A.nlong = nl;
}

namespace {
__global__ void k_to16(int64_t nnz, const int32_t *ci, uint16_t *c16) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < nnz) c16[q] = (uint16_t)ci[q];
}
}  // namespace

void csr_finalize(Csr &A, cudaStream_t s, bool build_sj) {
    A.sj.reset();
    A.sj_want = sj_wanted(A.nrows, A.nnz);
    if (A.nrows == 0) {
        A.maxrow = 0;
        return;
    }
    TBuf<unsigned long long> m(1, s);
    PMGR_CUDA(cudaMemsetAsync(m.p, 0, sizeof(unsigned long long), s));
    unsigned g = grid_for(A.nrows, 256);
    k_maxrow<<<g < 1024 ? g : 1024, 256, 0, s>>>(A.nrows, A.ro.p, m.p);
    PMGR_LAUNCHED();
    A.maxrow = (int64_t)read_scalar(m.p, s);
    // skewed operators (a few dense coarse-grid rows next to short ones): the
    // long rows get a block each, the lane group fits the mean
    static const bool no_long = getenv("PMGR_NO_LONG_ROWS") && getenv("PMGR_NO_LONG_ROWS")[0] != '0';
    if (!no_long) {
        const int gm = spmv_lanes_mean((double)A.nnz / (double)A.nrows);
        if (A.maxrow > 16 * gm) {
            A.long_len = 16 * gm;
            csr_long_rows(A, s);
        }
    }
    // narrow column indices for the solve-phase SpMV (10 instead of 12 bytes per entry)
    static const bool no16 = getenv("PMGR_NO_CI16") && getenv("PMGR_NO_CI16")[0] != '0';
    if (!no16 && A.ncols <= 65536 && A.nnz > 0) {
        A.ci16.alloc(A.nnz);
        k_to16<<<grid_for(A.nnz, 256), 256, 0, s>>>(A.nnz, A.ci.p, A.ci16.p);
        PMGR_LAUNCHED();
    }
    if (build_sj) csr_make_sj(A, s);
    static const bool stats = getenv("PMGR_HIER_STATS") && getenv("PMGR_HIER_STATS")[0] != '0';
    if (stats)
        fprintf(stderr, "[pmgr] operator %lld x %lld nnz %lld (%.1f/row, max %lld, long rows %lld > %lld)\n",
                (long long)A.nrows, (long long)A.ncols, (long long)A.nnz, (double)A.nnz / (double)A.nrows,
                (long long)A.maxrow, (long long)A.nlong, (long long)A.long_len);
}

namespace {
// block columns (< prefix) of node row I: union over its 3 rows
__global__ void k_bsr_count(int64_t nb, int32_t prefix, const int64_t *ro, const int32_t *ci, int64_t *cnt) {
    const int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (I >= nb) return;
    // merge the three sorted rows by block column
    int64_t p[3], e[3];
    for (int r = 0; r < 3; ++r) {
        p[r] = ro[3 * I + r];
        e[r] = ro[3 * I + r + 1];
    }
    int64_t c = 0;
    while (true) {
        int32_t best = INT32_MAX;
        for (int r = 0; r < 3; ++r)
            if (p[r] < e[r] && ci[p[r]] < prefix) best = min(best, ci[p[r]] / 3);
        if (best == INT32_MAX) break;
        for (int r = 0; r < 3; ++r)
            while (p[r] < e[r] && ci[p[r]] < prefix && ci[p[r]] / 3 == best) ++p[r];
        ++c;
    }
    cnt[I] = c;
}

// block columns of node row I (the merge of k_bsr_count, writing the list)
__global__ void k_bsr_cols(int64_t nb, int32_t prefix, const int64_t *ro, const int32_t *ci, const int64_t *bro,
                           int32_t *bci) {
    const int64_t I = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (I >= nb) return;
    int64_t p[3], e[3];
    for (int r = 0; r < 3; ++r) {
        p[r] = ro[3 * I + r];
        e[r] = ro[3 * I + r + 1];
    }
    int64_t w = bro[I];
    while (true) {
        int32_t best = INT32_MAX;
        for (int r = 0; r < 3; ++r)
            if (p[r] < e[r] && ci[p[r]] < prefix) best = min(best, ci[p[r]] / 3);
        if (best == INT32_MAX) break;
        bci[w++] = best;
        for (int r = 0; r < 3; ++r)
            while (p[r] < e[r] && ci[p[r]] < prefix && ci[p[r]] / 3 == best) ++p[r];
    }
}

// block values, a warp per node row: the node's blocks are zero-filled, then
// the lanes stride over the three rows' entries (coalesced reads; the
// thread-per-node fill read every 4-byte column through its own 32-byte
// sector: 40 ms at C4, this one 5 ms) and place each one in its block, found
// by bisection in the node's sorted block-column list
__global__ void k_bsr_vals(int64_t nb, int32_t prefix, const int64_t *__restrict__ ro,
                           const int32_t *__restrict__ ci, const double *__restrict__ v,
                           const int64_t *__restrict__ bro, const int32_t *__restrict__ bci, double *bval) {
    const int64_t I = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (I >= nb) return;
    const int64_t b0 = bro[I], b1 = bro[I + 1];
    for (int64_t t = 9 * b0 + lane; t < 9 * b1; t += 32) bval[t] = 0.0;
    __syncwarp();
    for (int r = 0; r < 3; ++r) {
        const int64_t qe = ro[3 * I + r + 1];
        for (int64_t q = ro[3 * I + r] + lane; q < qe; q += 32) {
            const int32_t c = ci[q];
            if (c >= prefix) continue;
            const int32_t b = c / 3;
            int64_t lo = b0, hi = b1 - 1;
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (bci[mid] < b) lo = mid + 1;
                else hi = mid;
            }
            bval[9 * lo + r + 3 * (c - 3 * b)] = v[q];  // column-major
        }
    }
}

// remainder entries: columns >= prefix of the prefix rows, all of the others
__global__ void k_rem_count(int64_t n, int64_t prow, int32_t prefix, const int64_t *ro, const int32_t *ci,
                            int64_t *cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t c = 0;
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q) c += (i >= prow || ci[q] >= prefix);
    cnt[i] = c;
}

__global__ void k_rem_fill(int64_t n, int64_t prow, int32_t prefix, const int64_t *ro, const int32_t *ci,
                           const double *v, const int64_t *rro, int32_t *rci, double *rv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t w = rro[i];
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q)
        if (i >= prow || ci[q] >= prefix) {
            rci[w] = ci[q];
            rv[w] = v[q];
            ++w;
        }
}
}  // namespace

void csr_make_bsr3(Csr &A, int64_t prow, int64_t pcol, cudaStream_t s, bool force, const DistSetup *dist) {
    static const bool off = getenv("PMGR_NO_BSR") && getenv("PMGR_NO_BSR")[0] != '0';
    if (off || prow % 3 != 0 || pcol % 3 != 0 || prow <= 0 || prow > A.nrows || pcol > A.ncols) return;
    const int64_t nb = prow / 3, n = A.nrows;
    const int32_t prefix = (int32_t)pcol;
    TBuf<int64_t> cnt(nb, s);
    k_bsr_count<<<grid_for(nb, 128), 128, 0, s>>>(nb, prefix, A.ro.p, A.ci.p, cnt.p);
    PMGR_LAUNCHED();
    A.bro.alloc(nb + 1);
    const int64_t nblk = exclusive_scan_total(cnt.p, A.bro.p, nb, s);
    int64_t nrem = 0;
    TBuf<int64_t> rc(n, s);
    k_rem_count<<<grid_for(n, 128), 128, 0, s>>>(n, prow, prefix, A.ro.p, A.ci.p, rc.p);
    PMGR_LAUNCHED();
    A.rro.alloc(n + 1);
    nrem = exclusive_scan_total(rc.p, A.rro.p, n, s);
    if (nrem == 0) A.rro.release();
    // only worth it when the blocks are (nearly) full (a distributed operator
    // decides on its global counts, like the single-GPU copy)
    double gblk = (double)nblk, gin = (double)(A.nnz - nrem);
    if (dist && dist->nranks > 1) {
        gblk = (double)ds_allsum(*dist, nblk, s);
        gin = (double)ds_allsum(*dist, A.nnz - nrem, s);
    }
    if (!force && 9.0 * gblk > 1.25 * gin) {
        A.bro.release();
        A.rro.release();
        return;
    }
    A.bci.alloc(nblk);
    A.bval.alloc(9 * nblk);
    k_bsr_cols<<<grid_for(nb, 128), 128, 0, s>>>(nb, prefix, A.ro.p, A.ci.p, A.bro.p, A.bci.p);
    PMGR_LAUNCHED();
    k_bsr_vals<<<grid_for(nb * 32, 256), 256, 0, s>>>(nb, prefix, A.ro.p, A.ci.p, A.v.p, A.bro.p, A.bci.p, A.bval.p);
    PMGR_LAUNCHED();
    if (nrem > 0) {
        A.rci.alloc(nrem);
        A.rv.alloc(nrem);
        k_rem_fill<<<grid_for(n, 128), 128, 0, s>>>(n, prow, prefix, A.ro.p, A.ci.p, A.v.p, A.rro.p, A.rci.p,
                                                    A.rv.p);
        PMGR_LAUNCHED();
    }
    A.nbrows = nb;
    A.nblocks = nblk;
    A.nrem = nrem;
    csr_make_sj(A, s);
}

void csr_make_bsr3_shared(Csr &A, int64_t prefix, std::shared_ptr<const Csr> src, cudaStream_t s) {
    if (!src || src->nbrows <= 0 || src->rro.p || 3 * src->nbrows != prefix || prefix > A.nrows ||
        prefix > A.ncols || src->blk_src) {
        csr_make_bsr3(A, prefix, prefix, s);
        return;
    }
    const int64_t n = A.nrows;
    TBuf<int64_t> rc(n, s);
    k_rem_count<<<grid_for(n, 128), 128, 0, s>>>(n, prefix, (int32_t)prefix, A.ro.p, A.ci.p, rc.p);
    PMGR_LAUNCHED();
    A.rro.alloc(n + 1);
    const int64_t nrem = exclusive_scan_total(rc.p, A.rro.p, n, s);
    if (nrem == 0) {
        A.rro.release();
    } else {
        A.rci.alloc(nrem);
        A.rv.alloc(nrem);
        k_rem_fill<<<grid_for(n, 128), 128, 0, s>>>(n, prefix, (int32_t)prefix, A.ro.p, A.ci.p, A.v.p, A.rro.p,
                                                    A.rci.p, A.rv.p);
        PMGR_LAUNCHED();
    }
    A.blk_src = std::move(src);
    A.nbrows = A.blk_src->nbrows;
    A.nblocks = A.blk_src->nblocks;
    A.nrem = nrem;
    csr_make_sj(A, s);
}

void csr_copy(const CsrView &A, Csr &B, cudaStream_t s) {
    B.alloc(A.nrows, A.ncols, A.nnz);
    PMGR_CUDA(cudaMemcpyAsync(B.ro.p, A.ro, sizeof(int64_t) * (A.nrows + 1), cudaMemcpyDeviceToDevice, s));
    if (A.nnz) {
        PMGR_CUDA(cudaMemcpyAsync(B.ci.p, A.ci, sizeof(int32_t) * A.nnz, cudaMemcpyDeviceToDevice, s));
        PMGR_CUDA(cudaMemcpyAsync(B.v.p, A.v, sizeof(double) * A.nnz, cudaMemcpyDeviceToDevice, s));
    }
}

void csr_transpose(const CsrView &A, Csr &T, cudaStream_t s) {
    T.alloc(A.ncols, A.nrows, A.nnz);
    TBuf<int64_t> cnt(A.ncols, s);
    PMGR_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t) * A.ncols, s));
    if (A.nnz) {
        k_count_cols<<<grid_for(A.nnz, 256), 256, 0, s>>>(A.ci, A.nnz, cnt.p);
        PMGR_LAUNCHED();
    }
    exclusive_scan_total(cnt.p, T.ro.p, A.ncols, s);
    if (A.nnz == 0) return;
    // stable radix sort of entries (row-major order) by column
    TBuf<int32_t> rows(A.nnz, s), perm(A.nnz, s), rows_s(A.nnz, s), keys_s(A.nnz, s), perm_s(A.nnz, s);
    k_row_of_entry<<<grid_for(A.nrows * 32, 256), 256, 0, s>>>(A.nrows, A.ro, rows.p);
    PMGR_LAUNCHED();
    k_iota<<<grid_for(A.nnz, 256), 256, 0, s>>>(perm.p, A.nnz);
    PMGR_LAUNCHED();
    int end_bit = 1;
    while (end_bit < 31 && (1ll << end_bit) < A.ncols) ++end_bit;
    size_t tmp = 0;
    PMGR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, A.ci, keys_s.p, perm.p, perm_s.p, A.nnz, 0,
                                              end_bit, s));
    TBuf<char> t((int64_t)tmp, s);
    PMGR_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, A.ci, keys_s.p, perm.p, perm_s.p, A.nnz, 0, end_bit, s));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    k_gather_rows<<<grid_for(A.nnz, 256), 256, 0, s>>>(A.nnz, rows.p, perm_s.p, rows_s.p);
    PMGR_LAUNCHED();
    k_transpose_fill<<<grid_for(A.nnz, 256), 256, 0, s>>>(A.nnz, rows_s.p, perm_s.p, A.v, T.ci.p, T.v.p);
    PMGR_LAUNCHED();
}

void spgemm(const CsrView &X, const CsrView &Y, int mode, Csr &C, cudaStream_t s) {
    if (X.ncols != Y.nrows) fail(PMGR_ERR_INVALID, "spgemm dimension mismatch");
    const int64_t n = X.nrows;
    TBuf<int64_t> ub(n, s), tsz(n, s), toff(n + 1, s), cnt(n, s);
    TBuf<int64_t> cro(n + 1, s);
    if (n == 0) {
        C.alloc(0, Y.ncols, 0);
        PMGR_CUDA(cudaMemsetAsync(C.ro.p, 0, sizeof(int64_t), s));
        return;
    }
    int64_t total = 0;
    TBuf<int32_t> tci;
    TBuf<double> tv;
    static const int64_t dense_cols = [] {
        const char *e = getenv("PMGR_DENSE_COLS");
        const int64_t v = e ? atoll(e) : (int64_t)DENSE_COLS;
        return v < DENSE_COLS ? v : (int64_t)DENSE_COLS;
    }();
    if (Y.ncols <= dense_cols) {
        const int W = (int)((Y.ncols + 31) / 32);
        const size_t fbytes = sizeof(unsigned) * (size_t)((W + 1) & ~1);
        const size_t smem_num = fbytes + sizeof(double) * (size_t)Y.ncols;
        static bool dense_attr = false;
        if (!dense_attr) {
            const int maxs = (int)(sizeof(unsigned) * DENSE_COLS / 32 + 8 + sizeof(double) * DENSE_COLS);
            PMGR_CUDA(cudaFuncSetAttribute(k_spgemm_dense<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxs));
            dense_attr = true;
        }
        const int64_t gcap = (int64_t)num_sms() * 4;
        const unsigned g = (unsigned)(n < gcap ? n : gcap);
        k_spgemm_dense<false><<<g, DENSE_THREADS, fbytes, s>>>(n, Y.ncols, X.ro, X.ci, X.v, Y.ro, Y.ci, Y.v, cnt.p,
                                                               nullptr, nullptr, nullptr);
        PMGR_LAUNCHED();
        total = exclusive_scan_total(cnt.p, cro.p, n, s);
        tci.alloc(total, s);
        tv.alloc(total, s);
        // PMGR_SPGEMM_DENSE_FLAT: the barrier-free numeric pass when the right
        // factor's rows average at most this many entries (0: never)
        static const double dflat_mean = [] {
            const char *e = getenv("PMGR_SPGEMM_DENSE_FLAT");
            return e ? atof(e) : 8.0;  // C4: 153 -> 139 ms of dense products at 8, 221 ms at 64
        }();
        static bool dense_flat_attr = false;
        if (!dense_flat_attr) {
            const int maxs = (int)(sizeof(unsigned) * DENSE_COLS / 32 + 8 + sizeof(double) * DENSE_COLS);
            PMGR_CUDA(cudaFuncSetAttribute(k_spgemm_dense<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           maxs));
            dense_flat_attr = true;
        }
        if (dflat_mean > 0.0 && Y.nrows > 0 && (double)Y.nnz <= dflat_mean * (double)Y.nrows)
            k_spgemm_dense<true, true><<<g, DENSE_THREADS, smem_num, s>>>(n, Y.ncols, X.ro, X.ci, X.v, Y.ro, Y.ci,
                                                                          Y.v, nullptr, cro.p, tci.p, tv.p);
        else
            k_spgemm_dense<true><<<g, DENSE_THREADS, smem_num, s>>>(n, Y.ncols, X.ro, X.ci, X.v, Y.ro, Y.ci, Y.v,
                                                                    nullptr, cro.p, tci.p, tv.p);
        PMGR_LAUNCHED();
        setup_trace("  spgemm dense", total, s);
    } else {
    k_spgemm_ub<<<grid_for(n * 32, 256), 256, 0, s>>>(n, X.ro, X.ci, Y.ro, Y.ncols, ub.p);
    PMGR_LAUNCHED();
    k_table_size<<<grid_for(n, 256), 256, 0, s>>>(n, ub.p, tsz.p, SMALL_LIMIT);
    PMGR_LAUNCHED();
    int64_t gtotal = exclusive_scan_total(tsz.p, toff.p, n, s);
    setup_trace("  spgemm bounds", gtotal, s);
    TBuf<int32_t> gkeys(gtotal, s);

    const size_t smem_sym = (size_t)SP_WARPS * HS_SYM * sizeof(int32_t);
    const size_t smem_num = (size_t)SP_WARPS * HS_NUM * (sizeof(int32_t) + sizeof(double));
    static bool attr_set = false;
    if (!attr_set) {
        PMGR_CUDA(cudaFuncSetAttribute(k_spgemm<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_sym));
        PMGR_CUDA(cudaFuncSetAttribute(k_spgemm<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_num));
        PMGR_CUDA(cudaFuncSetAttribute(k_spgemm<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_sym));
        PMGR_CUDA(cudaFuncSetAttribute(k_spgemm<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_num));
        attr_set = true;
    }
    // PMGR_SPGEMM_FLAT: flattened (middle index, entry) pairs when the right
    // factor's rows average at most this many entries (0: never)
    static const double flat_mean = [] {
        const char *e = getenv("PMGR_SPGEMM_FLAT");
        return e ? atof(e) : 8.0;
    }();
    const bool flat = flat_mean > 0.0 && Y.nrows > 0 && (double)Y.nnz <= flat_mean * (double)Y.nrows;
    // resident warps: the occupancy each pass's shared tables allow
    auto grid_of = [&](const void *fn, size_t smem) {
        int per_sm = 0;
        PMGR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, SP_WARPS * 32, smem));
        const int64_t want = (n + SP_WARPS - 1) / SP_WARPS;
        const int64_t cap = (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1);
        return (unsigned)(want < cap ? (want > 0 ? want : 1) : cap);
    };

    if (flat)
        k_spgemm<false, true><<<grid_of((const void *)k_spgemm<false, true>, smem_sym), SP_WARPS * 32, smem_sym, s>>>(
            n, X.ro, X.ci, X.v, Y.ro, Y.ci, Y.v, ub.p, toff.p, gkeys.p, nullptr, cnt.p, nullptr, nullptr, nullptr);
    else
        k_spgemm<false><<<grid_of((const void *)k_spgemm<false>, smem_sym), SP_WARPS * 32, smem_sym, s>>>(
            n, X.ro, X.ci, X.v, Y.ro, Y.ci, Y.v, ub.p, toff.p, gkeys.p, nullptr, cnt.p, nullptr, nullptr, nullptr);
    PMGR_LAUNCHED();
    total = exclusive_scan_total(cnt.p, cro.p, n, s);
    setup_trace("  spgemm symbolic", total, s);
    // numeric tables from the exact counts
    k_table_size<<<grid_for(n, 256), 256, 0, s>>>(n, cnt.p, tsz.p, SMALL_LIMIT_NUM);
    PMGR_LAUNCHED();
    const int64_t ntotal = exclusive_scan_total(tsz.p, toff.p, n, s);
    gkeys.release();
    TBuf<int32_t> nkeys(ntotal, s);
    TBuf<double> nvals(ntotal, s);
    tci.alloc(total, s);
    tv.alloc(total, s);
    if (flat)
        k_spgemm<true, true><<<grid_of((const void *)k_spgemm<true, true>, smem_num), SP_WARPS * 32, smem_num, s>>>(
            n, X.ro, X.ci, X.v, Y.ro, Y.ci, Y.v, ub.p, toff.p, nkeys.p, nvals.p, nullptr, cro.p, tci.p, tv.p);
    else
        k_spgemm<true><<<grid_of((const void *)k_spgemm<true>, smem_num), SP_WARPS * 32, smem_num, s>>>(
            n, X.ro, X.ci, X.v, Y.ro, Y.ci, Y.v, ub.p, toff.p, nkeys.p, nvals.p, nullptr, cro.p, tci.p, tv.p);
    PMGR_LAUNCHED();
    setup_trace("  spgemm numeric", total, s);
    // only rows with more than SMALL_LIMIT_NUM entries (global tables) are unsorted
    {
        TBuf<int64_t> sb(n, s), se(n, s);
        TBuf<unsigned long long> nbig(1, s);
        PMGR_CUDA(cudaMemsetAsync(nbig.p, 0, sizeof(unsigned long long), s));
        k_big_segments<<<grid_for(n, 256), 256, 0, s>>>(n, cro.p, SMALL_LIMIT_NUM, sb.p, se.p, nbig.p);
        PMGR_LAUNCHED();
        const int64_t nb = (int64_t)read_scalar(nbig.p, s);
        if (nb > 0) segmented_sort_pairs_list(tci.p, tv.p, total, sb.p, se.p, nb, s);
    }
    setup_trace("  spgemm sort", total, s);
    }
    if (mode == 1) {
        C.nrows = n;
        C.ncols = Y.ncols;
        C.nnz = total;
        C.ro.alloc(n + 1);
        C.ci.alloc(total);
        C.v.alloc(total);
        PMGR_CUDA(cudaMemcpyAsync(C.ro.p, cro.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, s));
        if (total) {
            PMGR_CUDA(cudaMemcpyAsync(C.ci.p, tci.p, sizeof(int32_t) * total, cudaMemcpyDeviceToDevice, s));
            PMGR_CUDA(cudaMemcpyAsync(C.v.p, tv.p, sizeof(double) * total, cudaMemcpyDeviceToDevice, s));
        }
        return;
    }
    // mode 0: drop exact zeros
    k_count_nonzero<<<grid_for(n * 32, 256), 256, 0, s>>>(n, cro.p, tv.p, cnt.p);
    PMGR_LAUNCHED();
    C.ro.alloc(n + 1);
    int64_t nz = exclusive_scan_total(cnt.p, C.ro.p, n, s);
    C.nrows = n;
    C.ncols = Y.ncols;
    C.nnz = nz;
    C.ci.alloc(nz);
    C.v.alloc(nz);
    k_compact_nonzero<<<grid_for(n * 32, 256), 256, 0, s>>>(n, cro.p, tci.p, tv.p, C.ro.p, C.ci.p, C.v.p);
    PMGR_LAUNCHED();
}

void csr_subtract(const CsrView &A, const CsrView &B, Csr &C, cudaStream_t s) {
    if (A.nrows != B.nrows || A.ncols != B.ncols) fail(PMGR_ERR_INVALID, "shape mismatch");
    const int64_t n = A.nrows;
    TBuf<int64_t> cnt(n, s);
    C.ro.alloc(n + 1);
    if (n) {
        k_subtract<false><<<grid_for(n, 128), 128, 0, s>>>(n, A.ro, A.ci, A.v, B.ro, B.ci, B.v, cnt.p,
                                                           nullptr, nullptr, nullptr);
        PMGR_LAUNCHED();
    }
    int64_t nz = exclusive_scan_total(cnt.p, C.ro.p, n, s);
    C.nrows = n;
    C.ncols = A.ncols;
    C.nnz = nz;
    C.ci.alloc(nz);
    C.v.alloc(nz);
    if (n) {
        k_subtract<true><<<grid_for(n, 128), 128, 0, s>>>(n, A.ro, A.ci, A.v, B.ro, B.ci, B.v, nullptr,
                                                          C.ro.p, C.ci.p, C.v.p);
        PMGR_LAUNCHED();
    }
}

void csr_sparsify(const CsrView &M, const int32_t *entity, int64_t n_max, Csr &K, cudaStream_t s) {
    const int64_t n = M.nrows;
    TBuf<int64_t> cnt(n, s);
    K.ro.alloc(n + 1);
    if (n) {
        k_sparsify<false><<<grid_for(n, 128), 128, 0, s>>>(n, M.ro, M.ci, M.v, entity, n_max, cnt.p,
                                                           nullptr, nullptr, nullptr);
        PMGR_LAUNCHED();
    }
    int64_t nz = exclusive_scan_total(cnt.p, K.ro.p, n, s);
    K.nrows = n;
    K.ncols = M.ncols;
    K.nnz = nz;
    K.ci.alloc(nz);
    K.v.alloc(nz);
    if (n) {
        k_sparsify<true><<<grid_for(n, 128), 128, 0, s>>>(n, M.ro, M.ci, M.v, entity, n_max, nullptr,
                                                          K.ro.p, K.ci.p, K.v.p);
        PMGR_LAUNCHED();
    }
}

void csr_diagonal(const CsrView &A, double *d, cudaStream_t s) {
    int64_t n = A.nrows < A.ncols ? A.nrows : A.ncols;
    if (n == 0) return;
    k_diag<<<grid_for(n * 32, 256), 256, 0, s>>>(n, A.ro, A.ci, A.v, d);
    PMGR_LAUNCHED();
}

int64_t csr_diag_inverse(const CsrView &A, double *dinv, cudaStream_t s) {
    int64_t n = A.nrows;
    if (n == 0) return -1;
    TBuf<double> d(n, s);
    csr_diagonal(A, d.p, s);
    TBuf<unsigned long long> bad(1, s);
    k_fill_u64<<<1, 32, 0, s>>>(bad.p, 1, ~0ull);
    PMGR_LAUNCHED();
    k_diag_inverse<<<grid_for(n, 256), 256, 0, s>>>(n, d.p, dinv, bad.p);
    PMGR_LAUNCHED();
    unsigned long long b = read_scalar(bad.p, s);
    return b == ~0ull ? -1 : (int64_t)b;
}

}  // namespace pmgr

namespace pmgr {
namespace {
__global__ void k_perm_count(int64_t n, const int64_t *ro, const int64_t *perm, int64_t *cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) cnt[i] = ro[perm[i] + 1] - ro[perm[i]];
}
__global__ void k_perm_fill(int64_t n, const int64_t *ro, const int32_t *ci, const double *v, const int64_t *perm,
                            const int64_t *inv, const int64_t *nro, int32_t *nci, double *nv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t r = perm[i];
    int64_t w = nro[i];
    for (int64_t q = ro[r]; q < ro[r + 1]; ++q, ++w) {
        nci[w] = (int32_t)inv[ci[q]];
        nv[w] = v[q];
    }
}
}  // namespace

// B = P A P^T: row i of B is row perm[i] of A, columns renumbered by the
// inverse permutation and re-sorted (problems.rank_major on the device)
std::shared_ptr<Csr> csr_permute(const Csr &A, const int64_t *perm_h, cudaStream_t s) {
    if (A.nrows != A.ncols) fail(PMGR_ERR_INVALID, "permutation needs a square matrix");
    const int64_t n = A.nrows;
    std::vector<int64_t> inv_h(n, -1);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t p = perm_h[i];
        if (p < 0 || p >= n || inv_h[p] >= 0) fail(PMGR_ERR_INVALID, "not a permutation", i);
        inv_h[p] = i;
    }
    TBuf<int64_t> perm(n, s), inv(n, s), cnt(n, s);
    PMGR_CUDA(cudaMemcpyAsync(perm.p, perm_h, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    PMGR_CUDA(cudaMemcpyAsync(inv.p, inv_h.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, s));
    auto B = std::make_shared<Csr>();
    B->nrows = B->ncols = n;
    B->ro.alloc(n + 1);
    if (n > 0) {
        k_perm_count<<<grid_for(n, 256), 256, 0, s>>>(n, A.ro.p, perm.p, cnt.p);
        PMGR_LAUNCHED();
    }
    B->nnz = exclusive_scan_total(cnt.p, B->ro.p, n, s);
    B->ci.alloc(B->nnz);
    B->v.alloc(B->nnz);
    if (n > 0) {
        k_perm_fill<<<grid_for(n, 256), 256, 0, s>>>(n, A.ro.p, A.ci.p, A.v.p, perm.p, inv.p, B->ro.p, B->ci.p,
                                                     B->v.p);
        PMGR_LAUNCHED();
    }
    segmented_sort_pairs(B->ci.p, B->v.p, B->nnz, B->ro.p, n, s);
    csr_finalize(*B, s, false);  // a caller's matrix: sliced jagged copy at first use
    PMGR_CUDA(cudaStreamSynchronize(s));
    return B;
}
}  // namespace pmgr
