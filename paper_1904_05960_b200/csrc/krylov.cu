// krylov.cu -- right-preconditioned restarted GMRES on the device
// (reference krylov.py:39-117).
//
// Outer semantics follow the reference exactly: x0 = 0 unless given;
// convergence on ||b - A x|| <= max(rtol*||r0||, atol); Givens least
// squares; at each restart x += M^{-1}(V y) and the true residual replaces
// the last history entry; an Arnoldi breakdown counts as convergence in the
// subspace; a dead Givens column (rho == 0) is discarded.
//
// B200 design:
//  * The whole Arnoldi step -- MGR apply, SpMV, projections, Hessenberg /
//    Givens update, normalisation -- reads the step index j from device
//    memory, so one captured CUDA graph serves every step.  The restart cycle
//    is a graph WHILE node: the Givens kernel sets the loop condition with
//    cudaGraphSetConditional, and the host synchronises once per cycle.
//  * Orthogonalisation is classical Gram-Schmidt with the re-orthogonalising
//    second projection taken from the basis Gram matrix G = V^T V
//    (h = a + (a - G a) with a = V^T w): the Gram column of the newest basis
//    vector rides along in the same streaming pass as a, so each step reads
//    the Krylov basis twice (projection + update) instead of MGS's
//    2(j+1) vector sweeps, and stays as orthogonal as CGS2 (SURVEY §7.4 (8):
//    not bitwise MGS; iteration counts within +-1).
//  * With kernel timing enabled (pmgr_prof_enable) the same kernels are
//    launched step by step with CUDA events around them (event nodes are not
//    allowed inside conditional bodies).
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include <cooperative_groups.h>

#include "hier.cuh"

namespace cg = cooperative_groups;

namespace pmgr {

namespace {

constexpr int DOT_BLOCK = 256;

struct Dev {
    int j;       // current step within the cycle
    int total;   // iterations over all cycles
    int active;  // loop condition
    int brk;     // breakdown in the last step
    int dead;    // dead Givens column
    int m, max_iters;
    double tol;
    double hn;   // ||w|| after the projections
};

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// block-wide sum of two values; valid in thread 0
__device__ __forceinline__ void block_sum2(double &a, double &b, double *sh) {
    a = warp_sum(a);
    b = warp_sum(b);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        sh[2 * w] = a;
        sh[2 * w + 1] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double x = 0.0, y = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
            x += sh[2 * k];
            y += sh[2 * k + 1];
        }
        a = x;
        b = y;
    }
}

// ---- one cooperative kernel per Arnoldi step --------------------------
// Every block owns a contiguous slice of rows.  Phase 1 streams the basis
// once (warp per basis vector, lanes over the slice's rows) for the
// projections a_k = V_k.w and the Gram column g_k = V_k.V_j; phase 2 turns
// the slice partials into h = a + (a - G a); phase 3 updates w on the same
// rows (the basis slice is re-read from L2, not HBM); phase 4 normalises and
// block 0 does the Hessenberg / Givens / convergence bookkeeping
// (krylov.py:75-104) and sets the WHILE condition.  Three grid barriers
// replace five launches and half of the basis traffic.
constexpr int AO_THREADS = 256;
constexpr int AO_UM = 10;  // phase 1: double2 loads per lane per basis vector batch
constexpr int AO_WARPS = AO_THREADS / 32;
// rows per shared-memory tile of the projection phase when the block's slice
// does not fit (PMGR_ARNOLDI_TILE, multiple of 32; 0: off)
inline int arnoldi_tile() {
    static const int t = [] {
        const char *e = getenv("PMGR_ARNOLDI_TILE");
        // (768-row tiles: 2.22 ms per projection phase at C4; 1,024 / 2,048 /
        // 4,096 rows: 1.97-1.98 ms)
        int v = e ? atoi(e) : 2048;
        if (v < 0) v = 0;
        if (v > 8192) v = 8192;
        return v / 32 * 32;
    }();
    return t;
}

struct AoParams {
    double *V;
    int64_t n, ldv, chunk;  // basis leading dimension and rows per block (multiples of 32)
    double *w, *vin;
    Dev *dev;
    double *pa, *pg, *pn;  // slice partials: (m+1) x nblk, (m+1) x nblk, nblk
    double *G;
    int ldg;
    double *a, *h;
    double *H, *cs, *sn, *g, *hist;
    cudaGraphConditionalHandle cond;
    int use_cond;
    unsigned long long *stamps;  // PMGR_ARNOLDI_STAMPS: phase timestamps of block 0 (diagnostics)
    // split modes (row-distributed GMRES): projections and the squared norm
    // leave the kernel for a cross-rank all-reduce
    double *red, *nrm2;
    // SM = false: rows per shared-memory tile of the projection phase (0: the
    // w / V_j slices are re-read from L2 for every pair of basis vectors)
    int tile;
};

__device__ __forceinline__ void stamp(const AoParams &P, int slot) {
    if (P.stamps && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicAdd(P.stamps + slot, t);
    }
}

__device__ __forceinline__ double block_sum1(double v, double *sh) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];  // every thread, same order
    return t;
}

// SM = true: the block's slices of w and V_j live in shared memory, so the
// basis stream is the only per-vector L2/HBM traffic and w never returns to
// global memory (small and medium n); SM = false streams them from L2.
// MODE 0: the whole step in one cooperative launch.  Split modes for the
// row-distributed solve (each a plain launch; all-reduces in between):
// 1 = projections' slice partials, 2 = their block sums into red (a, g),
// 3 = coefficients h and the update w -= V h with slice norms, 4 = the
// normalisation with ||w||^2 from nrm2 and the Givens bookkeeping.
template <bool SM, int MODE = 0>
__global__ void __launch_bounds__(AO_THREADS, 2) k_arnoldi(AoParams P) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double slice[];  // SM: w slice, then V_j slice
    __shared__ double sh[AO_WARPS];
    __shared__ double hs[1024];   // h
    __shared__ double as_[1024];  // a
    __shared__ double red[AO_WARPS][128];
    const int nblk = gridDim.x, b = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int j = P.dev->j;
    const int64_t n = P.n;
    const int64_t ldv = P.ldv, chunk = P.chunk;
    const int64_t lo = (int64_t)b * chunk;
    const int64_t hi = lo + chunk < n ? lo + chunk : (n > lo ? n : lo);
    stamp(P, 0);
    const double *vjg = P.V + (int64_t)j * ldv;
    double *wsl = slice;
    double *vsl = slice + chunk;
    if (SM) {
        for (int64_t i = lo + threadIdx.x; i < hi; i += AO_THREADS) {
            wsl[i - lo] = P.w[i];
            vsl[i - lo] = vjg[i];
        }
        __syncthreads();
    }
    // row-indexed accessors for the w / V_j slices (shared or global)
    auto wv = [&](int64_t i) { return SM ? wsl[i - lo] : P.w[i]; };
    auto vj = [&](int64_t i) { return SM ? vsl[i - lo] : vjg[i]; };

    // phase 1: slice partials of V_k.w and V_k.V_j.  A warp takes two basis
    // vectors at a time and issues every 16-byte load of both slices before
    // consuming them (one memory latency per pair for slices up to 640 rows);
    // slices are 256-byte aligned (ldv, chunk multiples of 32).
    if constexpr (!SM && (MODE == 0 || MODE == 1)) {
        // large n: the block's slice does not fit shared memory.  Walk it in
        // tiles of P.tile rows whose w / V_j parts are staged in shared memory
        // once and reused by every pair of basis vectors (streaming them from
        // L2 per pair doubled the phase's L2 traffic: 2.55 ms against 1.95 ms
        // for the update phase at C4); the per-vector partials of the tiles
        // are summed in tile order in hs / as_ (free until phase 2b).
        if (P.tile > 0) {
            const int tile = P.tile;
            for (int k = threadIdx.x; k <= j; k += AO_THREADS) {
                hs[k] = 0.0;
                as_[k] = 0.0;
            }
            __syncthreads();
            for (int64_t t0 = lo; t0 < hi; t0 += tile) {
                const int64_t t1 = t0 + tile < hi ? t0 + tile : hi;
                const int len = (int)(t1 - t0), len2 = len >> 1;
                for (int64_t i = t0 + threadIdx.x; i < t1; i += AO_THREADS) {
                    slice[i - t0] = P.w[i];
                    slice[tile + (i - t0)] = vjg[i];
                }
                __syncthreads();
                const double2 *w2 = reinterpret_cast<const double2 *>(slice);
                const double2 *v2 = reinterpret_cast<const double2 *>(slice + tile);
                for (int k = 2 * warp; k <= j; k += 2 * AO_WARPS) {
                    double a0[2] = {0.0, 0.0}, a1[2] = {0.0, 0.0}, g0[2] = {0.0, 0.0}, g1[2] = {0.0, 0.0};
                    for (int base = 0; base < len2; base += 32 * AO_UM) {
                        double2 xs[2][AO_UM];
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            const double2 *x2 = reinterpret_cast<const double2 *>(P.V + (int64_t)(k + q) * ldv + t0);
#pragma unroll
                            for (int u = 0; u < AO_UM; ++u) {
                                const int p = base + lane + 32 * u;
                                xs[q][u] = (k + q <= j && p < len2) ? x2[p] : make_double2(0.0, 0.0);
                            }
                        }
#pragma unroll
                        for (int u = 0; u < AO_UM; ++u) {
                            const int p = base + lane + 32 * u;
                            if (p < len2) {
                                const double2 ww = w2[p], vv = v2[p];
#pragma unroll
                                for (int q = 0; q < 2; ++q) {
                                    a0[q] = fma(xs[q][u].x, ww.x, a0[q]);
                                    a1[q] = fma(xs[q][u].y, ww.y, a1[q]);
                                    g0[q] = fma(xs[q][u].x, vv.x, g0[q]);
                                    g1[q] = fma(xs[q][u].y, vv.y, g1[q]);
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        if ((len & 1) && lane == 0 && k + q <= j) {  // odd last tile: its final row
                            const double xl = P.V[(int64_t)(k + q) * ldv + t1 - 1];
                            a0[q] = fma(xl, slice[len - 1], a0[q]);
                            g0[q] = fma(xl, slice[tile + len - 1], g0[q]);
                        }
                        const double sa = warp_sum(a0[q] + a1[q]);
                        const double sg = warp_sum(g0[q] + g1[q]);
                        if (lane == 0 && k + q <= j) {  // this warp owns k and k + 1 in every tile
                            hs[k + q] += sa;
                            as_[k + q] += sg;
                        }
                    }
                }
                __syncthreads();
            }
            for (int k = threadIdx.x; k <= j; k += AO_THREADS) {
                P.pa[(int64_t)k * nblk + b] = hs[k];
                P.pg[(int64_t)k * nblk + b] = as_[k];
            }
            __syncthreads();
        }
    }
    if constexpr (MODE == 0 || MODE == 1)
    if (SM || P.tile <= 0) {
        const int len = (int)(hi - lo), len2 = len >> 1;
        const double2 *w2 = reinterpret_cast<const double2 *>(SM ? wsl : P.w + lo);
        const double2 *v2 = reinterpret_cast<const double2 *>(SM ? vsl : vjg + lo);
        for (int k = 2 * warp; k <= j; k += 2 * AO_WARPS) {
            double a0[2] = {0.0, 0.0}, a1[2] = {0.0, 0.0}, g0[2] = {0.0, 0.0}, g1[2] = {0.0, 0.0};
            for (int base = 0; base < len2; base += 32 * AO_UM) {
                double2 xs[2][AO_UM];
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const double2 *x2 = reinterpret_cast<const double2 *>(P.V + (int64_t)(k + q) * ldv + lo);
#pragma unroll
                    for (int u = 0; u < AO_UM; ++u) {
                        const int p = base + lane + 32 * u;
                        xs[q][u] = (k + q <= j && p < len2) ? x2[p] : make_double2(0.0, 0.0);
                    }
                }
#pragma unroll
                for (int u = 0; u < AO_UM; ++u) {
                    const int p = base + lane + 32 * u;
                    if (p < len2) {
                        const double2 ww = w2[p], vv = v2[p];
#pragma unroll
                        for (int q = 0; q < 2; ++q) {
                            a0[q] = fma(xs[q][u].x, ww.x, a0[q]);
                            a1[q] = fma(xs[q][u].y, ww.y, a1[q]);
                            g0[q] = fma(xs[q][u].x, vv.x, g0[q]);
                            g1[q] = fma(xs[q][u].y, vv.y, g1[q]);
                        }
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if ((len & 1) && lane == 0 && k + q <= j) {  // odd last slice: its final row
                    const double xl = P.V[(int64_t)(k + q) * ldv + hi - 1];
                    a0[q] = fma(xl, wv(hi - 1), a0[q]);
                    g0[q] = fma(xl, vj(hi - 1), g0[q]);
                }
                const double sa = warp_sum(a0[q] + a1[q]);
                const double sg = warp_sum(g0[q] + g1[q]);
                if (lane == 0 && k + q <= j) {
                    P.pa[(int64_t)(k + q) * nblk + b] = sa;
                    P.pg[(int64_t)(k + q) * nblk + b] = sg;
                }
            }
        }
    }
    if constexpr (MODE == 1) return;
    stamp(P, 1);
    if constexpr (MODE == 0) grid.sync();
    stamp(P, 2);
    // phase 2a: a_k and the Gram column, one block per coefficient (a warp
    // per coefficient measured slower: 2.9 -> 3.8 us)
    if constexpr (MODE == 0 || MODE == 2)
    for (int k = b; k <= j; k += nblk) {
        double sa = 0.0, sg = 0.0;
        for (int t = threadIdx.x; t < nblk; t += AO_THREADS) {
            sa += P.pa[(int64_t)k * nblk + t];
            sg += P.pg[(int64_t)k * nblk + t];
        }
        sa = block_sum1(sa, sh);
        sg = block_sum1(sg, sh);
        if (threadIdx.x == 0) {
            if constexpr (MODE == 2) {
                P.red[k] = sa;
                P.red[P.ldg + k] = sg;
            } else {
                P.a[k] = sa;
                P.G[(int64_t)k * P.ldg + j] = sg;
                P.G[(int64_t)j * P.ldg + k] = sg;
            }
        }
    }
    if constexpr (MODE == 2) return;
    stamp(P, 3);
    if constexpr (MODE == 0) grid.sync();
    stamp(P, 4);
    if constexpr (MODE == 0 || MODE == 3) {
    // phase 2b: h = a + (a - G a), every block for itself.  G is symmetric,
    // so (G a)_k = sum_l G[l][k] a_l: warps split l, lanes take k (coalesced
    // rows of G, every load of a lane independent), then a fixed-order sum
    // over the warps.
    for (int k = threadIdx.x; k <= j; k += AO_THREADS) as_[k] = P.a[k];
    __syncthreads();
    for (int c0 = 0; c0 <= j; c0 += 128) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 4
        for (int l = warp; l <= j; l += AO_WARPS) {
            const double al = as_[l];
            const double *row = P.G + (int64_t)l * P.ldg;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int k = c0 + 32 * c + lane;
                if (k <= j) acc[c] = fma(row[k], al, acc[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) red[warp][32 * c + lane] = acc[c];
        __syncthreads();
        if (threadIdx.x < 128 && c0 + (int)threadIdx.x <= j) {
            const int k = c0 + threadIdx.x;
            double ga = 0.0;
            for (int w = 0; w < AO_WARPS; ++w) ga += red[w][threadIdx.x];
            hs[k] = as_[k] + (as_[k] - ga);
        }
        __syncthreads();
    }
    if (b == 0)
        for (int k = threadIdx.x; k <= j; k += AO_THREADS) P.h[k] = hs[k];
    stamp(P, 7);
    // phase 3: w -= sum_k h_k V_k on this slice (row pairs, 16 basis vectors
    // per batch: 32 independent L2 loads in flight per thread), ||w||^2 partial
    double nrm = 0.0;
    if constexpr (SM) {
        // the update mirrors phase 1's mapping: a warp takes basis vectors
        // k = warp (mod 8), its lanes the slice's row pairs (10 16-byte loads
        // in flight per lane), so every thread streams the same amount; the
        // eight warps' partial sums meet in shared memory in a fixed order
        const int len = (int)(hi - lo), len2 = len >> 1;
        double2 *wo2 = reinterpret_cast<double2 *>(wsl);
        double2 *rp = reinterpret_cast<double2 *>(slice + 2 * chunk);  // [AO_WARPS][32 * AO_UM]
        for (int base = 0; base < len2; base += 32 * AO_UM) {
            double2 acc[AO_UM];
#pragma unroll
            for (int u = 0; u < AO_UM; ++u) acc[u] = make_double2(0.0, 0.0);
            for (int k = warp; k <= j; k += AO_WARPS) {
                const double hk = -hs[k];
                const double2 *x2 = reinterpret_cast<const double2 *>(P.V + (int64_t)k * ldv + lo);
                double2 xs[AO_UM];
#pragma unroll
                for (int u = 0; u < AO_UM; ++u) {
                    const int p = base + lane + 32 * u;
                    xs[u] = p < len2 ? x2[p] : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int u = 0; u < AO_UM; ++u) {
                    acc[u].x = fma(hk, xs[u].x, acc[u].x);
                    acc[u].y = fma(hk, xs[u].y, acc[u].y);
                }
            }
#pragma unroll
            for (int u = 0; u < AO_UM; ++u) rp[warp * 32 * AO_UM + lane + 32 * u] = acc[u];
            __syncthreads();
            const int nb2 = len2 - base < 32 * AO_UM ? len2 - base : 32 * AO_UM;
            for (int q = threadIdx.x; q < nb2; q += AO_THREADS) {
                double2 t = wo2[base + q];
#pragma unroll
                for (int w = 0; w < AO_WARPS; ++w) {
                    const double2 r = rp[w * 32 * AO_UM + q];
                    t.x += r.x;
                    t.y += r.y;
                }
                wo2[base + q] = t;
                nrm = fma(t.x, t.x, nrm);
                nrm = fma(t.y, t.y, nrm);
            }
            __syncthreads();
        }
        if ((len & 1) && threadIdx.x == 0) {  // odd last slice: its final row
            const int64_t i = hi - 1;
            double acc = wsl[i - lo];
            for (int k = 0; k <= j; ++k) acc = fma(-hs[k], P.V[(int64_t)k * ldv + i], acc);
            wsl[i - lo] = acc;
            nrm = fma(acc, acc, nrm);
        }
    } else {
        const int len = (int)(hi - lo), len2 = len >> 1;
        double2 *wo2 = reinterpret_cast<double2 *>(SM ? wsl : P.w + lo);
        const double2 *Vb = reinterpret_cast<const double2 *>(P.V + lo);
        const int64_t ld2 = ldv >> 1;
        for (int p = threadIdx.x; p < len2; p += AO_THREADS) {
            double2 acc[4];
            acc[0] = wo2[p];
            acc[1] = acc[2] = acc[3] = make_double2(0.0, 0.0);
            for (int k = 0; k <= j; k += 16) {
                double2 vv[16];
                double hc[16];
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    const bool ok = k + t <= j;
                    vv[t] = ok ? Vb[(int64_t)(k + t) * ld2 + p] : make_double2(0.0, 0.0);
                    hc[t] = ok ? -hs[k + t] : 0.0;
                }
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    acc[t & 3].x = fma(hc[t], vv[t].x, acc[t & 3].x);
                    acc[t & 3].y = fma(hc[t], vv[t].y, acc[t & 3].y);
                }
            }
            double2 wi;
            wi.x = (acc[0].x + acc[1].x) + (acc[2].x + acc[3].x);
            wi.y = (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y);
            wo2[p] = wi;
            nrm = fma(wi.x, wi.x, nrm);
            nrm = fma(wi.y, wi.y, nrm);
        }
        if ((len & 1) && threadIdx.x == 0) {  // odd last slice: its final row
            const int64_t i = hi - 1;
            double acc = wv(i);
            for (int k = 0; k <= j; ++k) acc = fma(-hs[k], P.V[(int64_t)k * ldv + i], acc);
            if (SM) wsl[i - lo] = acc;
            else P.w[i] = acc;
            nrm = fma(acc, acc, nrm);
        }
    }
    nrm = block_sum1(nrm, sh);
    if (threadIdx.x == 0) P.pn[b] = nrm;
    }  // phases 2b and 3
    if constexpr (MODE == 3) {
        if constexpr (SM) {  // the next split launch reads w from global memory
            __syncthreads();
            for (int64_t i = lo + threadIdx.x; i < hi; i += AO_THREADS) P.w[i] = wsl[i - lo];
        }
        return;
    }
    stamp(P, 5);
    if constexpr (MODE == 0) grid.sync();
    stamp(P, 6);
    // phase 4: ||w||, breakdown test, normalisation (every block, same order)
    double s2 = 0.0;
    if constexpr (MODE == 4) {
        for (int k = threadIdx.x; k <= j; k += AO_THREADS) hs[k] = P.h[k];
        __syncthreads();
        s2 = *P.nrm2;
    } else {
        for (int t = threadIdx.x; t < nblk; t += AO_THREADS) s2 += P.pn[t];
        s2 = block_sum1(s2, sh);
    }
    const double hn = sqrt(s2);
    // ||h||^2 by every warp (lanes over k, butterfly sum: the same value in
    // every thread)
    double c2 = 0.0;
    for (int k = lane; k <= j; k += 32) c2 = fma(hs[k], hs[k], c2);
    c2 = warp_sum(c2);
    c2 += hn * hn;
    const int brk = !(hn > 1e-12 * fmax(sqrt(c2), 1e-300));
    if (!brk && j + 1 <= P.dev->m) {
        double *vn = P.V + (int64_t)(j + 1) * ldv;
        for (int64_t i = lo + threadIdx.x; i < hi; i += AO_THREADS) {
            const double t = (SM ? wsl[i - lo] : P.w[i]) / hn;
            vn[i] = t;
            P.vin[i] = t;
        }
    }
    stamp(P, 8);
    if (b != 0) return;
    // Hessenberg column j and Givens rotation: block 0 stages the previous
    // rotations in shared memory, one thread applies them (carry in registers)
    double *css = as_;  // a is no longer needed
    __shared__ double sns[1024];
    for (int i = threadIdx.x; i < j; i += AO_THREADS) {
        css[i] = P.cs[i];
        sns[i] = P.sn[i];
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const int m = P.dev->m;
    double carry = hs[0];
    for (int i = 0; i < j; ++i) {
        const double next = hs[i + 1];
        const double c = css[i], sn = sns[i];
        P.H[(int64_t)i * m + j] = c * carry + sn * next;
        carry = -sn * carry + c * next;
    }
    const double av = carry, bv = hn;
    const double rho = hypot(av, bv);
    Dev *dv = P.dev;
    dv->hn = hn;
    if (rho == 0.0) {
        dv->brk = 1;
        dv->dead = 1;
        dv->active = 0;
        if (P.use_cond) cudaGraphSetConditional(P.cond, 0);
        return;
    }
    P.cs[j] = av / rho;
    P.sn[j] = bv / rho;
    P.H[(int64_t)j * m + j] = rho;
    P.H[(int64_t)(j + 1) * m + j] = 0.0;
    P.g[j + 1] = -P.sn[j] * P.g[j];
    P.g[j] = P.cs[j] * P.g[j];
    const double est = fabs(P.g[j + 1]);
    P.hist[dv->total] = est;
    const int total = dv->total + 1;
    const int jn = j + 1;
    dv->total = total;
    dv->j = jn;
    dv->brk = brk;
    const int act = !(est <= dv->tol || brk) && jn < m && total < dv->max_iters;
    dv->active = act;
    if (P.use_cond) cudaGraphSetConditional(P.cond, act);
}

__global__ void k_cycle_init(Dev *dev, double *H, double *G, int ldg, double *cs, double *sn, double *g, int m,
                             const double *beta) {
    for (int64_t i = threadIdx.x; i < (int64_t)(m + 1) * m; i += blockDim.x) H[i] = 0.0;
    for (int64_t i = threadIdx.x; i < (int64_t)ldg * ldg; i += blockDim.x) G[i] = 0.0;
    for (int i = threadIdx.x; i <= m; i += blockDim.x) {
        g[i] = (i == 0) ? *beta : 0.0;
        cs[i] = sn[i] = 0.0;
    }
    if (threadIdx.x == 0) {
        dev->j = 0;
        dev->brk = 0;
        dev->dead = 0;
        dev->active = dev->total < dev->max_iters;
    }
}

__global__ void k_scale2(const double *x, int64_t n, const double *den, double *y, double *y2) {
    const double d = *den;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double t = x[i] / d;
        y[i] = t;
        y2[i] = t;
    }
}

// back substitution H[:j,:j] y = g[:j], right-looking, one block
__global__ void k_trsv(const double *H, int m, int j, const double *g, double *y) {
    extern __shared__ double rhs[];
    __shared__ double yc_s;
    for (int i = threadIdx.x; i < j; i += blockDim.x) rhs[i] = g[i];
    __syncthreads();
    for (int c = j - 1; c >= 0; --c) {
        if (threadIdx.x == 0) {
            yc_s = rhs[c] / H[(int64_t)c * m + c];
            rhs[c] = yc_s;
        }
        __syncthreads();
        const double yc = yc_s;
        for (int i = threadIdx.x; i < c; i += blockDim.x) rhs[i] -= H[(int64_t)i * m + c] * yc;
        __syncthreads();
    }
    for (int i = threadIdx.x; i < j; i += blockDim.x) y[i] = rhs[i];
}

// u = sum_{k<j} y_k V_k
__global__ void k_combine(const double *__restrict__ V, int64_t n, int64_t ldv, int nk, const double *__restrict__ y,
                          double *u) {
    __shared__ double ys[1024];
    for (int k = threadIdx.x; k < nk; k += blockDim.x) ys[k] = y[k];
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double s0 = 0.0, s1 = 0.0;
        int k = 0;
        for (; k + 1 < nk; k += 2) {
            s0 = fma(ys[k], V[(int64_t)k * ldv + i], s0);
            s1 = fma(ys[k + 1], V[(int64_t)(k + 1) * ldv + i], s1);
        }
        if (k < nk) s0 = fma(ys[k], V[(int64_t)k * ldv + i], s0);
        u[i] = s0 + s1;
    }
}

__global__ void k_norm_partial(const double *x, int64_t n, double *pn) {
    __shared__ double sh[2 * DOT_BLOCK / 32];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)DOT_BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * DOT_BLOCK)
        s = fma(x[i], x[i], s);
    double z = 0.0;
    block_sum2(s, z, sh);
    if (threadIdx.x == 0) pn[blockIdx.x] = s;
}

__global__ void k_norm_final(const double *pn, int npn, double *out) {
    double s = 0.0;
    for (int b = threadIdx.x; b < npn; b += 32) s += pn[b];
    s = warp_sum(s);
    if (threadIdx.x == 0) *out = sqrt(s);
}

// split-mode helpers (row-distributed GMRES)
__global__ void k_split_fix(Dev *dev, const double *red, int ldg, double *a, double *G) {
    const int j = dev->j;
    for (int k = threadIdx.x; k <= j; k += blockDim.x) {
        a[k] = red[k];
        G[(int64_t)k * ldg + j] = red[ldg + k];
        G[(int64_t)j * ldg + k] = red[ldg + k];
    }
}
__global__ void k_sum_fixed(const double *p, int np, double *out) {  // one thread: fixed order
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < np; ++i) s += p[i];
        *out = s;
    }
}
__global__ void k_sqrt_inplace(double *x) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *x = sqrt(*x);
}
__global__ void k_sub(const double *b, const double *y, int64_t n, double *r) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) r[i] = b[i] - y[i];
}

// generic helpers for the Python-callable path
__global__ void __launch_bounds__(DOT_BLOCK) k_mdot_plain(const double *__restrict__ V, int64_t n,
                                                           const double *__restrict__ w, double *part, int nsplit,
                                                           int64_t chunk) {
    __shared__ double sh[2 * DOT_BLOCK / 32];
    const int k = blockIdx.y;
    const double *x = V + (int64_t)k * n;
    const int64_t lo = blockIdx.x * chunk, hi = lo + chunk < n ? lo + chunk : n;
    double a = 0.0, z = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += DOT_BLOCK) a = fma(x[i], w[i], a);
    block_sum2(a, z, sh);
    if (threadIdx.x == 0) part[(int64_t)k * nsplit + blockIdx.x] = a;
}

__global__ void k_sum_slices(const double *part, int nsplit, int nk, double *out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nk) return;
    double s = 0.0;
    for (int b = 0; b < nsplit; ++b) s += part[(int64_t)k * nsplit + b];
    out[k] = s;
}

__global__ void k_maxpy(const double *__restrict__ V, int64_t n, int nk, const double *__restrict__ h, double *w) {
    __shared__ double hs[1024];
    for (int k = threadIdx.x; k < nk; k += blockDim.x) hs[k] = h[k];
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double a = w[i];
        for (int k = 0; k < nk; ++k) a = fma(-hs[k], V[(int64_t)k * n + i], a);
        w[i] = a;
    }
}

// --------------------------------------------------------------- workspace

struct Ws {
    const pmgr_csr *A = nullptr;
    pmgr_mgr *M = nullptr;
    int m = 0, max_iters = 0;
    int64_t n = 0;
    int nblk = 1, nupd = 1;
    int64_t ldv = 0, chunk = 0;
    bool use_smem = false;
    int tile = 0;  // projection tile rows of the global-memory variant
    size_t smem = 0;
    DBuf<double> V, w, z, r, vin, u;
    DBuf<double> H, G, cs, sn, g, a, h, y, hist, pa, pg, pn, beta;
    DBuf<Dev> dev;
    DBuf<unsigned long long> stamps;  // diagnostics (null unless PMGR_ARNOLDI_STAMPS)
    Dev *hdev = nullptr;  // pinned mirror
    cudaStream_t cap = nullptr;
    cudaGraphExec_t cycle = nullptr;
    int64_t body_kernels = 0;  // kernels per Arnoldi step in the WHILE body

    ~Ws() {
        if (cycle) cudaGraphExecDestroy(cycle);
        if (cap) cudaStreamDestroy(cap);
        if (hdev) cudaFreeHost(hdev);
    }
};

// keyed on (A, M, restart): max_iters only sizes the history buffer, which
// grows on demand (the captured cycle graph is rebuilt when it moves).  One
// mutex serialises the solves that share the cache (ctypes releases the GIL).
std::map<std::tuple<const pmgr_csr *, pmgr_mgr *, int>, std::unique_ptr<Ws>> g_ws;
std::recursive_mutex g_ws_mu;

Ws &workspace(const pmgr_csr *A, pmgr_mgr *M, int m, int max_iters, int64_t n) {
    auto key = std::make_tuple(A, M, m);
    auto it = g_ws.find(key);
    if (it != g_ws.end()) {
        Ws &w = *it->second;
        if (max_iters > w.max_iters) {
            w.hist.alloc((int64_t)max_iters + 2);
            w.max_iters = max_iters;
            if (w.cycle) {
                cudaGraphExecDestroy(w.cycle);
                w.cycle = nullptr;
            }
        }
        return w;
    }
    auto w = std::make_unique<Ws>();
    w->A = A;
    w->M = M;
    w->m = m;
    w->max_iters = max_iters;
    w->n = n;
    w->ldv = (n + 31) / 32 * 32;
    w->V.alloc((int64_t)(m + 1) * w->ldv);
    w->w.alloc(n);
    w->z.alloc(n);
    w->r.alloc(n);
    w->vin.alloc(n);
    w->u.alloc(n);
    w->H.alloc((int64_t)(m + 1) * m);
    w->G.alloc((int64_t)(m + 1) * (m + 1));
    w->cs.alloc(m + 1);
    w->sn.alloc(m + 1);
    w->g.alloc(m + 2);
    w->a.alloc(m + 1);
    w->h.alloc(m + 1);
    w->y.alloc(m + 1);
    w->hist.alloc((int64_t)max_iters + 2);
    // the cooperative Arnoldi kernel: every block resident at once
    int per_sm = 0;
    PMGR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_arnoldi<false>, AO_THREADS, 0));
    if (per_sm < 1) fail(PMGR_ERR_CUDA, "Arnoldi kernel cannot be resident");
    int bps = 2;
    if (const char *e = getenv("PMGR_ARNOLDI_BPS")) bps = atoi(e) > 0 ? atoi(e) : 2;
    w->nblk = (per_sm < bps ? per_sm : bps) * num_sms();
    {
        const int64_t chunk = ((n + w->nblk - 1) / w->nblk + 31) / 32 * 32;
        w->chunk = chunk;
        int per_sm_sm = 0;
        // w and V_j slices, then the update's per-warp partial sums
        w->smem = (size_t)(16 * chunk) + (size_t)AO_WARPS * 32 * AO_UM * 16;
        cudaFuncSetAttribute(k_arnoldi<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)w->smem);
        if (chunk <= 3072 &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_sm, k_arnoldi<true>, AO_THREADS, w->smem) ==
                cudaSuccess &&
            per_sm_sm * num_sms() >= w->nblk) {
            w->use_smem = true;
        } else {
            cudaGetLastError();
            w->use_smem = false;
            w->smem = 0;
            // projection tiles of the global-memory variant
            const int tile = arnoldi_tile();
            int per_sm_t = 0;
            if (tile > 0 && chunk > tile &&
                cudaFuncSetAttribute(k_arnoldi<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * tile) ==
                    cudaSuccess &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_t, k_arnoldi<false>, AO_THREADS,
                                                              (size_t)16 * tile) == cudaSuccess &&
                (int64_t)per_sm_t * num_sms() >= w->nblk) {
                w->tile = tile;
                w->smem = (size_t)16 * tile;
            } else {
                cudaGetLastError();
            }
        }
    }
    w->pa.alloc((int64_t)(m + 1) * w->nblk);
    w->pg.alloc((int64_t)(m + 1) * w->nblk);
    w->nupd = 4 * num_sms();
    w->pn.alloc(w->nblk > w->nupd ? w->nblk : w->nupd);
    w->beta.alloc(1);
    w->dev.alloc(1);
    if (getenv("PMGR_ARNOLDI_STAMPS")) {
        w->stamps.alloc(16);
        PMGR_CUDA(cudaMemset(w->stamps.p, 0, 16 * sizeof(unsigned long long)));
    }
    PMGR_CUDA(cudaMallocHost((void **)&w->hdev, sizeof(Dev)));
    PMGR_CUDA(cudaStreamCreateWithFlags(&w->cap, cudaStreamNonBlocking));
    Ws &ref = *w;
    g_ws[key] = std::move(w);
    return ref;
}

int vec_grid(int64_t n) {
    int64_t g = (n + 255) / 256;
    int64_t cap = 4LL * num_sms();
    return (int)(g < 1 ? 1 : (g < cap ? g : cap));
}

// one Arnoldi step on stream s (graph body or direct launches)
void arnoldi_step(const CsrView &Av, Ws &W, cudaStream_t s, cudaGraphConditionalHandle cond, int use_cond) {
    const int64_t n = W.n;
    const bool prof = !use_cond && prof_on();
    {
        ProfScope ps(prof ? PROF_MGR_APPLY : PROF_KINDS, 0.0, s);
        if (W.M) mgr_apply_direct(*W.M, W.vin.p, W.z.p, s);
        else vec_copy(W.vin.p, W.z.p, n, s);
    }
    {
        ProfScope ps(prof ? PROF_OUTER_SPMV : PROF_KINDS, csr_pass_bytes(Av), s);
        spmv(Av, W.z.p, W.w.p, s);
    }
    // compulsory bytes of the step's orthogonalisation: the basis V_0..V_j
    // read once, w read and written, V_{j+1} and the preconditioner copy written
    const double bytes = prof ? 8.0 * n * ((W.hdev->j + 1) + 4.0) : 0.0;
    ProfScope ps(prof ? PROF_ORTHO : PROF_KINDS, bytes, s);
    AoParams P;
    P.V = W.V.p;
    P.n = n;
    P.ldv = W.ldv;
    P.chunk = W.chunk;
    P.w = W.w.p;
    P.vin = W.vin.p;
    P.dev = W.dev.p;
    P.pa = W.pa.p;
    P.pg = W.pg.p;
    P.pn = W.pn.p;
    P.G = W.G.p;
    P.ldg = W.m + 1;
    P.a = W.a.p;
    P.h = W.h.p;
    P.H = W.H.p;
    P.cs = W.cs.p;
    P.sn = W.sn.p;
    P.g = W.g.p;
    P.hist = W.hist.p;
    P.cond = cond;
    P.use_cond = use_cond;
    P.stamps = W.stamps.p;
    P.tile = W.use_smem ? 0 : W.tile;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(W.nblk);
    cfg.blockDim = dim3(AO_THREADS);
    cfg.dynamicSmemBytes = W.smem;
    cfg.stream = s;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeCooperative;
    at.val.cooperative = 1;
    cfg.attrs = &at;
    cfg.numAttrs = 1;
    if (W.use_smem) PMGR_CUDA(cudaLaunchKernelEx(&cfg, k_arnoldi<true>, P));
    else PMGR_CUDA(cudaLaunchKernelEx(&cfg, k_arnoldi<false>, P));
    PMGR_LAUNCHED();
}

void build_cycle_graph(const CsrView &Av, Ws &W) {
    cudaGraph_t graph;
    PMGR_CUDA(cudaGraphCreate(&graph, 0));
    cudaGraphConditionalHandle cond;
    PMGR_CUDA(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    PMGR_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    PMGR_CUDA(cudaStreamBeginCaptureToGraph(W.cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    W.body_kernels = 0;
    g_capture_count = &W.body_kernels;
    try {
        arnoldi_step(Av, W, W.cap, cond, 1);
        g_capture_count = nullptr;
    } catch (...) {
        g_capture_count = nullptr;
        cudaStreamEndCapture(W.cap, &body);
        cudaGraphDestroy(graph);
        throw;
    }
    PMGR_CUDA(cudaStreamEndCapture(W.cap, &body));
    PMGR_CUDA(cudaGraphInstantiate(&W.cycle, graph, 0));
    PMGR_CUDA(cudaGraphDestroy(graph));
}

void norm_into(const double *x, int64_t n, Ws &W, double *out, cudaStream_t s) {
    k_norm_partial<<<W.nupd, DOT_BLOCK, 0, s>>>(x, n, W.pn.p);
    PMGR_LAUNCHED();
    k_norm_final<<<1, 32, 0, s>>>(W.pn.p, W.nupd, out);
    PMGR_LAUNCHED();
}

bool use_cycle_graphs() {
    static const bool on = [] {
        const char *e = getenv("PMGR_NO_GRAPHS");
        return !(e && e[0] != '0');
    }();
    return on;
}

}  // namespace

void gmres_forget(const void *obj) {
    std::lock_guard<std::recursive_mutex> lk(g_ws_mu);
    for (auto it = g_ws.begin(); it != g_ws.end();) {
        if ((const void *)std::get<0>(it->first) == obj || (const void *)std::get<1>(it->first) == obj)
            it = g_ws.erase(it);
        else
            ++it;
    }
}

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
    const int max_iters = cfg.max_iters > 0 ? cfg.max_iters : 0;
    std::lock_guard<std::recursive_mutex> lk(g_ws_mu);
    Ws &W = workspace(A, M, m, max_iters, n);
    const bool prof = prof_on();
    const bool graph_mode = use_cycle_graphs() && !prof;

    std::vector<double> hist;
    if (nonzero_x0) spmv_residual(Av, x, b, W.r.p, s);
    else vec_copy(b, W.r.p, n, s);
    norm_into(W.r.p, n, W, W.beta.p, s);
    double beta = read_scalar(W.beta.p, s);
    hist.push_back(beta);
    const double tol = std::fmax(cfg.rtol * beta, cfg.atol);
    Dev d0 = {};
    d0.m = m;
    d0.max_iters = max_iters;
    d0.tol = tol;
    PMGR_CUDA(cudaMemcpyAsync(W.dev.p, &d0, sizeof(Dev), cudaMemcpyHostToDevice, s));
    int total = 0, restarts = 0;
    bool brk = false;
    if (beta > tol) {
        if (graph_mode && !W.cycle) build_cycle_graph(Av, W);
        while (total < max_iters) {
            k_cycle_init<<<1, 256, 0, s>>>(W.dev.p, W.H.p, W.G.p, m + 1, W.cs.p, W.sn.p, W.g.p, m, W.beta.p);
            PMGR_LAUNCHED();
            k_scale2<<<vec_grid(n), 256, 0, s>>>(W.r.p, n, W.beta.p, W.V.p, W.vin.p);
            PMGR_LAUNCHED();
            if (graph_mode) {
                PMGR_CUDA(cudaGraphLaunch(W.cycle, s));
                PMGR_CUDA(cudaMemcpyAsync(W.hdev, W.dev.p, sizeof(Dev), cudaMemcpyDeviceToHost, s));
                PMGR_CUDA(cudaStreamSynchronize(s));
                g_launches.fetch_add(W.body_kernels * (W.hdev->total - total + (W.hdev->dead ? 1 : 0)),
                                     std::memory_order_relaxed);
            } else {
                while (true) {
                    PMGR_CUDA(cudaMemcpyAsync(W.hdev, W.dev.p, sizeof(Dev), cudaMemcpyDeviceToHost, s));
                    PMGR_CUDA(cudaStreamSynchronize(s));
                    if (prof && M) mgr_collect(*M);
                    if (!W.hdev->active) break;
                    arnoldi_step(Av, W, s, 0, 0);
                }
            }
            const Dev dv = *W.hdev;
            const int j = dv.j;
            const int new_total = dv.total;
            if (new_total > total) {
                std::vector<double> hh(new_total - total);
                PMGR_CUDA(cudaMemcpyAsync(hh.data(), W.hist.p + total, sizeof(double) * hh.size(),
                                          cudaMemcpyDeviceToHost, s));
                PMGR_CUDA(cudaStreamSynchronize(s));
                hist.insert(hist.end(), hh.begin(), hh.end());
            }
            total = new_total;
            brk = dv.brk != 0;
            if (j > 0) {
                k_trsv<<<1, 256, sizeof(double) * j, s>>>(W.H.p, m, j, W.g.p, W.y.p);
                PMGR_LAUNCHED();
                k_combine<<<vec_grid(n), 256, 0, s>>>(W.V.p, n, W.ldv, j, W.y.p, W.u.p);
                PMGR_LAUNCHED();
                if (M) mgr_apply(*M, W.u.p, W.z.p, s);
                else vec_copy(W.u.p, W.z.p, n, s);
                vec_axpy(1.0, W.z.p, x, n, s);
                spmv_residual(Av, x, b, W.r.p, s);
                norm_into(W.r.p, n, W, W.beta.p, s);
                beta = read_scalar(W.beta.p, s);
                if (prof && M) mgr_collect(*M);
                hist.back() = beta;
            }
            ++restarts;
            if (beta <= tol || brk) break;
        }
    }
    if (W.stamps.p && total > 0) {
        unsigned long long st[16];
        PMGR_CUDA(cudaMemcpy(st, W.stamps.p, sizeof(st), cudaMemcpyDeviceToHost));
        static const char *names[] = {"phase1", "sync1", "phase2a", "sync2", "phase2b", "phase3", "sync3",
                                      "phase4"};
        const int order[] = {0, 1, 2, 3, 4, 7, 5, 6, 8};
        fprintf(stderr, "[k_arnoldi stamps, mean over %d steps, block 0]", total);
        for (int q = 0; q + 1 < 9; ++q) {
            const int a = order[q], b2 = order[q + 1];
            fprintf(stderr, " %s=%.2fus", names[q], (double)(st[b2] - st[a]) / total / 1e3);
        }
        fprintf(stderr, "\n");
        PMGR_CUDA(cudaMemset(W.stamps.p, 0, sizeof(st)));
    }
    stats.iterations = total;
    stats.converged = beta <= tol;
    stats.restarts = restarts;
    const int32_t nh = (int32_t)hist.size();
    stats.history_len = nh < history_cap ? nh : history_cap;
    if (history)
        for (int32_t i = 0; i < stats.history_len; ++i) history[i] = hist[i];
}

// ---------------------------------------------------------------------------
// GMRES over row-distributed vectors (dist.cu supplies the operators and the
// all-reduce): the same Arnoldi kernels as the single-GPU path in split mode,
// one host synchronisation per step to read the device state.
// ---------------------------------------------------------------------------

struct SplitWs {
    int m = 0, max_iters = 0;
    int64_t n = 0, ldv = 0, chunk = 0;
    int nblk = 0, nparts = 0;
    DBuf<double> V, r, u, z, t, H, G, cs, sn, g, a, h, y, hist, pa, pg, pn, red, nrm2, beta;
    DBuf<Dev> dev;
    Dev *hdev = nullptr;
    cudaGraphExec_t exec = nullptr;  // one captured Arnoldi step
    bool captured = false;
    int64_t graph_kernels = 0;
    ~SplitWs() {
        if (exec) cudaGraphExecDestroy(exec);
        if (hdev) cudaFreeHost(hdev);
    }
};

void gmres_split(SplitOps &ops, const double *b, double *x, int nonzero_x0, const pmgr_gmres_cfg &cfg,
                 pmgr_gmres_stats &stats, double *history, int32_t history_cap, cudaStream_t s) {
    if (cfg.restart < 1) fail(PMGR_ERR_INVALID, "restart must be >= 1");
    if (cfg.restart > 1000) fail(PMGR_ERR_INVALID, "restart above 1000 is not supported");
    if (!(cfg.rtol > 0) || !(cfg.atol > 0)) fail(PMGR_ERR_INVALID, "tolerances must be positive");
    const int64_t n = ops.n;
    const int m = cfg.restart;
    const int max_iters = cfg.max_iters > 0 ? cfg.max_iters : 0;
    // workspace (and the captured step graph) persist across solves in the caller's slot
    std::shared_ptr<SplitWs> &slot = *ops.cache;
    if (!slot || slot->m != m || slot->max_iters != max_iters || slot->n != n) {
        auto w = std::make_shared<SplitWs>();
        w->m = m;
        w->max_iters = max_iters;
        w->n = n;
        w->ldv = (n + 31) / 32 * 32 + 32;
        w->nblk = 2 * num_sms();
        w->chunk = ((n + w->nblk - 1) / w->nblk + 31) / 32 * 32;
        w->nparts = 4 * num_sms();
        const int64_t ldv = w->ldv;
        w->V.alloc((int64_t)(m + 1) * ldv);
        w->r.alloc(ldv);
        w->u.alloc(ldv);
        w->z.alloc(ldv);
        w->t.alloc(ldv);
        w->H.alloc((int64_t)(m + 1) * m);
        w->G.alloc((int64_t)(m + 1) * (m + 1));
        w->cs.alloc(m + 1);
        w->sn.alloc(m + 1);
        w->g.alloc(m + 2);
        w->a.alloc(m + 1);
        w->h.alloc(m + 1);
        w->y.alloc(m + 1);
        w->hist.alloc((int64_t)max_iters + 2);
        w->pa.alloc((int64_t)(m + 1) * w->nblk);
        w->pg.alloc((int64_t)(m + 1) * w->nblk);
        w->pn.alloc(w->nparts > w->nblk ? w->nparts : w->nblk);
        w->red.alloc(2 * (int64_t)(m + 1));
        w->nrm2.alloc(1);
        w->beta.alloc(1);
        w->dev.alloc(1);
        PMGR_CUDA(cudaMallocHost((void **)&w->hdev, sizeof(Dev)));
        PMGR_CUDA(cudaMemsetAsync(w->red.p, 0, sizeof(double) * w->red.n, s));
        slot = w;
    }
    SplitWs &W = *slot;
    const int64_t ldv = W.ldv, chunk = W.chunk;
    const int nblk = W.nblk, nparts = W.nparts;
    DBuf<double> &V = W.V, &r = W.r, &u = W.u, &z = W.z, &t = W.t, &H = W.H, &G = W.G, &cs = W.cs, &sn = W.sn,
                 &g = W.g, &a = W.a, &h = W.h, &y = W.y, &hist = W.hist, &pa = W.pa, &pg = W.pg, &pn = W.pn,
                 &red = W.red, &nrm2 = W.nrm2, &beta = W.beta;
    DBuf<Dev> &dev = W.dev;
    Dev *hdev = W.hdev;

    auto gnorm = [&](const double *v, double *out) {  // out = ||v|| over all ranks
        k_norm_partial<<<nparts, DOT_BLOCK, 0, s>>>(v, n, pn.p);
        PMGR_LAUNCHED();
        k_sum_fixed<<<1, 32, 0, s>>>(pn.p, nparts, out);
        PMGR_LAUNCHED();
        ops.allreduce(out, 1, s);
        k_sqrt_inplace<<<1, 32, 0, s>>>(out);
        PMGR_LAUNCHED();
    };
    auto residual = [&]() {  // r = b - A x
        ops.spmv(x, t.p, s);
        if (n > 0) {
            k_sub<<<grid_for(n, 256), 256, 0, s>>>(b, t.p, n, r.p);
            PMGR_LAUNCHED();
        }
    };
    AoParams P = {};
    P.V = V.p;
    P.n = n;
    P.ldv = ldv;
    P.chunk = chunk;
    P.w = ops.w;
    P.vin = ops.vin;
    P.dev = dev.p;
    P.pa = pa.p;
    P.pg = pg.p;
    P.pn = pn.p;
    P.G = G.p;
    P.ldg = m + 1;
    P.a = a.p;
    P.h = h.p;
    P.H = H.p;
    P.cs = cs.p;
    P.sn = sn.p;
    P.g = g.p;
    P.hist = hist.p;
    P.red = red.p;
    P.nrm2 = nrm2.p;
    // slices in shared memory (projections read w and V_j once; the update is
    // the balanced warps-over-vectors pass) when they fit, as in the
    // single-GPU kernel; PMGR_SPLIT_SM=0 keeps the global-memory variant
    static const bool split_sm = !(getenv("PMGR_SPLIT_SM") && getenv("PMGR_SPLIT_SM")[0] == '0');
    const size_t smem = (size_t)(16 * chunk) + (size_t)AO_WARPS * 32 * AO_UM * 16;
    const bool sm = split_sm && n > 0 && chunk <= 3072;
    if (sm) {
        PMGR_CUDA(cudaFuncSetAttribute(k_arnoldi<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        PMGR_CUDA(cudaFuncSetAttribute(k_arnoldi<true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        PMGR_CUDA(cudaFuncSetAttribute(k_arnoldi<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    // (split mode: tiles of at most 1,024 rows, 16 KB next to 17 KB of static
    // shared memory -- no opt-in above 48 KB, which failed at launch from the
    // emulated ranks' threads)
    size_t smem_t = 0;
    const int split_tile = arnoldi_tile() < 1024 ? arnoldi_tile() : 1024;
    if (!sm && n > 0 && split_tile > 0 && chunk > split_tile) {
        P.tile = split_tile;
        smem_t = (size_t)16 * P.tile;
    }
    auto step = [&](cudaStream_t st) {
        ops.step(st);  // w = A M vin
        if (sm) k_arnoldi<true, 1><<<nblk, AO_THREADS, smem, st>>>(P);
        else k_arnoldi<false, 1><<<nblk, AO_THREADS, smem_t, st>>>(P);
        PMGR_LAUNCHED();
        k_arnoldi<false, 2><<<nblk, AO_THREADS, 0, st>>>(P);
        PMGR_LAUNCHED();
        ops.allreduce(red.p, 2 * (int64_t)(m + 1), st);
        k_split_fix<<<1, 256, 0, st>>>(dev.p, red.p, m + 1, a.p, G.p);
        PMGR_LAUNCHED();
        if (sm) k_arnoldi<true, 3><<<nblk, AO_THREADS, smem, st>>>(P);
        else k_arnoldi<false, 3><<<nblk, AO_THREADS, 0, st>>>(P);
        PMGR_LAUNCHED();
        k_sum_fixed<<<1, 32, 0, st>>>(pn.p, nblk, nrm2.p);
        PMGR_LAUNCHED();
        ops.allreduce(nrm2.p, 1, st);
        if (sm) k_arnoldi<true, 4><<<nblk, AO_THREADS, smem, st>>>(P);
        else k_arnoldi<false, 4><<<nblk, AO_THREADS, 0, st>>>(P);
        PMGR_LAUNCHED();
    };
    // one captured graph per step when the transport can be captured (NCCL;
    // a device-side WHILE loop around NCCL calls measured 20x slower);
    // captured once per workspace
    if (!W.captured && ops.capturable && use_cycle_graphs()) {
        W.captured = true;
        int64_t &graph_kernels = W.graph_kernels;
        cudaGraphExec_t &exec = W.exec;
        cudaStream_t cap;
        PMGR_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        cudaGraph_t graph = nullptr;
        PMGR_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        g_capture_count = &graph_kernels;
        try {
            step(cap);
        } catch (...) {
            g_capture_count = nullptr;
            cudaStreamEndCapture(cap, &graph);
            if (graph) cudaGraphDestroy(graph);
            cudaStreamDestroy(cap);
            throw;
        }
        g_capture_count = nullptr;
        PMGR_CUDA(cudaStreamEndCapture(cap, &graph));
        PMGR_CUDA(cudaGraphInstantiate(&exec, graph, 0));
        PMGR_CUDA(cudaGraphDestroy(graph));
        PMGR_CUDA(cudaStreamDestroy(cap));
    }
    cudaGraphExec_t exec = W.exec, cycle = nullptr;
    const int64_t graph_kernels = W.graph_kernels;

    std::vector<double> hl;
    if (!nonzero_x0 && n > 0) PMGR_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
    residual();
    gnorm(r.p, beta.p);
    double bt = read_scalar(beta.p, s);
    hl.push_back(bt);
    // reference krylov.py: tol = max(rtol * ||b - A x0||, atol)
    const double tol = std::fmax(cfg.rtol * bt, cfg.atol);
    Dev d0 = {};
    d0.m = m;
    d0.max_iters = max_iters;
    d0.tol = tol;
    PMGR_CUDA(cudaMemcpyAsync(dev.p, &d0, sizeof(Dev), cudaMemcpyHostToDevice, s));
    int total = 0, restarts = 0;
    bool brk = false;
    while (bt > tol && total < max_iters) {
        k_cycle_init<<<1, 256, 0, s>>>(dev.p, H.p, G.p, m + 1, cs.p, sn.p, g.p, m, beta.p);
        PMGR_LAUNCHED();
        if (n > 0) {
            k_scale2<<<vec_grid(n), 256, 0, s>>>(r.p, n, beta.p, V.p, ops.vin);
            PMGR_LAUNCHED();
        }
        if (cycle) {
            PMGR_CUDA(cudaGraphLaunch(cycle, s));
            PMGR_CUDA(cudaMemcpyAsync(hdev, dev.p, sizeof(Dev), cudaMemcpyDeviceToHost, s));
            PMGR_CUDA(cudaStreamSynchronize(s));
            g_launches.fetch_add(graph_kernels * (hdev->total - total + (hdev->dead ? 1 : 0)),
                                 std::memory_order_relaxed);
        }
        while (!cycle) {
            PMGR_CUDA(cudaMemcpyAsync(hdev, dev.p, sizeof(Dev), cudaMemcpyDeviceToHost, s));
            PMGR_CUDA(cudaStreamSynchronize(s));
            if (!hdev->active) break;
            if (exec) {
                PMGR_CUDA(cudaGraphLaunch(exec, s));
                g_launches.fetch_add(graph_kernels, std::memory_order_relaxed);
            } else {
                step(s);
            }
        }
        const Dev dv = *hdev;
        const int j = dv.j;
        if (dv.total > total) {
            std::vector<double> hh(dv.total - total);
            PMGR_CUDA(cudaMemcpyAsync(hh.data(), hist.p + total, sizeof(double) * hh.size(), cudaMemcpyDeviceToHost,
                                      s));
            PMGR_CUDA(cudaStreamSynchronize(s));
            hl.insert(hl.end(), hh.begin(), hh.end());
        }
        total = dv.total;
        brk = dv.brk != 0;
        if (j > 0) {
            k_trsv<<<1, 256, sizeof(double) * j, s>>>(H.p, m, j, g.p, y.p);
            PMGR_LAUNCHED();
            if (n > 0) {
                k_combine<<<vec_grid(n), 256, 0, s>>>(V.p, n, ldv, j, y.p, u.p);
                PMGR_LAUNCHED();
            }
            ops.apply(u.p, z.p, s);
            if (n > 0) vec_axpy(1.0, z.p, x, n, s);
            residual();
            gnorm(r.p, beta.p);
            bt = read_scalar(beta.p, s);
            hl.back() = bt;
        }
        ++restarts;
        if (bt <= tol || brk) break;
    }
    stats.iterations = total;
    stats.converged = bt <= tol;
    stats.restarts = restarts;
    const int32_t nh = (int32_t)hl.size();
    stats.history_len = history ? (nh < history_cap ? nh : history_cap) : nh;
    if (history)
        for (int32_t i = 0; i < stats.history_len; ++i) history[i] = hl[i];
}

void multidot(const double *V, int64_t n, int32_t nvec, const double *w, double *h, cudaStream_t s) {
    if (nvec <= 0) return;
    int ns = (int)((n + 8191) / 8192);
    if (ns > 64) ns = 64;
    if (ns < 1) ns = 1;
    const int64_t chunk = (n + ns - 1) / ns;
    TBuf<double> part((int64_t)nvec * ns, s);
    k_mdot_plain<<<dim3(ns, nvec), DOT_BLOCK, 0, s>>>(V, n, w, part.p, ns, chunk);
    PMGR_LAUNCHED();
    k_sum_slices<<<(nvec + 127) / 128, 128, 0, s>>>(part.p, ns, nvec, h);
    PMGR_LAUNCHED();
}

void multiaxpy(const double *V, int64_t n, int32_t nvec, const double *h, double *w, cudaStream_t s) {
    if (nvec <= 0 || nvec > 1024) fail(PMGR_ERR_INVALID, "multiaxpy supports 1..1024 vectors");
    k_maxpy<<<vec_grid(n), 256, 0, s>>>(V, n, nvec, h, w);
    PMGR_LAUNCHED();
}

namespace {
__global__ void k_axpby(double a, const double *__restrict__ x, double b, double *__restrict__ y, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = b == 0.0 ? a * x[i] : fma(b, y[i], a * x[i]);  // b = 0: y may hold garbage
}
}  // namespace

double vec_norm2(const double *x, int64_t n, cudaStream_t s) {
    const int np = vec_grid(n);
    TBuf<double> part((int64_t)np + 1, s);
    k_norm_partial<<<np, DOT_BLOCK, 0, s>>>(x, n, part.p);
    PMGR_LAUNCHED();
    k_norm_final<<<1, 32, 0, s>>>(part.p, np, part.p + np);
    PMGR_LAUNCHED();
    return read_scalar(part.p + np, s);
}

void vec_axpby(double a, const double *x, double b, double *y, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    k_axpby<<<vec_grid(n), 256, 0, s>>>(a, x, b, y, n);
    PMGR_LAUNCHED();
}

void vec_combine(const double *V, int64_t n, int64_t ldv, int32_t nvec, const double *y, double *u,
                 cudaStream_t s) {
    if (nvec < 0 || nvec > 1024) fail(PMGR_ERR_INVALID, "combine supports 0..1024 vectors");
    if (n <= 0) return;
    if (nvec == 0) {
        vec_axpby(0.0, u, 0.0, u, n, s);
        return;
    }
    k_combine<<<vec_grid(n), 256, 0, s>>>(V, n, ldv, nvec, y, u);
    PMGR_LAUNCHED();
}

}  // namespace pmgr
