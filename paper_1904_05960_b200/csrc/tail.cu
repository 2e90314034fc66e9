// tail.cu -- the coarse end of an AMG V(1,1) cycle as ONE thread-block-
// cluster kernel.
//
// Below a few thousand rows every level of the cycle (residual, restriction,
// prolongation + post-sweep; amg.py:220-231) is a latency-bound launch of a
// handful of CTAs, and the coarse levels of an elasticity hierarchy are
// dozens deep.  Here one cluster of 16 CTAs (16 SMs) walks all of them:
// phases are separated by the hardware cluster barrier (~0.2 us on
// Blackwell) instead of kernel boundaries (several us each).  A level costs
// four barriers: residual | restriction (+ the next level's first sweep
// x = b/dtilde) | ... | prolongation | post-sweep.  Rows are spread over all
// 16K threads of the cluster in lane groups sized to the level's row length.
#include <cooperative_groups.h>

#include "hier.cuh"

namespace cg = cooperative_groups;

namespace pmgr {

namespace {

constexpr int TAIL_THREADS = 1024;

constexpr int TAIL_U = 8;  // entries prefetched per lane before the gathers

template <class Fx, class Fout>
__device__ __forceinline__ void rows_spmv(int n, const int64_t *__restrict__ ro, const int32_t *__restrict__ ci,
                                          const double *__restrict__ v, int G, int gt, int nt, Fx xval, Fout out) {
    // gt / nt: global thread index / count over the cluster; G lanes per row
    const int lane = gt & (G - 1);
    const int ng = nt / G;
    const int wbase = (gt & ~31) / G;  // first row of this warp: warp-uniform trip count
    for (int it = 0; wbase + it * ng < n; ++it) {
        const int i = gt / G + it * ng;
        const bool act = i < n;
        int64_t b = 0, e = 0;
        if (act) {
            b = __ldg(ro + i);
            e = __ldg(ro + i + 1);
        }
        double s = 0.0;
        for (int64_t q = b + lane; q < e; q += TAIL_U * G) {
            double vv[TAIL_U];
            int cc[TAIL_U];
#pragma unroll
            for (int u = 0; u < TAIL_U; ++u) {
                const int64_t k = q + (int64_t)u * G;
                vv[u] = k < e ? __ldg(v + k) : 0.0;
                cc[u] = k < e ? __ldg(ci + k) : -1;
            }
#pragma unroll
            for (int u = 0; u < TAIL_U; ++u)
                if (cc[u] >= 0) s = fma(vv[u], xval(cc[u]), s);
        }
        for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o, G);
        if (act && lane == 0) out(i, s);
    }
}

__global__ void __launch_bounds__(TAIL_THREADS) k_tail(const TailParams *__restrict__ pp) {
    const TailParams &P = *pp;
    cg::cluster_group cl = cg::this_cluster();
    const int nt = (int)cl.num_blocks() * TAIL_THREADS;
    const int gt = (int)cl.block_rank() * TAIL_THREADS + threadIdx.x;
    // down: residual | restriction (+ first sweep of the next level)
    for (int l = 0; l < P.nlev; ++l) {
        const TailLevel &L = P.lev[l];
        const int G = L.gA;
        const double *x = L.x;
        const double *b = L.b;
        double *r = L.r;
        rows_spmv(L.n, L.ro, L.ci, L.v, G, gt, nt, [=](int j) { return x[j]; },
                  [=](int i, double s) { r[i] = b[i] - s; });
        cl.sync();
        const int nn = (l + 1 < P.nlev) ? P.lev[l + 1].n : P.nc;
        const int GR = L.gR;
        if (l + 1 < P.nlev) {
            const TailLevel &N = P.lev[l + 1];
            double *bn = N.b, *xn = N.x;
            const double *dn = N.dt;
            rows_spmv(nn, L.Rro, L.Rci, L.Rv, GR, gt, nt, [=](int j) { return r[j]; }, [=](int k, double s) {
                bn[k] = s;
                xn[k] = s / dn[k];
            });
        } else {
            double *cb = P.cb;
            rows_spmv(nn, L.Rro, L.Rci, L.Rv, GR, gt, nt, [=](int j) { return r[j]; },
                      [=](int k, double s) { cb[k] = s; });
        }
        cl.sync();
    }
    // coarsest: cx = C^{-1} cb (dense rows, a warp per row)
    {
        const int lane = threadIdx.x & 31;
        const int gw = gt >> 5, nw = nt >> 5;
        for (int i = gw; i < P.nc; i += nw) {
            double s = 0.0;
            for (int j = lane; j < P.nc; j += 32) s = fma(__ldg(P.cinv + (int64_t)i * P.nc + j), P.cb[j], s);
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
            if (lane == 0) P.cx[i] = s;
        }
    }
    cl.sync();
    // up: prolongation | post-sweep
    for (int l = P.nlev - 1; l >= 0; --l) {
        const TailLevel &L = P.lev[l];
        const double *e = (l + 1 < P.nlev) ? P.lev[l + 1].xo : P.cx;
        double *x = L.x;
        rows_spmv(L.n, L.Pro, L.Pci, L.Pv, L.gP, gt, nt, [=](int j) { return e[j]; },
                  [=](int i, double s) { x[i] += s; });
        cl.sync();
        const double *b = L.b, *dt = L.dt;
        double *out = (l == 0) ? P.out : L.xo;
        rows_spmv(L.n, L.ro, L.ci, L.v, L.gA, gt, nt, [=](int j) { return x[j]; },
                  [=](int i, double s) { out[i] = x[i] + (b[i] - s) / dt[i]; });
        if (l > 0) cl.sync();
    }
}

int g_cluster = 0;

int cluster_size() {
    if (!g_cluster) {
        PMGR_CUDA(cudaFuncSetAttribute(k_tail, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(TAIL_THREADS);
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = 16;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_tail, &cfg) == cudaSuccess && n > 0) {
            g_cluster = 16;
        } else {
            cudaGetLastError();
            g_cluster = 8;
        }
    }
    return g_cluster;
}

}  // namespace

bool tail_qualifies(const Csr &A) { return A.nrows <= 2048 && A.nnz <= 200000; }

int tail_group(const Csr &A) {
    const double mean = A.nrows ? (double)A.nnz / (double)A.nrows : 0.0;
    int g = mean <= 3 ? 2 : mean <= 12 ? 4 : mean <= 48 ? 8 : mean <= 160 ? 16 : 32;
    if (A.maxrow > (int64_t)TAIL_U * g) g = 32;  // a dense row must not serialise its group
    while (g > 2 && A.nrows * g > 4 * 16 * 1024) g >>= 1;
    return g;
}

void tail_launch(const TailParams *dev_params, cudaStream_t s) {
    const int cs = cluster_size();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(TAIL_THREADS);
    cfg.stream = s;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cs;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    PMGR_CUDA(cudaLaunchKernelEx(&cfg, k_tail, dev_params));
    PMGR_LAUNCHED();
}

}  // namespace pmgr
