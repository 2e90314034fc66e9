// tail.cu -- the coarse end of an AMG V(1,1) cycle as ONE thread-block-
// cluster kernel.
//
// Below a few thousand rows every level of the cycle (residual, restriction,
// prolongation + post-sweep; amg.py:220-231) is a latency-bound launch of a
// handful of CTAs, and the coarse levels of an elasticity hierarchy are
// dozens deep.  Here one cluster of 16 CTAs (16 SMs) walks all of them:
// phases are separated by the hardware cluster barrier (~0.2 us on
// Blackwell) instead of kernel boundaries (several us each).  The
// prolongation is folded into the post-smoothing sweep (x'_j = x_j + P_j e
// recomputed per stored entry; the tail's P rows hold 1-10 entries), so a
// level costs three barriers: residual | restriction (+ next level's first
// sweep x = b/dtilde) | ... | prolongation-and-sweep.
#include <cooperative_groups.h>

#include "hier.cuh"

namespace cg = cooperative_groups;

namespace pmgr {

namespace {

constexpr int TAIL_THREADS = 512;
constexpr int TAIL_WARPS = TAIL_THREADS / 32;

__device__ __forceinline__ double warp_sum_d(double s) {
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
    return s;
}

// r = b - A x
__device__ void phase_residual(const TailLevel &L, int gw, int nw, int lane) {
    for (int i = gw; i < L.n; i += nw) {
        double s = 0.0;
        for (int64_t q = L.ro[i] + lane; q < L.ro[i + 1]; q += 32) s = fma(L.v[q], L.x[L.ci[q]], s);
        s = warp_sum_d(s);
        if (lane == 0) L.r[i] = L.b[i] - s;
    }
}

// b_next = R r ; x_next = b_next / dtilde_next (next level smoothed) ;
// or cb = R r at the coarsest
__device__ void phase_restrict(const TailLevel &L, double *bn, double *xn, const double *dn, int nn, int gw,
                               int nw, int lane) {
    for (int k = gw; k < nn; k += nw) {
        double s = 0.0;
        for (int64_t q = L.Rro[k] + lane; q < L.Rro[k + 1]; q += 32) s = fma(L.Rv[q], L.r[L.Rci[q]], s);
        s = warp_sum_d(s);
        if (lane == 0) {
            bn[k] = s;
            if (xn) xn[k] = s / dn[k];
        }
    }
}

__device__ __forceinline__ double prolonged(const TailLevel &L, const double *e, int j) {
    double t = L.x[j];
    for (int64_t p = L.Pro[j]; p < L.Pro[j + 1]; ++p) t = fma(L.Pv[p], e[L.Pci[p]], t);
    return t;
}

// out = x' + (b - A x') / dtilde with x' = x + P e
__device__ void phase_up(const TailLevel &L, const double *e, double *out, int gw, int nw, int lane) {
    for (int i = gw; i < L.n; i += nw) {
        double s = 0.0;
        for (int64_t q = L.ro[i] + lane; q < L.ro[i + 1]; q += 32) s = fma(L.v[q], prolonged(L, e, L.ci[q]), s);
        s = warp_sum_d(s);
        if (lane == 0) {
            const double xi = prolonged(L, e, i);
            out[i] = xi + (L.b[i] - s) / L.dt[i];
        }
    }
}

__global__ void __launch_bounds__(TAIL_THREADS) k_tail(const TailParams *__restrict__ pp) {
    const TailParams &P = *pp;
    cg::cluster_group cl = cg::this_cluster();
    const int lane = threadIdx.x & 31;
    const int gw = (int)cl.block_rank() * TAIL_WARPS + (threadIdx.x >> 5);
    const int nw = (int)cl.num_blocks() * TAIL_WARPS;
    // down: residual, restriction
    for (int l = 0; l < P.nlev; ++l) {
        const TailLevel &L = P.lev[l];
        phase_residual(L, gw, nw, lane);
        cl.sync();
        if (l + 1 < P.nlev) {
            const TailLevel &N = P.lev[l + 1];
            phase_restrict(L, N.b, N.x, N.dt, N.n, gw, nw, lane);
        } else {
            phase_restrict(L, P.cb, nullptr, nullptr, P.nc, gw, nw, lane);
        }
        cl.sync();
    }
    // coarsest: cx = C^{-1} cb (dense, warp per row)
    for (int i = gw; i < P.nc; i += nw) {
        double s = 0.0;
        for (int j = lane; j < P.nc; j += 32) s = fma(P.cinv[(int64_t)i * P.nc + j], P.cb[j], s);
        s = warp_sum_d(s);
        if (lane == 0) P.cx[i] = s;
    }
    cl.sync();
    // up: prolongation folded into the post-sweep
    for (int l = P.nlev - 1; l >= 0; --l) {
        const TailLevel &L = P.lev[l];
        const double *e = (l + 1 < P.nlev) ? P.lev[l + 1].xo : P.cx;
        phase_up(L, e, l == 0 ? P.out : L.xo, gw, nw, lane);
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

bool tail_qualifies(const Csr &A) { return A.nrows <= 16384 && A.nnz <= 600000; }

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
