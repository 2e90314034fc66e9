// Microbenchmark for the Arnoldi projection phase (phase 1 of k_arnoldi):
// slice partials of V_k.w and V_k.V_j for k <= j over a 173,347-row basis.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bp1 tools/bench_phase1.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// (a) current: warp per vector, 8 scalar rows per lane per round, w/vj from smem
template <int T>
__global__ void __launch_bounds__(T) k_a(const double *V, const double *w, int64_t n, int64_t ldv, int j, int64_t chunk,
                                         double *pa, double *pg) {
    extern __shared__ double sl[];
    const int nblk = gridDim.x, b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t lo = (int64_t)b * chunk, hi = lo + chunk < n ? lo + chunk : n;
    const double *vjg = V + (int64_t)j * ldv;
    double *wsl = sl, *vsl = sl + chunk;
    for (int64_t i = lo + threadIdx.x; i < hi; i += T) {
        wsl[i - lo] = w[i];
        vsl[i - lo] = vjg[i];
    }
    __syncthreads();
    for (int k = warp; k <= j; k += T / 32) {
        const double *x = V + (int64_t)k * ldv;
        double aa[8], gg[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) aa[u] = gg[u] = 0.0;
        int64_t i = lo + lane;
        for (; i + 7 * 32 < hi; i += 8 * 32) {
            double xs[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) xs[u] = x[i + 32 * u];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                aa[u] = fma(xs[u], wsl[i + 32 * u - lo], aa[u]);
                gg[u] = fma(xs[u], vsl[i + 32 * u - lo], gg[u]);
            }
        }
        for (; i < hi; i += 32) {
            aa[0] = fma(x[i], wsl[i - lo], aa[0]);
            gg[0] = fma(x[i], vsl[i - lo], gg[0]);
        }
        const double sa = warp_sum(((aa[0] + aa[1]) + (aa[2] + aa[3])) + ((aa[4] + aa[5]) + (aa[6] + aa[7])));
        const double sg = warp_sum(((gg[0] + gg[1]) + (gg[2] + gg[3])) + ((gg[4] + gg[5]) + (gg[6] + gg[7])));
        if (lane == 0) {
            pa[(int64_t)k * nblk + b] = sa;
            pg[(int64_t)k * nblk + b] = sg;
        }
    }
}

// (b) double2 loads, U double2 per lane per round
template <int T, int U>
__global__ void __launch_bounds__(T) k_b(const double *V, const double *w, int64_t n, int64_t ldv, int j, int64_t chunk,
                                         double *pa, double *pg) {
    extern __shared__ double sl[];
    const int nblk = gridDim.x, b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t lo = (int64_t)b * chunk, hi = lo + chunk < n ? lo + chunk : n;
    const double *vjg = V + (int64_t)j * ldv;
    double *wsl = sl, *vsl = sl + chunk;
    for (int64_t i = lo + threadIdx.x; i < hi; i += T) {
        wsl[i - lo] = w[i];
        vsl[i - lo] = vjg[i];
    }
    __syncthreads();
    const int64_t len = hi - lo;
    const int64_t len2 = len / 2;  // ldv and chunk are multiples of 32: every slice is 16B aligned
    for (int k = warp; k <= j; k += T / 32) {
        const double *x = V + (int64_t)k * ldv + lo;
        const double2 *x2 = reinterpret_cast<const double2 *>(x);
        const double2 *w2 = reinterpret_cast<const double2 *>(wsl);
        const double2 *v2 = reinterpret_cast<const double2 *>(vsl);
        double a0 = 0, a1 = 0, g0 = 0, g1 = 0;
        int64_t p = lane;
        for (; p + (U - 1) * 32 < len2; p += U * 32) {
            double2 xs[U];
#pragma unroll
            for (int u = 0; u < U; ++u) xs[u] = __ldcs(x2 + p + 32 * u);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double2 ww = w2[p + 32 * u], vv = v2[p + 32 * u];
                a0 = fma(xs[u].x, ww.x, a0);
                a1 = fma(xs[u].y, ww.y, a1);
                g0 = fma(xs[u].x, vv.x, g0);
                g1 = fma(xs[u].y, vv.y, g1);
            }
        }
        for (; p < len2; p += 32) {
            const double2 xx = x2[p], ww = w2[p], vv = v2[p];
            a0 = fma(xx.x, ww.x, a0);
            a1 = fma(xx.y, ww.y, a1);
            g0 = fma(xx.x, vv.x, g0);
            g1 = fma(xx.y, vv.y, g1);
        }
        for (int64_t i = 2 * len2 + lane; i < len; i += 32) {
            a0 = fma(x[i], wsl[i], a0);
            g0 = fma(x[i], vsl[i], g0);
        }
        const double sa = warp_sum(a0 + a1), sg = warp_sum(g0 + g1);
        if (lane == 0) {
            pa[(int64_t)k * nblk + b] = sa;
            pg[(int64_t)k * nblk + b] = sg;
        }
    }
}

// (c) block-cooperative: all threads over rows, 4 vectors at a time, smem reduction
template <int T, int KV>
__global__ void __launch_bounds__(T) k_c(const double *V, const double *w, int64_t n, int64_t ldv, int j, int64_t chunk,
                                         double *pa, double *pg) {
    extern __shared__ double sl[];
    __shared__ double red[T / 32][2 * KV];
    const int nblk = gridDim.x, b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t lo = (int64_t)b * chunk, hi = lo + chunk < n ? lo + chunk : n;
    const double *vjg = V + (int64_t)j * ldv;
    double wr[4], vr[4];
    int cnt = 0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += T, ++cnt) {
        wr[cnt] = w[i];
        vr[cnt] = vjg[i];
    }
    for (int k0 = 0; k0 <= j; k0 += KV) {
        double xs[KV][4];
#pragma unroll
        for (int q = 0; q < KV; ++q)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int64_t i = lo + threadIdx.x + (int64_t)c * T;
                xs[q][c] = (k0 + q <= j && i < hi) ? __ldcs(V + (int64_t)(k0 + q) * ldv + i) : 0.0;
            }
        double sa[KV], sg[KV];
#pragma unroll
        for (int q = 0; q < KV; ++q) {
            sa[q] = sg[q] = 0.0;
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (c < cnt) {
                    sa[q] = fma(xs[q][c], wr[c], sa[q]);
                    sg[q] = fma(xs[q][c], vr[c], sg[q]);
                }
            sa[q] = warp_sum(sa[q]);
            sg[q] = warp_sum(sg[q]);
        }
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < KV; ++q) {
                red[warp][2 * q] = sa[q];
                red[warp][2 * q + 1] = sg[q];
            }
        __syncthreads();
        if (threadIdx.x < 2 * KV) {
            double t = 0;
            for (int ww = 0; ww < T / 32; ++ww) t += red[ww][threadIdx.x];
            const int q = threadIdx.x >> 1;
            if (k0 + q <= j) ((threadIdx.x & 1) ? pg : pa)[(int64_t)(k0 + q) * nblk + b] = t;
        }
        __syncthreads();
    }
}

// (d) whole slice per vector in one predicated batch, PV vectors per warp batch
template <int T, int UM, int PV>
__global__ void __launch_bounds__(T) k_d(const double *V, const double *w, int64_t n, int64_t ldv, int j, int64_t chunk,
                                         double *pa, double *pg) {
    extern __shared__ double sl[];
    const int nblk = gridDim.x, b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t lo = (int64_t)b * chunk, hi = lo + chunk < n ? lo + chunk : n;
    const double *vjg = V + (int64_t)j * ldv;
    double *wsl = sl, *vsl = sl + chunk;
    for (int64_t i = lo + threadIdx.x; i < hi; i += T) {
        wsl[i - lo] = w[i];
        vsl[i - lo] = vjg[i];
    }
    __syncthreads();
    const int len = hi > lo ? (int)(hi - lo) : 0, len2 = len / 2;
    const double2 *w2 = reinterpret_cast<const double2 *>(wsl);
    const double2 *v2 = reinterpret_cast<const double2 *>(vsl);
    for (int k = warp * PV; k <= j; k += (T / 32) * PV) {
        double2 xs[PV][UM];
#pragma unroll
        for (int q = 0; q < PV; ++q) {
            const double2 *x2 = reinterpret_cast<const double2 *>(V + (int64_t)(k + q) * ldv + lo);
#pragma unroll
            for (int u = 0; u < UM; ++u) {
                const int p = lane + 32 * u;
                xs[q][u] = (k + q <= j && p < len2) ? __ldcs(x2 + p) : make_double2(0.0, 0.0);
            }
        }
#pragma unroll
        for (int q = 0; q < PV; ++q) {
            double a0 = 0, a1 = 0, g0 = 0, g1 = 0;
#pragma unroll
            for (int u = 0; u < UM; ++u) {
                const int p = lane + 32 * u;
                if (p < len2) {
                    const double2 ww = w2[p], vv = v2[p];
                    a0 = fma(xs[q][u].x, ww.x, a0);
                    a1 = fma(xs[q][u].y, ww.y, a1);
                    g0 = fma(xs[q][u].x, vv.x, g0);
                    g1 = fma(xs[q][u].y, vv.y, g1);
                }
            }
            if ((len & 1) && lane == 0 && k + q <= j) {
                const double xl = V[(int64_t)(k + q) * ldv + lo + len - 1];
                a0 = fma(xl, wsl[len - 1], a0);
                g0 = fma(xl, vsl[len - 1], g0);
            }
            const double sa = warp_sum(a0 + a1), sg = warp_sum(g0 + g1);
            if (lane == 0 && k + q <= j) {
                pa[(int64_t)(k + q) * nblk + b] = sa;
                pg[(int64_t)(k + q) * nblk + b] = sg;
            }
        }
    }
}

int main() {
    const int64_t n = 173347;
    const int m = 100;
    const int64_t ldv = (n + 31) / 32 * 32;
    double *V, *w, *pa, *pg, *flush;
    CK(cudaMalloc(&V, (m + 1) * ldv * 8));
    CK(cudaMalloc(&w, n * 8));
    CK(cudaMalloc(&pa, (m + 1) * 2048 * 8));
    CK(cudaMalloc(&pg, (m + 1) * 2048 * 8));
    CK(cudaMalloc(&flush, 512 << 20));
    CK(cudaMemset(V, 0, (m + 1) * ldv * 8));
    CK(cudaMemset(w, 0, n * 8));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto run = [&](const char *name, auto launch) {
        for (int j : {15, 46, 91}) {
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                CK(cudaMemsetAsync(flush, rep, 512 << 20));
                CK(cudaEventRecord(e0));
                launch(j);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                best = ms < best ? ms : best;
            }
            CK(cudaGetLastError());
            const double bytes = 8.0 * n * (j + 1);
            printf("%-28s j=%3d  %7.2f us  %7.0f GB/s\n", name, j, best * 1e3, bytes / (best * 1e-3) / 1e9);
        }
    };
    for (int bps : {1, 2, 3}) {
        const int nblk = bps * sms;
        const int64_t chunk = ((n + nblk - 1) / nblk + 31) / 32 * 32;
        const size_t smem = 16 * chunk;
        char nm[64];
        snprintf(nm, 64, "a bps=%d T=512", bps);
        if (bps <= 2) run(nm, [&](int j) { k_a<512><<<nblk, 512, smem>>>(V, w, n, ldv, j, chunk, pa, pg); });
        snprintf(nm, 64, "a bps=%d T=256", bps);
        run(nm, [&](int j) { k_a<256><<<nblk, 256, smem>>>(V, w, n, ldv, j, chunk, pa, pg); });
        snprintf(nm, 64, "b4 bps=%d T=512", bps);
        if (bps <= 2) run(nm, [&](int j) { k_b<512, 4><<<nblk, 512, smem>>>(V, w, n, ldv, j, chunk, pa, pg); });
        snprintf(nm, 64, "b8 bps=%d T=512", bps);
        if (bps <= 2) run(nm, [&](int j) { k_b<512, 8><<<nblk, 512, smem>>>(V, w, n, ldv, j, chunk, pa, pg); });
        snprintf(nm, 64, "b4 bps=%d T=256", bps);
        run(nm, [&](int j) { k_b<256, 4><<<nblk, 256, smem>>>(V, w, n, ldv, j, chunk, pa, pg); });
        snprintf(nm, 64, "c4 bps=%d T=512", bps);
        if (bps <= 2 && chunk <= 4 * 512)
            run(nm, [&](int j) { k_c<512, 4><<<nblk, 512, 0>>>(V, w, n, ldv, j, chunk, pa, pg); });
        snprintf(nm, 64, "c8 bps=%d T=512", bps);
        if (bps <= 2 && chunk <= 4 * 512)
            run(nm, [&](int j) { k_c<512, 8><<<nblk, 512, 0>>>(V, w, n, ldv, j, chunk, pa, pg); });
    }
    for (int bps : {2, 3, 4}) {
        for (int T : {256, 512}) {
            if (T * bps > 2048) continue;
            const int nblk = bps * sms;
            const int64_t chunk = ((n + nblk - 1) / nblk + 31) / 32 * 32;
            const size_t smem = 16 * chunk;
            const int um = (int)((chunk / 2 + 31) / 32);
            char nm[64];
            for (int pv : {1, 2}) {
                snprintf(nm, 64, "d bps=%d T=%d UM=%d PV=%d", bps, T, um, pv);
#define DV(TT, U, P) if (T == TT && um == U && pv == P) run(nm, [&](int j) { k_d<TT, U, P><<<nblk, TT, smem>>>(V, w, n, ldv, j, chunk, pa, pg); });
                DV(256, 3, 1) DV(256, 3, 2) DV(256, 4, 1) DV(256, 4, 2) DV(256, 5, 1) DV(256, 5, 2) DV(256, 6, 1) DV(256, 6, 2)
                DV(256, 10, 1) DV(256, 10, 2) DV(512, 10, 1) DV(512, 10, 2) DV(512, 5, 1) DV(512, 5, 2) DV(512, 4, 1) DV(512, 4, 2)
                DV(512, 3, 1) DV(512, 3, 2) DV(512, 6, 1) DV(512, 6, 2) DV(512, 7, 1) DV(512, 7, 2) DV(256, 7, 1) DV(256, 7, 2)
            }
        }
    }
    // plain streaming read bandwidth for reference
    return 0;
}
