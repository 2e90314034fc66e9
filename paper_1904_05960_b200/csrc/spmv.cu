// spmv.cu -- fp64 CSR SpMV family and the fused smoother / transfer kernels
// of the solve phase.
//
// One kernel template, k_spmv<G, Op>: a group of G lanes per row walks the
// row's (value, column) pairs with coalesced loads, gathers x through the
// read-only path, reduces with shuffles and hands the row sum to an epilogue
// functor.  The functors fuse what the reference does as separate numpy
// passes around scipy's csr_matvec (sparse.py:261-266):
//   OpY            y = A x                                  (matvec)
//   OpResidual     r = b - A x                              (amg.py:227, mgr.py:421)
//   OpJacobi       x' = x + (b - A x) / dtilde              (l1_gs_kernel, n partitions)
//   OpSweep0       x = b / dtilde ; r = b - A x  (first sweep from x = 0, fused)
//   OpAdd          x += P e                                 (amg.py:230)
//   OpResidRows    r_C = v_C - A_CF z_F                     (mgr.py:419-422, C rows only)
//   OpProlong      z = [z_F ; 0] + P e_C                    (mgr.py:424-425)
// The solve phase only needs 1e-10 agreement, so these use FMA.
#include <cstdlib>

#include "common.cuh"

namespace pmgr {

namespace {

template <bool STREAM>
__device__ __forceinline__ double ldv(const double *p) {
    return STREAM ? __ldcs(p) : __ldg(p);
}
template <bool STREAM>
__device__ __forceinline__ int ldc(const int32_t *p) {
    return STREAM ? __ldcs(p) : __ldg(p);
}
template <bool STREAM>
__device__ __forceinline__ int ldc(const uint16_t *p) {
    return (int)(STREAM ? __ldcs(reinterpret_cast<const unsigned short *>(p))
                        : __ldg(reinterpret_cast<const unsigned short *>(p)));
}

template <int G, bool STREAM, class Op, class IT, int U = 2>
__global__ void __launch_bounds__(256) k_spmv(int64_t nrows, const int64_t *__restrict__ ro,
                                              const IT *__restrict__ ci,
                                              const double *__restrict__ v, Op op, int64_t row_off, int trigger,
                                              int64_t long_len, const int32_t *__restrict__ lrows,
                                              unsigned nshort) {
    // The operator is constant during the solve: its row bounds (and, in the
    // short-row path, the first two entries per lane) are loaded before
    // griddepcontrol.wait, overlapping the predecessor's tail; only the
    // gathers of x and the epilogue wait for it.
    if (blockIdx.x >= nshort) {
        // a long row: the whole block, four independent load chains per
        // thread, then a fixed-order reduction (warps, then the 8 warp sums)
        __shared__ double ws[8];
        const int64_t row = __ldg(lrows + (blockIdx.x - nshort));
        const int64_t b = __ldg(ro + row), e = __ldg(ro + row + 1);
        if (threadIdx.x == 0) op.pre(row + row_off);
        pdl_wait();
        if (trigger) pdl_trigger();
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int64_t q = b + threadIdx.x;
        for (; q + 768 < e; q += 1024) {
            const double v0 = ldv<STREAM>(v + q), v1 = ldv<STREAM>(v + q + 256), v2 = ldv<STREAM>(v + q + 512),
                         v3 = ldv<STREAM>(v + q + 768);
            const int c0 = ldc<STREAM>(ci + q), c1 = ldc<STREAM>(ci + q + 256), c2 = ldc<STREAM>(ci + q + 512),
                      c3 = ldc<STREAM>(ci + q + 768);
            s0 = fma(v0, op.x(c0), s0);
            s1 = fma(v1, op.x(c1), s1);
            s2 = fma(v2, op.x(c2), s2);
            s3 = fma(v3, op.x(c3), s3);
        }
        for (; q < e; q += 256) s0 = fma(ldv<STREAM>(v + q), op.x(ldc<STREAM>(ci + q)), s0);
        double s = (s0 + s1) + (s2 + s3);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o);
        if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) t += ws[w];
            op.out(row + row_off, t);
        }
        return;
    }
    const int lane = threadIdx.x & (G - 1);
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    bool active = row < nrows;
    int64_t b = 0, e = 0;
    if (active) {
        b = __ldg(ro + row);
        e = __ldg(ro + row + 1);
        if (long_len > 0 && e - b > long_len) {  // summed by its own block
            active = false;
            e = b;
        }
    }
    // U independent accumulators keep U (value, column, x) load chains in
    // flight per lane (U = 4 for the long-row lane groups); the first U
    // entries per lane are loaded before the wait, and every later round
    // issues its U predicated loads at once, so a row of up to U G entries
    // costs one gather round trip after the wait
    int64_t q = b + lane;
    double vv[U];
    int cc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const bool h = q + u * G < e;
        vv[u] = h ? ldv<STREAM>(v + q + u * G) : 0.0;
        cc[u] = h ? ldc<STREAM>(ci + q + u * G) : -1;
    }
    if (active && lane == 0) op.pre(row + row_off);
    pdl_wait();
    if (trigger) pdl_trigger();
    double sa[U];
#pragma unroll
    for (int u = 0; u < U; ++u) sa[u] = cc[u] >= 0 ? fma(vv[u], op.x(cc[u]), 0.0) : 0.0;
    for (q += U * G; q < e; q += U * G) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool h = q + u * G < e;
            vv[u] = h ? ldv<STREAM>(v + q + u * G) : 0.0;
            cc[u] = h ? ldc<STREAM>(ci + q + u * G) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (cc[u] >= 0) sa[u] = fma(vv[u], op.x(cc[u]), sa[u]);
    }
    double s0 = sa[0], s1 = sa[1];
    if constexpr (U == 4) {
        s0 += sa[2];
        s1 += sa[3];
    }
    double s = s0 + s1;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(FULL, s, o, G);
    if (active && lane == 0) op.out(row + row_off, s);
}

// Software-pipelined CSR SpMV (G lanes per row, U entries per lane in
// flight): a resident grid of lane groups strides over the rows; the next
// row's bounds are fetched two rows ahead and its first U G entries are
// issued before the current row's gathers are consumed.  Per-row arithmetic
// is exactly k_spmv<G, ..., U>'s (same lanes, accumulators and reduction).
template <int G, int U, class Op, class IT, int MINB>
__global__ void __launch_bounds__(256, MINB) k_spmv_pipe(int64_t nrows, const int64_t *__restrict__ ro,
                                                         const IT *__restrict__ ci, const double *__restrict__ v,
                                                         Op op, int64_t row_off, int trigger) {
    const int lane = threadIdx.x & (G - 1);
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x / G);
    int64_t I = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
    int64_t b0 = 0, e0 = 0, nb = 0, ne = 0;
    if (I < nrows) {
        b0 = __ldg(ro + I);
        e0 = __ldg(ro + I + 1);
    }
    double vv[U];
    int cc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int64_t q = b0 + lane + G * u;
        const bool h = q < e0;
        vv[u] = h ? __ldg(v + q) : 0.0;
        cc[u] = h ? ldc<false>(ci + q) : -1;
    }
    if (I + nw < nrows) {
        nb = __ldg(ro + I + nw);
        ne = __ldg(ro + I + nw + 1);
    }
    pdl_wait();
    if (trigger) pdl_trigger();
    // every lane of a warp runs the same number of iterations (the shuffles
    // need the whole warp): the loop bound is the warp's first row group's
    const int64_t warp_first = ((blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) / G);
    for (int64_t Iw = warp_first; Iw < nrows; Iw += nw, I += nw) {
        double xs[U];
#pragma unroll
        for (int u = 0; u < U; ++u) xs[u] = cc[u] >= 0 ? op.x(cc[u]) : 0.0;
        double nvv[U];
        int ncc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t q = nb + lane + G * u;
            const bool h = q < ne;
            nvv[u] = h ? __ldg(v + q) : 0.0;
            ncc[u] = h ? ldc<false>(ci + q) : -1;
        }
        const int64_t cb = b0, ce = e0;
        b0 = nb;
        e0 = ne;
        nb = ne = 0;
        if (I + 2 * nw < nrows) {
            nb = __ldg(ro + I + 2 * nw);
            ne = __ldg(ro + I + 2 * nw + 1);
        }
        double sa[U];
#pragma unroll
        for (int u = 0; u < U; ++u) sa[u] = cc[u] >= 0 ? fma(vv[u], xs[u], 0.0) : 0.0;
        for (int64_t q = cb + lane + U * G; q < ce; q += U * G) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool h = q + G * u < ce;
                vv[u] = h ? __ldg(v + q + G * u) : 0.0;
                cc[u] = h ? ldc<false>(ci + q + G * u) : -1;
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (cc[u] >= 0) sa[u] = fma(vv[u], op.x(cc[u]), sa[u]);
        }
        double s0 = sa[0], s1 = sa[1];
        if constexpr (U == 4) {
            s0 += sa[2];
            s1 += sa[3];
        }
        double t = s0 + s1;
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o, G);
        if (lane == 0 && I < nrows) {
            Op o = op;
            o.pre(I + row_off);
            o.out(I + row_off, t);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            vv[u] = nvv[u];
            cc[u] = ncc[u];
        }
    }
}

// rows past the block prefix (A0's flow rows): 8 lanes per row, four entries
// per lane in flight, for the blocks from tail_blk0 on (k_bsr3, k_bsr3p)
template <bool STREAM, class Op>
__device__ __forceinline__ void bsr3_tail_rows(int64_t nb, int64_t n, const int64_t *__restrict__ rro,
                                               const int32_t *__restrict__ rci, const double *__restrict__ rv,
                                               Op op, int64_t row_off, int trigger, unsigned tail_blk0) {
    const int gl = threadIdx.x & 7;
    const int64_t row = 3 * nb + ((int64_t)(blockIdx.x - tail_blk0) * blockDim.x + threadIdx.x) / 8;
    const bool act = row < n;
    int64_t q = 0, e = 0;
    if (act) {
        q = __ldg(rro + row) + gl;
        e = __ldg(rro + row + 1);
    }
    double vv[4];
    int cc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const bool h = q + 8 * u < e;
        vv[u] = h ? ldv<STREAM>(rv + q + 8 * u) : 0.0;
        cc[u] = h ? ldc<STREAM>(rci + q + 8 * u) : -1;
    }
    if (act && gl == 0) op.pre(row + row_off);
    pdl_wait();
    if (trigger) pdl_trigger();
    double sa[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) sa[u] = cc[u] >= 0 ? fma(vv[u], op.x(cc[u]), 0.0) : 0.0;
    for (q += 32; q < e; q += 32) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const bool h = q + 8 * u < e;
            vv[u] = h ? ldv<STREAM>(rv + q + 8 * u) : 0.0;
            cc[u] = h ? ldc<STREAM>(rci + q + 8 * u) : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (cc[u] >= 0) sa[u] = fma(vv[u], op.x(cc[u]), sa[u]);
    }
    double t = (sa[0] + sa[2]) + (sa[1] + sa[3]);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o, 8);
    if (act && gl == 0) op.out(row + row_off, t);
}

// Block-prefix SpMV: a warp per row triple.  Triples inside the node-blocked
// prefix stream their 3x3 blocks: lane 3k+c (k < 10) owns column c of every
// 10th block -- one column index, one x gather and three values feeding the
// three row sums, 76 B per 9 entries instead of CSR's 108 B (blocks stored
// column-major).  Remainder entries (coupling columns, rows past the
// prefix) are read as CSR by three 10-lane groups, one per row.
//
// tail_blk0 < gridDim.x: the rows past the prefix (A0's flow rows, no blocks)
// are summed by the blocks from tail_blk0 on, 8 lanes per row with four
// entries per lane in flight, instead of by 10-lane groups of row triples.
template <class Op, bool STREAM = false, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_bsr3(int64_t ntrip, int64_t nb, int64_t n, const int64_t *__restrict__ bro,
                                              const int32_t *__restrict__ bci, const double *__restrict__ bval,
                                              const int64_t *__restrict__ rro, const int32_t *__restrict__ rci,
                                              const double *__restrict__ rv, Op op, int64_t row_off, int trigger,
                                              unsigned tail_blk0 = 0xffffffffu) {
    if (blockIdx.x >= tail_blk0) {
        bsr3_tail_rows<STREAM>(nb, n, rro, rci, rv, op, row_off, trigger, tail_blk0);
        return;
    }
    const int64_t I = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int kk = lane / 3, c = lane - 3 * kk;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    // the row bounds do not depend on the predecessor: loaded before the wait
    int64_t k0 = 0, k1 = 0;
    if (I < nb) {
        k0 = __ldg(bro + I);
        k1 = __ldg(bro + I + 1);
    }
    if (I < ntrip && lane < 3 && 3 * I + lane < n) op.pre(3 * I + lane + row_off);
    pdl_wait();
    if (trigger) pdl_trigger();
    if (I < nb) {
        // batches of 30 blocks: every column index and value load of a lane's
        // three blocks is issued before the dependent x gathers
        for (int64_t kb = k0; kb < k1; kb += 30) {
            int cc[3];
            double vv[3][3];
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const int64_t k = kb + kk + 10 * t;
                const bool ok = lane < 30 && k < k1;
                cc[t] = ok ? ldc<STREAM>(bci + k) : -1;
                const double *p = bval + 9 * k + 3 * c;
#pragma unroll
                for (int r = 0; r < 3; ++r) vv[t][r] = ok ? ldv<STREAM>(p + r) : 0.0;
            }
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                if (cc[t] >= 0) {
                    const double xv = op.x(3 * cc[t] + c);
                    a0 = fma(vv[t][0], xv, a0);
                    a1 = fma(vv[t][1], xv, a1);
                    a2 = fma(vv[t][2], xv, a2);
                }
            }
        }
    }
    if (rro != nullptr && I < ntrip) {
        const int g = lane / 10, gl = lane - 10 * g;
        const int64_t row = 3 * I + g;
        if (g < 3 && row < n) {
            const int64_t q1 = __ldg(rro + row + 1);
            double t0 = 0.0, t1 = 0.0;
            int64_t q = __ldg(rro + row) + gl;
            for (; q + 10 < q1; q += 20) {
                const double v0 = ldv<STREAM>(rv + q), v1 = ldv<STREAM>(rv + q + 10);
                const int c0 = ldc<STREAM>(rci + q), c1 = ldc<STREAM>(rci + q + 10);
                t0 = fma(v0, op.x(c0), t0);
                t1 = fma(v1, op.x(c1), t1);
            }
            if (q < q1) t0 = fma(ldv<STREAM>(rv + q), op.x(ldc<STREAM>(rci + q)), t0);
            const double t = t0 + t1;
            if (g == 0) a0 += t;
            else if (g == 1) a1 += t;
            else a2 += t;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(FULL, a0, o);
        a1 += __shfl_xor_sync(FULL, a1, o);
        a2 += __shfl_xor_sync(FULL, a2, o);
    }
    if (I < ntrip && lane < 3 && 3 * I + lane < n)
        op.out(3 * I + lane + row_off, lane == 0 ? a0 : lane == 1 ? a1 : a2);
}

// Operators with a CSR remainder (A0: displacement blocks plus the coupling
// columns and the flow rows): the same per-row arithmetic as k_bsr3, but the
// remainder's row bounds are read before the PDL wait and its first four
// entries per lane are issued together with the first block batch, so a
// warp pays one load round trip and one gather round trip instead of two of
// each.  Summation order (and hence every bit) matches k_bsr3.
template <class Op, int MINB>
__global__ void __launch_bounds__(256, MINB) k_bsr3r(int64_t ntrip, int64_t nb, int64_t n,
                                                     const int64_t *__restrict__ bro,
                                                     const int32_t *__restrict__ bci, const double *__restrict__ bval,
                                                     const int64_t *__restrict__ rro, const int32_t *__restrict__ rci,
                                                     const double *__restrict__ rv, Op op, int64_t row_off,
                                                     int trigger) {
    const int64_t I = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int kk = lane / 3, c = lane - 3 * kk;
    const int g = lane / 10, gl = lane - 10 * g;
    const int64_t row = 3 * I + g;
    const bool rok = g < 3 && I < ntrip && row < n;
    int64_t k0 = 0, k1 = 0, q0 = 0, q1 = 0;
    if (I < nb) {
        k0 = __ldg(bro + I);
        k1 = __ldg(bro + I + 1);
    }
    if (rok) {
        q0 = __ldg(rro + row) + gl;
        q1 = __ldg(rro + row + 1);
    }
    if (I < ntrip && lane < 3 && 3 * I + lane < n) op.pre(3 * I + lane + row_off);
    pdl_wait();
    if (trigger) pdl_trigger();
    int cc[3];
    double vv[3][3];
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        const int64_t k = k0 + kk + 10 * t;
        const bool ok = lane < 30 && k < k1;
        cc[t] = ok ? __ldg(bci + k) : -1;
        const double *p = bval + 9 * k + 3 * c;
#pragma unroll
        for (int r = 0; r < 3; ++r) vv[t][r] = ok ? __ldg(p + r) : 0.0;
    }
    int rc[4];
    double rvv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t q = q0 + 10 * u;
        const bool ok = q < q1;
        rc[u] = ok ? __ldg(rci + q) : -1;
        rvv[u] = ok ? __ldg(rv + q) : 0.0;
    }
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    {
        double xv[3], rx[4];
#pragma unroll
        for (int t = 0; t < 3; ++t) xv[t] = cc[t] >= 0 ? op.x(3 * cc[t] + c) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) rx[u] = rc[u] >= 0 ? op.x(rc[u]) : 0.0;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            if (cc[t] >= 0) {
                a0 = fma(vv[t][0], xv[t], a0);
                a1 = fma(vv[t][1], xv[t], a1);
                a2 = fma(vv[t][2], xv[t], a2);
            }
        }
        // rows with more than 30 blocks
        for (int64_t kb = k0 + 30; kb < k1; kb += 30) {
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const int64_t k = kb + kk + 10 * t;
                const bool ok = lane < 30 && k < k1;
                cc[t] = ok ? __ldg(bci + k) : -1;
                const double *p = bval + 9 * k + 3 * c;
#pragma unroll
                for (int r = 0; r < 3; ++r) vv[t][r] = ok ? __ldg(p + r) : 0.0;
            }
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                if (cc[t] >= 0) {
                    const double x = op.x(3 * cc[t] + c);
                    a0 = fma(vv[t][0], x, a0);
                    a1 = fma(vv[t][1], x, a1);
                    a2 = fma(vv[t][2], x, a2);
                }
            }
        }
        if (rok) {
            // k_bsr3's order: entries gl, gl+20, ... into t0 and gl+10,
            // gl+30, ... into t1
            double t0 = 0.0, t1 = 0.0;
            if (rc[0] >= 0) t0 = fma(rvv[0], rx[0], t0);
            if (rc[1] >= 0) t1 = fma(rvv[1], rx[1], t1);
            if (rc[2] >= 0) t0 = fma(rvv[2], rx[2], t0);
            if (rc[3] >= 0) t1 = fma(rvv[3], rx[3], t1);
            int64_t q = q0 + 40;
            for (; q + 10 < q1; q += 20) {
                const double v0 = __ldg(rv + q), v1 = __ldg(rv + q + 10);
                const int e0 = __ldg(rci + q), e1 = __ldg(rci + q + 10);
                t0 = fma(v0, op.x(e0), t0);
                t1 = fma(v1, op.x(e1), t1);
            }
            if (q < q1) t0 = fma(__ldg(rv + q), op.x(__ldg(rci + q)), t0);
            const double t = t0 + t1;
            if (g == 0) a0 += t;
            else if (g == 1) a1 += t;
            else a2 += t;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(FULL, a0, o);
        a1 += __shfl_xor_sync(FULL, a1, o);
        a2 += __shfl_xor_sync(FULL, a2, o);
    }
    if (I < ntrip && lane < 3 && 3 * I + lane < n)
        op.out(3 * I + lane + row_off, lane == 0 ? a0 : lane == 1 ? a1 : a2);
}

// Software-pipelined variant: a grid of resident warps strides over the
// row triples; the next triple's row bounds are fetched two triples ahead
// and its first batch of blocks is issued before the current triple's x
// gathers are consumed, so every warp keeps one triple's stream in flight
// instead of paying row-bound, stream and gather latencies in sequence.
template <class Op, int MINB>
__global__ void __launch_bounds__(256, MINB) k_bsr3p(int64_t ntrip, int64_t nb, int64_t n,
                                                     const int64_t *__restrict__ bro,
                                                     const int32_t *__restrict__ bci, const double *__restrict__ bval,
                                                     const int64_t *__restrict__ rro, const int32_t *__restrict__ rci,
                                                     const double *__restrict__ rv, Op op, int64_t row_off,
                                                     int trigger, unsigned tail_blk0 = 0xffffffffu) {
    if (blockIdx.x >= tail_blk0) {
        bsr3_tail_rows<false>(nb, n, rro, rci, rv, op, row_off, trigger, tail_blk0);
        return;
    }
    const int lane = threadIdx.x & 31;
    const int kk = lane / 3, c = lane - 3 * kk;
    const unsigned nbr = tail_blk0 < gridDim.x ? tail_blk0 : gridDim.x;  // block-role blocks
    const int64_t nw = (int64_t)nbr * (blockDim.x >> 5);
    int64_t I = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int cc[3];
    double vv[3][3];
    int64_t k0 = 0, k1 = 0;
#define PMGR_BSR3P_BATCH(KB, K1, CC, VV)                                                  \
    _Pragma("unroll") for (int t = 0; t < 3; ++t) {                                      \
        const int64_t k = (KB) + kk + 10 * t;                                            \
        const bool ok = lane < 30 && k < (K1);                                           \
        CC[t] = ok ? __ldg(bci + k) : -1;                                                \
        const double *p = bval + 9 * k + 3 * c;                                          \
        _Pragma("unroll") for (int r = 0; r < 3; ++r) VV[t][r] = ok ? __ldg(p + r) : 0.0; \
    }
    if (I < nb) {
        k0 = __ldg(bro + I);
        k1 = __ldg(bro + I + 1);
    }
    PMGR_BSR3P_BATCH(k0, k1, cc, vv)
    // bounds of the next triple
    int64_t n0 = 0, n1 = 0;
    if (I + nw < nb) {
        n0 = __ldg(bro + I + nw);
        n1 = __ldg(bro + I + nw + 1);
    }
    pdl_wait();
    if (trigger) pdl_trigger();
    for (; I < ntrip; I += nw) {
        double xv[3];
#pragma unroll
        for (int t = 0; t < 3; ++t) xv[t] = cc[t] >= 0 ? op.x(3 * cc[t] + c) : 0.0;
        // issue the next triple's first batch (and the bounds after it)
        int ncc[3];
        double nvv[3][3];
        PMGR_BSR3P_BATCH(n0, n1, ncc, nvv)
        const int64_t c0 = k0, c1 = k1;
        k0 = n0;
        k1 = n1;
        n0 = n1 = 0;
        if (I + 2 * nw < nb) {
            n0 = __ldg(bro + I + 2 * nw);
            n1 = __ldg(bro + I + 2 * nw + 1);
        }
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            if (cc[t] >= 0) {
                a0 = fma(vv[t][0], xv[t], a0);
                a1 = fma(vv[t][1], xv[t], a1);
                a2 = fma(vv[t][2], xv[t], a2);
            }
        }
        // rows with more than 30 blocks: the rest unpipelined
        for (int64_t kb = c0 + 30; kb < c1; kb += 30) {
            PMGR_BSR3P_BATCH(kb, c1, cc, vv)
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                if (cc[t] >= 0) {
                    const double x = op.x(3 * cc[t] + c);
                    a0 = fma(vv[t][0], x, a0);
                    a1 = fma(vv[t][1], x, a1);
                    a2 = fma(vv[t][2], x, a2);
                }
            }
        }
        if (rro != nullptr) {
            const int g = lane / 10, gl = lane - 10 * g;
            const int64_t row = 3 * I + g;
            if (g < 3 && row < n) {
                const int64_t q1 = __ldg(rro + row + 1);
                double t0 = 0.0, t1 = 0.0;
                int64_t q = __ldg(rro + row) + gl;
                for (; q + 10 < q1; q += 20) {
                    const double v0 = __ldg(rv + q), v1 = __ldg(rv + q + 10);
                    const int e0 = __ldg(rci + q), e1 = __ldg(rci + q + 10);
                    t0 = fma(v0, op.x(e0), t0);
                    t1 = fma(v1, op.x(e1), t1);
                }
                if (q < q1) t0 = fma(__ldg(rv + q), op.x(__ldg(rci + q)), t0);
                const double t = t0 + t1;
                if (g == 0) a0 += t;
                else if (g == 1) a1 += t;
                else a2 += t;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a0 += __shfl_xor_sync(FULL, a0, o);
            a1 += __shfl_xor_sync(FULL, a1, o);
            a2 += __shfl_xor_sync(FULL, a2, o);
        }
        if (lane < 3 && 3 * I + lane < n) {
            Op o = op;  // the pipelined kernel keeps no prefetch registers (measured: +20 % with them)
            o.pre(3 * I + lane + row_off);
            o.out(3 * I + lane + row_off, lane == 0 ? a0 : lane == 1 ? a1 : a2);
        }
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            cc[t] = ncc[t];
#pragma unroll
            for (int r = 0; r < 3; ++r) vv[t][r] = nvv[t][r];
        }
    }
#undef PMGR_BSR3P_BATCH
}

// ---------------------------------------------------------------------------
// TMA-staged block SpMV (pure BSR3 operators: the level-0 F-relaxation sweeps)
// ---------------------------------------------------------------------------
//
// A persistent grid of CTAs with 8 consumer warps and one producer warp.  The
// operator is cut into tiles of TPT = 8 * TPW consecutive row triples; a
// tile's blocks are one contiguous range of the value stream (72 B each,
// column-major) and of the block-column stream, so the producer moves them
// with two cp.async.bulk copies (TMA 1D) into a ring of shared-memory stages,
// signalled through mbarriers -- the loads are decoupled from the x gathers
// and issued by one thread instead of by every lane.  The operator is
// constant, so the producer starts streaming before griddepcontrol.wait
// (overlapping the predecessor's tail); only the consumers' x gathers and
// epilogues wait.  Consumer warp w sums triples w*TPW.. of each tile with
// exactly k_bsr3p's lane mapping and summation order (lane 3k+c owns column c
// of blocks k, k+10, k+20 of the triple, then the xor-shuffle tree), so the
// results are bitwise those of the register-streamed kernels.  Tiles larger
// than a stage (rows with more than 30 blocks on average) are read straight
// from global memory.

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_1d(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

constexpr int BT_CW = 8;               // consumer warps per CTA
constexpr int BT_THREADS = 32 * (BT_CW + 1);
constexpr int BT_BLK_PER_TRIPLE = 30;  // stage capacity per row triple (27-point stencil: 27)

struct BsrTileGeom {
    int64_t vb0, vbytes, cb0, cbytes;
};
__device__ __forceinline__ BsrTileGeom bsr_tile_geom(int64_t k0, int64_t k1) {
    BsrTileGeom g;
    g.vb0 = (72 * k0) & ~(int64_t)15;
    g.vbytes = ((72 * k1 + 15) & ~(int64_t)15) - g.vb0;
    g.cb0 = (4 * k0) & ~(int64_t)15;
    g.cbytes = ((4 * k1 + 15) & ~(int64_t)15) - g.cb0;
    return g;
}

template <class Op, int TPW>
__global__ void __launch_bounds__(BT_THREADS) k_bsr3t(int64_t ntrip, int64_t nb, int64_t n,
                                                      const int64_t *__restrict__ bro,
                                                      const int32_t *__restrict__ bci,
                                                      const double *__restrict__ bval, Op op, int64_t row_off,
                                                      int trigger, int stages, unsigned capv, unsigned capc) {
    constexpr int TPT = BT_CW * TPW;
    extern __shared__ __align__(128) unsigned char bt_smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(bt_smem);
    uint64_t *empty = full + stages;
    unsigned char *buf = bt_smem + 128;  // stage s: values at s*(capv+capc), columns after them
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (nb + TPT - 1) / TPT;
    if (threadIdx.x == 0) {
        for (int st = 0; st < stages; ++st) {
            mbar_init(full + st, 1);
            mbar_init(empty + st, BT_CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == BT_CW) {  // producer: one elected lane streams the tiles of this CTA
        if (lane == 0) {
            int st = 0;
            unsigned ph = 0;
            const char *vsrc = reinterpret_cast<const char *>(bval);
            const char *csrc = reinterpret_cast<const char *>(bci);
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                mbar_wait(empty + st, ph ^ 1);
                const int64_t I0 = t * TPT, I1 = I0 + TPT < nb ? I0 + TPT : nb;
                const BsrTileGeom g = bsr_tile_geom(__ldg(bro + I0), __ldg(bro + I1));
                unsigned char *vs = buf + (size_t)st * (capv + capc);
                if (g.vbytes <= (int64_t)capv && g.cbytes <= (int64_t)capc) {
                    mbar_arrive_tx(full + st, (unsigned)(g.vbytes + g.cbytes));
                    tma_1d(vs, vsrc + g.vb0, (unsigned)g.vbytes, full + st);
                    tma_1d(vs + capv, csrc + g.cb0, (unsigned)g.cbytes, full + st);
                } else {
                    mbar_arrive(full + st);  // oversize tile: the consumers read global memory
                }
                if (++st == stages) {
                    st = 0;
                    ph ^= 1;
                }
            }
        }
        return;
    }
    const int kk = lane / 3, c = lane - 3 * kk;
    pdl_wait();
    if (trigger) pdl_trigger();
    int st = 0;
    unsigned ph = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t I0 = t * TPT, I1 = I0 + TPT < nb ? I0 + TPT : nb;
        const int64_t k0 = __ldg(bro + I0);
        const BsrTileGeom g = bsr_tile_geom(k0, __ldg(bro + I1));
        const bool staged = g.vbytes <= (int64_t)capv && g.cbytes <= (int64_t)capc;
        const unsigned char *vs = buf + (size_t)st * (capv + capc);
        const double *sv = reinterpret_cast<const double *>(vs + (72 * k0 - g.vb0));
        const int32_t *sc = reinterpret_cast<const int32_t *>(vs + capv + (4 * k0 - g.cb0));
        int64_t kb[TPW], ke[TPW];
        Op ops[TPW];
#pragma unroll
        for (int p = 0; p < TPW; ++p) {
            const int64_t I = I0 + warp * TPW + p;
            kb[p] = ke[p] = 0;
            ops[p] = op;
            if (I < nb) {
                kb[p] = __ldg(bro + I);
                ke[p] = __ldg(bro + I + 1);
            }
            // the epilogue's setup-constant row data, loaded ahead of the gathers
            if (I < ntrip && lane < 3 && 3 * I + lane < n) ops[p].pre(3 * I + lane + row_off);
        }
        mbar_wait(full + st, ph);
        double a0[TPW], a1[TPW], a2[TPW];
        if (staged) {
            // every smem load and gather of the warp's triples issued before the FMAs
            int cc[TPW][3];
            double vv[TPW][3][3], xv[TPW][3];
#pragma unroll
            for (int p = 0; p < TPW; ++p)
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const int64_t k = kb[p] + kk + 10 * q;
                    const bool ok = lane < 30 && k < ke[p] && k < kb[p] + BT_BLK_PER_TRIPLE;
                    const int64_t r = k - k0;
                    cc[p][q] = ok ? sc[r] : -1;
#pragma unroll
                    for (int e = 0; e < 3; ++e) vv[p][q][e] = ok ? sv[9 * r + 3 * c + e] : 0.0;
                }
#pragma unroll
            for (int p = 0; p < TPW; ++p)
#pragma unroll
                for (int q = 0; q < 3; ++q) xv[p][q] = cc[p][q] >= 0 ? op.x(3 * cc[p][q] + c) : 0.0;
#pragma unroll
            for (int p = 0; p < TPW; ++p) {
                a0[p] = a1[p] = a2[p] = 0.0;
#pragma unroll
                for (int q = 0; q < 3; ++q)
                    if (cc[p][q] >= 0) {
                        a0[p] = fma(vv[p][q][0], xv[p][q], a0[p]);
                        a1[p] = fma(vv[p][q][1], xv[p][q], a1[p]);
                        a2[p] = fma(vv[p][q][2], xv[p][q], a2[p]);
                    }
                // rows with more than 30 blocks: the rest from global memory
                for (int64_t kq = kb[p] + BT_BLK_PER_TRIPLE; kq < ke[p]; kq += 30)
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const int64_t k = kq + kk + 10 * q;
                        if (lane < 30 && k < ke[p]) {
                            const double x = op.x(3 * __ldg(bci + k) + c);
                            const double *pv = bval + 9 * k + 3 * c;
                            a0[p] = fma(__ldg(pv), x, a0[p]);
                            a1[p] = fma(__ldg(pv + 1), x, a1[p]);
                            a2[p] = fma(__ldg(pv + 2), x, a2[p]);
                        }
                    }
            }
        } else {
#pragma unroll
            for (int p = 0; p < TPW; ++p) {
                a0[p] = a1[p] = a2[p] = 0.0;
                for (int64_t kq = kb[p]; kq < ke[p]; kq += 30)
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        const int64_t k = kq + kk + 10 * q;
                        if (lane < 30 && k < ke[p]) {
                            const double x = op.x(3 * __ldg(bci + k) + c);
                            const double *pv = bval + 9 * k + 3 * c;
                            a0[p] = fma(__ldg(pv), x, a0[p]);
                            a1[p] = fma(__ldg(pv + 1), x, a1[p]);
                            a2[p] = fma(__ldg(pv + 2), x, a2[p]);
                        }
                    }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + st);  // the stage may be refilled
        if (++st == stages) {
            st = 0;
            ph ^= 1;
        }
#pragma unroll
        for (int p = 0; p < TPW; ++p) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                a0[p] += __shfl_xor_sync(FULL, a0[p], o);
                a1[p] += __shfl_xor_sync(FULL, a1[p], o);
                a2[p] += __shfl_xor_sync(FULL, a2[p], o);
            }
            const int64_t I = I0 + warp * TPW + p;
            if (I < ntrip && lane < 3 && 3 * I + lane < n)
                ops[p].out(3 * I + lane + row_off, lane == 0 ? a0[p] : lane == 1 ? a1[p] : a2[p]);
        }
    }
}

struct OpY {
    static constexpr bool kTmaDefault = true;
    static double row_bytes(const OpY &) { return 0.0; }

    const double *xv;
    double *y;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ void pre(int64_t) {}
    __device__ void out(int64_t i, double s) const { y[i] = s; }
};
struct OpResidual {
    static constexpr bool kTmaDefault = true;
    static double row_bytes(const OpResidual &) { return 8.0; }  // b

    const double *xv, *b;
    double *r;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ void pre(int64_t) {}
    __device__ void out(int64_t i, double s) const { r[i] = b[i] - s; }
};
struct OpJacobi {
    static double row_bytes(const OpJacobi &) { return 16.0; }  // b, d (SURVEY 8(d) sweep rule)

    const double *xv, *b, *d;
    double *xo;
    __device__ double x(int j) const { return __ldg(xv + j); }
    double di = 1.0;  // pre(): setup-constant data of the output row, loaded before the PDL wait
    __device__ void pre(int64_t i) { di = __ldg(d + i); }
    __device__ void out(int64_t i, double s) const { xo[i] = xv[i] + (b[i] - s) / di; }
};
// post-sweep whose right-hand side is not written by the predecessor kernel
// (the AMG cycle: b_l was written by the restriction, long before)
struct OpJacobiPre {
    static double row_bytes(const OpJacobiPre &) { return 16.0; }

    const double *xv, *b, *d;
    double *xo;
    double di = 1.0, bi = 0.0;
    __device__ double x(int j) const { return __ldg(xv + j); }
    __device__ void pre(int64_t i) {
        di = __ldg(d + i);
        bi = b[i];
    }
    __device__ void out(int64_t i, double s) const { xo[i] = xv[i] + (bi - s) / di; }
};
struct OpSweep0 {
    static double row_bytes(const OpSweep0 &) { return 24.0; }  // b, d read; r written
    static constexpr double kColBytes = 8.0;            // x(j) = b_j / d_j

    const double *b, *d;
    double *xo, *r;
    __device__ double x(int j) const { return __ldg(b + j) / __ldg(d + j); }
    double di = 1.0;
    __device__ void pre(int64_t i) { di = __ldg(d + i); }
    __device__ void out(int64_t i, double s) const {
        xo[i] = b[i] / di;
        r[i] = b[i] - s;
    }
};
struct OpRestrictDiv {
    static double row_bytes(const OpRestrictDiv &) { return 16.0; }  // d read, x_c written
  // b_c = R r, and the first smoother iterate x_c = b_c / dtilde_c
    const double *r, *d;
    double *b, *xo;
    __device__ double x(int j) const { return __ldg(r + j); }
    double dk = 1.0;
    __device__ void pre(int64_t k) { dk = __ldg(d + k); }
    __device__ void out(int64_t k, double s) const {
        b[k] = s;
        xo[k] = s / dk;
    }
};
struct OpAdd {
    static double row_bytes(const OpAdd &) { return 8.0; }  // x read

    const double *e;
    double *xio;
    __device__ double x(int j) const { return __ldg(e + j); }
    __device__ void pre(int64_t) {}
    __device__ void out(int64_t i, double s) const { xio[i] += s; }
};
// x += P e where the predecessor kernel does not write x (the AMG cycle's
// prolongation: x was written by the level's pre-sweep, long before), so
// x_i is read before the PDL wait
struct OpAddPre {
    static double row_bytes(const OpAddPre &) { return 8.0; }

    const double *e;
    double *xio;
    double xi = 0.0;
    __device__ double x(int j) const { return __ldg(e + j); }
    __device__ void pre(int64_t i) { xi = xio[i]; }
    __device__ void out(int64_t i, double s) const { xio[i] = xi + s; }
};
struct OpResidRows {
    static double row_bytes(const OpResidRows &o) {
        return 16.0 + (o.x2 ? 16.0 : 0.0) + (o.sidx ? 24.0 : 0.0);  // row map, v; next level's first step
    }

    const double *zf, *v;
    const int64_t *rows;
    double *r;
    // the next level's first step, fused: its l1-Jacobi entry x2 = r / d2,
    // or its Jacobi F-relaxation sz[f] = sd[f] r for its F rows f = sidx[k]
    const double *d2;
    double *x2;
    const int64_t *sidx;
    const double *sd;
    double *sz;
    int64_t rk = 0, fk = -1;
    double d2k = 1.0, sdf = 0.0;
    __device__ double x(int j) const { return __ldg(zf + j); }
    __device__ void pre(int64_t k) {
        rk = __ldg(rows + k);
        if (x2) d2k = __ldg(d2 + k);
        if (sidx) {
            fk = __ldg(sidx + k);
            if (fk >= 0) sdf = __ldg(sd + fk);
        }
    }
    __device__ void out(int64_t k, double s) const {
        const double t = v[rk] - s;
        r[k] = t;
        if (x2) x2[k] = t / d2k;
        if (fk >= 0) sz[fk] = sdf * t;
    }
};
struct OpProlong {
    static double row_bytes(const OpProlong &) { return 16.0; }  // F map, z_F

    const double *ec, *zf;
    const int64_t *findex;
    double *z;
    __device__ double x(int j) const { return __ldg(ec + j); }
    // pre: the F map and z_F (written by this level's F-relaxation, never by
    // the coarse levels that run between it and this kernel)
    int64_t fi = -1;
    double zfv = 0.0;
    __device__ void pre(int64_t i) {
        fi = findex ? __ldg(findex + i) : -1;
        zfv = fi >= 0 ? zf[fi] : 0.0;
    }
    __device__ void out(int64_t i, double s) const { z[i] = zfv + s; }
};

// ---------------------------------------------------------------------------
// Sliced jagged kernels (SjView, sj.cu): one lane per row / row triple.
// ---------------------------------------------------------------------------

// One scalar slice: lane `lane` sums its row (len entries) onto acc, in stored
// order with one accumulator.  Positions are taken U at a time: the next
// chunk's (value, column) loads are issued before the current chunk's x
// gathers are consumed.  WAIT: the PDL wait sits between the first chunk's
// operator loads and the first gathers.
template <int U, bool WAIT, class Op>
__device__ __forceinline__ double sj_scalar_slice(const int32_t *__restrict__ ci, const double *__restrict__ v,
                                                  int64_t off0, int len, bool mine, int lane, const Op &op,
                                                  double acc, int trigger) {
    const unsigned lt = (1u << lane) - 1u;
    const int maxlen = __reduce_max_sync(FULL, len);
    const int minlen = __reduce_min_sync(FULL, len);  // positions [0, minlen) hold all 32 lanes
    const double *vb = v + off0;
    const int32_t *cb = ci + off0;
    int off = 0;  // entries of the slice before the next position to fetch (warp-uniform)
    double nv[U];
    int nc[U];
    auto fetch = [&](int t0) {
        int q[U];
        unsigned act = 0;
        if (t0 + U <= minlen) {  // full positions: lane-strided, no ranks
#pragma unroll
            for (int u = 0; u < U; ++u) q[u] = off + lane + 32 * u;
            off += 32 * U;
            act = mine ? 0xffffffffu : 0u;
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool a = t0 + u < len;
                const unsigned m = __ballot_sync(FULL, a);
                q[u] = off + __popc(m & lt);
                off += __popc(m);
                if (a && mine) act |= 1u << u;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ld = (act >> u) & 1u;
            // streamed once per pass: evict-first, so the gathered vector keeps
            // its lines (C4 AMG level 1: 737 -> 725 us, MGR apply -0.09 ms)
            nv[u] = ld ? __ldcs(vb + q[u]) : 0.0;
            nc[u] = ld ? __ldcs(cb + q[u]) : -1;
        }
    };
    fetch(0);
    if (WAIT) {
        pdl_wait();
        if (trigger) pdl_trigger();
    }
    for (int t0 = 0; t0 < maxlen; t0 += U) {
        double vv[U], xs[U];
        int cc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            vv[u] = nv[u];
            cc[u] = nc[u];
        }
#pragma unroll
        for (int u = 0; u < U; ++u) xs[u] = cc[u] >= 0 ? op.x(cc[u]) : 0.0;
        if (t0 + U < maxlen) fetch(t0 + U);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (cc[u] >= 0) acc = fma(vv[u], xs[u], acc);
    }
    return acc;
}

// role B: a warp per scalar slice of 32 / g consecutive rows, g = 2^lg lanes
// per row (lane gl of a row takes its entries g t + gl; the g partial sums
// are added pairwise at the end)
template <int U, class Op>
__device__ __forceinline__ void sj_role_b(const SjView &S, const Op &op, int trigger, int64_t sl, int lane,
                                          int64_t r1) {
    if (sl >= S.ncslice) return;
    const int lg = S.lg;
    const int64_t gs = S.ntslice + sl;
    const int64_t row = S.row0 + ((32 >> lg) * sl) + (lane >> lg);
    const bool mine = row >= S.r0 && row < r1;
    const bool head = (lane & ((1 << lg) - 1)) == 0;
    const int len = __ldg(S.slen + gs * 32 + lane);
    const int64_t off = __ldg(S.sptr + gs);
    Op o = op;
    if (mine && head) o.pre(row + S.row_off);
    double acc = sj_scalar_slice<U, true>(S.sci, S.sv, off, len, mine, lane, op, 0.0, trigger);
    for (int w = (1 << lg) >> 1; w > 0; w >>= 1) acc += __shfl_xor_sync(FULL, acc, w);
    if (mine && head) o.out(row + S.row_off, acc);
}

// role A (blockIdx.x < nblkA): a warp per block slice -- lane = row triple:
// its 3x3 blocks (UB positions per chunk), then the three triple-mode scalar
// slices holding the rows' entries outside the blocks.
// role B: a warp per scalar slice over consecutive rows.
template <int U, int UB, class Op>
__global__ void __launch_bounds__(128) k_sj(SjView S, Op op, int trigger, unsigned nblkA, int64_t bs0, int64_t cs0) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t r1 = S.r1 < 0 ? S.nrows : S.r1;
    if (blockIdx.x < nblkA) {
        const int64_t Sb = bs0 + (int64_t)blockIdx.x * 4 + w;
        if (Sb >= S.nbslice) return;
        const int64_t I = 32 * Sb + lane;
        const int64_t row = 3 * I;
        // whole triples only: a triple belongs to the range with its first row
        const bool mine = row >= S.r0 && row < r1 && I < S.nbrows;
        const int len = __ldg(S.blen + Sb * 32 + lane);
        int64_t off = __ldg(S.bptr + Sb);
        const unsigned lt = (1u << lane) - 1u;
        const int maxlen = __reduce_max_sync(FULL, len);
        int slen[3] = {0, 0, 0};
        int64_t soff[3] = {0, 0, 0};
        if (S.ntslice > 0) {
#pragma unroll
            for (int g = 0; g < 3; ++g) {
                slen[g] = __ldg(S.slen + (3 * Sb + g) * 32 + lane);
                soff[g] = __ldg(S.sptr + 3 * Sb + g);
            }
        }
        Op o0 = op, o1 = op, o2 = op;
        if (mine) {
            o0.pre(row + S.row_off);
            if (row + 1 < S.nrows) o1.pre(row + 1 + S.row_off);
            if (row + 2 < S.nrows) o2.pre(row + 2 + S.row_off);
        }
        double nv[UB][9];
        int nc[UB];
        auto fetch = [&](int t0) {
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const bool a = t0 + u < len;
                const unsigned m = __ballot_sync(FULL, a);
                const int k = __popc(m);
                const int r = __popc(m & lt);
                const bool ld = a && mine;
                nc[u] = ld ? __ldg(S.bci + off + r) : -1;
                const double *p = S.bval + 9 * off + r;
#pragma unroll
                for (int e = 0; e < 9; ++e) nv[u][e] = ld ? __ldg(p + (int64_t)e * k) : 0.0;
                off += k;
            }
        };
        fetch(0);
        pdl_wait();
        if (trigger) pdl_trigger();
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        for (int t0 = 0; t0 < maxlen; t0 += UB) {
            double vv[UB][9], xs[UB][3];
            int cc[UB];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                cc[u] = nc[u];
#pragma unroll
                for (int e = 0; e < 9; ++e) vv[u][e] = nv[u][e];
            }
#pragma unroll
            for (int u = 0; u < UB; ++u)
#pragma unroll
                for (int c = 0; c < 3; ++c) xs[u][c] = cc[u] >= 0 ? op.x(3 * cc[u] + c) : 0.0;
            if (t0 + UB < maxlen) fetch(t0 + UB);
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                if (cc[u] >= 0) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        a0 = fma(vv[u][3 * c + 0], xs[u][c], a0);
                        a1 = fma(vv[u][3 * c + 1], xs[u][c], a1);
                        a2 = fma(vv[u][3 * c + 2], xs[u][c], a2);
                    }
                }
            }
        }
        if (S.ntslice > 0) {
            a0 = sj_scalar_slice<U, false>(S.sci, S.sv, soff[0], slen[0], mine, lane, op, a0, 0);
            a1 = sj_scalar_slice<U, false>(S.sci, S.sv, soff[1], slen[1], mine, lane, op, a1, 0);
            a2 = sj_scalar_slice<U, false>(S.sci, S.sv, soff[2], slen[2], mine, lane, op, a2, 0);
        }
        if (mine) {
            o0.out(row + S.row_off, a0);
            if (row + 1 < S.nrows) o1.out(row + 1 + S.row_off, a1);
            if (row + 2 < S.nrows) o2.out(row + 2 + S.row_off, a2);
        }
        return;
    }
    sj_role_b<U>(S, op, trigger, cs0 + (int64_t)(blockIdx.x - nblkA) * 4 + w, lane, r1);
}

// operators without blocks: role B only (a fraction of k_sj's registers)
// (six blocks per SM: 80 registers; level 1 of C4 704 us, 712 us uncapped at 92)
template <int U, class Op, int MINB = 6>
__global__ void __launch_bounds__(128, MINB) k_sjs(SjView S, Op op, int trigger, int64_t cs0) {
    const int64_t r1 = S.r1 < 0 ? S.nrows : S.r1;
    sj_role_b<U>(S, op, trigger, cs0 + (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5), threadIdx.x & 31, r1);
}

// a kernel lets its successor launch early (PDL) only when its own grid is
// at most this many blocks per SM (PMGR_TRIG_BPS).  Default: every grid
// triggers (the successor's blocks take free slots during the last wave and
// issue their setup-constant loads): C2 solve 23.84 -> 23.05 ms against a
// 2-blocks-per-SM limit, C4 unchanged.  Safe for any value: every kernel
// triggers after its own griddepcontrol.wait, so a kernel's pre-wait reads
// never overtake the kernel two launches back.
int trigger_blocks_per_sm() {
    static const int v = [] {
        const char *e = getenv("PMGR_TRIG_BPS");
        return e ? atoi(e) : 1 << 20;
    }();
    return v;
}

// operators at least this large (PMGR_SPMV_BIG_NNZ; streamed from HBM, far
// beyond L2) keep four entries per lane in flight and take the pipelined
// kernel whatever their lane group: the small, latency-bound levels stay on
// two entries (more resident warps)
int64_t big_nnz() {
    static const int64_t v = [] {
        const char *e = getenv("PMGR_SPMV_BIG_NNZ");
        return e ? atoll(e) : (int64_t)1 << 62;  // off: C4 MGR apply 7.87 -> 8.00 ms with 2^25
    }();
    return v;
}

template <int G, class Op, class IT>
void go_t(const CsrView &A, const IT *ci, const Op &op, bool stream, cudaStream_t s) {
    const int block = 256;
    const unsigned nshort = grid_for(A.nrows * G, block);
    const int64_t nlong = A.long_len > 0 ? A.nlong : 0;
    const unsigned grid = nshort + (unsigned)nlong;
    // let the next kernel's launch overlap this one only when this grid is a
    // single wave (its early blocks must not crowd out ours)
    const int trigger = grid <= (unsigned)(trigger_blocks_per_sm() * num_sms()) ? 1 : 0;
    // PMGR_SPMV_U4: lane groups of at least this many lanes keep four
    // entries per lane in flight (0: always two)
    static const int u4 = [] {
        const char *e = getenv("PMGR_SPMV_U4");
        return e ? atoi(e) : 16;
    }();
    const bool four = A.lanes_u > 0 ? A.lanes_u == 4 : spmv_u_for(A.nnz, A.nrows, G) == 4;
    if (stream && four)
        launch_pdl(k_spmv<G, true, Op, IT, 4>, dim3(grid), dim3(block), 0, s, A.nrows, A.ro, ci, A.v, op,
                   A.row_off, trigger, A.long_len, A.lrows, nshort);
    else if (stream)
        launch_pdl(k_spmv<G, true, Op, IT>, dim3(grid), dim3(block), 0, s, A.nrows, A.ro, ci, A.v, op, A.row_off,
                   trigger, A.long_len, A.lrows, nshort);
    else if (four)
        launch_pdl(k_spmv<G, false, Op, IT, 4>, dim3(grid), dim3(block), 0, s, A.nrows, A.ro, ci, A.v, op,
                   A.row_off, trigger, A.long_len, A.lrows, nshort);
    else
        launch_pdl(k_spmv<G, false, Op, IT>, dim3(grid), dim3(block), 0, s, A.nrows, A.ro, ci, A.v, op, A.row_off,
                   trigger, A.long_len, A.lrows, nshort);
}

template <int G, class Op>
void go(const CsrView &A, const Op &op, bool stream, cudaStream_t s) {
    // PMGR_SPMV_PIPE: blocks per SM of the pipelined warp-per-row kernel for
    // lane group 32 without block-per-row long rows (0: off)
    static const int pipe = [] {
        const char *e = getenv("PMGR_SPMV_PIPE");
        return e ? atoi(e) : 4;
    }();
    static const int u4 = [] {
        const char *e = getenv("PMGR_SPMV_U4");
        return e ? atoi(e) : 16;
    }();
    // PMGR_SPMV_PIPE_MIN: smallest lane group that takes the pipelined kernel
    static const int pmin = [] {
        const char *e = getenv("PMGR_SPMV_PIPE_MIN");
        return e ? atoi(e) : 32;
    }();
    // PMGR_SPMV_PIPE_MAXNNZ: the pipelined kernel helps latency-bound levels
    // (C2: 24.6 -> 24.1 ms) but not HBM-streaming ones (C4 MGR apply 7.76 ->
    // 7.88 ms), so operators above this size keep the one-row-per-group kernel
    static const int64_t pmax = [] {
        const char *e = getenv("PMGR_SPMV_PIPE_MAXNNZ");
        return e ? atoll(e) : (int64_t)1 << 23;
    }();
    if (G >= 8 && (G >= pmin || A.nnz >= big_nnz()) && pipe == 4 && !stream && A.long_len <= 0 && A.nnz <= pmax) {
        const int64_t want = (int64_t)pipe * num_sms();
        const unsigned need = grid_for(A.nrows * G, 256);
        const unsigned pg = (unsigned)((int64_t)need < want ? (int64_t)need : want);
        const int trig = pg <= (unsigned)(trigger_blocks_per_sm() * num_sms()) ? 1 : 0;
        const bool four = A.lanes_u > 0 ? A.lanes_u == 4 : spmv_u_for(A.nnz, A.nrows, G) == 4;
        if (four) {
            if (A.ci16) launch_pdl(k_spmv_pipe<G, 4, Op, uint16_t, 4>, dim3(pg), dim3(256), 0, s, A.nrows, A.ro, A.ci16, A.v, op, A.row_off, trig);
            else launch_pdl(k_spmv_pipe<G, 4, Op, int32_t, 4>, dim3(pg), dim3(256), 0, s, A.nrows, A.ro, A.ci, A.v, op, A.row_off, trig);
        } else {
            if (A.ci16) launch_pdl(k_spmv_pipe<G, 2, Op, uint16_t, 4>, dim3(pg), dim3(256), 0, s, A.nrows, A.ro, A.ci16, A.v, op, A.row_off, trig);
            else launch_pdl(k_spmv_pipe<G, 2, Op, int32_t, 4>, dim3(pg), dim3(256), 0, s, A.nrows, A.ro, A.ci, A.v, op, A.row_off, trig);
        }
        return;
    }
    if (A.ci16) go_t<G>(A, A.ci16, op, stream, s);
    else go_t<G>(A, A.ci, op, stream, s);
}

}  // namespace

// lane group per row the CSR kernel picks for A (row-distributed copies of an
// operator reuse the global choice so their per-row sums are bitwise equal)
int spmv_lanes_mean(double mean) {
    static const double g32_mean = [] {
        const char *e = getenv("PMGR_SPMV_G32_MEAN");
        return e ? atof(e) : 100.0;
    }();
    return mean <= 3.0 ? 2 : mean <= 12.0 ? 4 : mean <= 48.0 ? 8 : mean <= g32_mean ? 16 : 32;
}

int spmv_u_for(int64_t nnz, int64_t nrows, int G) {
    static const int u4 = [] {
        const char *e = getenv("PMGR_SPMV_U4");
        return e ? atoi(e) : 16;
    }();
    // PMGR_SPMV_U4_MEAN: four entries once rows average more than this many
    // per lane (C2: 24.11 -> 23.94 ms at 2; 0: lane-group rule only)
    static const int umean = [] {
        const char *e = getenv("PMGR_SPMV_U4_MEAN");
        return e ? atoi(e) : 2;
    }();
    if (u4 > 0 && G >= u4) return 4;
    if (nnz >= big_nnz() && G >= 4) return 4;
    if (umean > 0 && nrows > 0 && nnz > (int64_t)umean * G * nrows) return 4;
    return 2;
}

int spmv_lanes(const CsrView &A) {
    double mean = A.nrows ? (double)A.nnz / (double)A.nrows : 0.0;
    // skewed rows (a few dense coarse-grid rows next to short ones) get a
    // whole warp unless they have the block-per-row path, otherwise the
    // longest row serialises its lane group
    if (A.maxrow >= 0 && A.long_len <= 0 && A.maxrow > 16 * spmv_lanes_mean(mean)) mean = 1e9;
    return spmv_lanes_mean(mean);
}

namespace {

template <class Op, class = void>
struct col_bytes_of {
    static constexpr double v = 0.0;
};
template <class Op>
struct col_bytes_of<Op, std::void_t<decltype(Op::kColBytes)>> {
    static constexpr double v = Op::kColBytes;
};

// TMA-staged block SpMV for pure BSR3 operators (PMGR_BSR_TMA=0: the
// register-streamed k_bsr3p); PMGR_BSR_TPW triples per consumer warp and
// tile (1 / 2), PMGR_BSR_STAGES stages, PMGR_BSR_CPS CTAs per SM
template <class Op, int TPW>
void launch_bsr3t_t(const CsrView &A, const Op &op, int stages, int cps, cudaStream_t s) {
    constexpr int tpt = BT_CW * TPW;
    const unsigned capv = (unsigned)((tpt * BT_BLK_PER_TRIPLE * 72 + 16 + 15) & ~15);
    const unsigned capc = (unsigned)((tpt * BT_BLK_PER_TRIPLE * 4 + 16 + 15) & ~15);
    const size_t smem = 128 + (size_t)stages * (capv + capc);
    static size_t set_for = 0;
    if (set_for < smem) {
        PMGR_CUDA(cudaFuncSetAttribute(k_bsr3t<Op, TPW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        set_for = smem;
    }
    const int64_t ntiles = (A.nbrows + tpt - 1) / tpt;
    const int64_t want = (int64_t)cps * num_sms();
    const unsigned grid = (unsigned)(ntiles < want ? ntiles : want);
    const int trig = grid <= (unsigned)(trigger_blocks_per_sm() * num_sms()) ? 1 : 0;
    launch_pdl(k_bsr3t<Op, TPW>, dim3(grid), dim3(BT_THREADS), smem, s, A.nbrows, A.nbrows, A.nrows, A.bro, A.bci,
               A.bval, op, A.row_off, trig, stages, capv, capc);
}

// epilogues with no per-row prefetch state take the TMA kernel by default
// (measured at C4: residual pass 944 -> 884 us); the Jacobi-type epilogues
// keep k_bsr3p, whose register budget suits them better (PMGR_BSR_TMA=2:
// every pure block operator, for A/B runs)
template <class Op, class = void>
struct tma_default {
    static constexpr bool v = false;
};
template <class Op>
struct tma_default<Op, std::void_t<decltype(Op::kTmaDefault)>> {
    static constexpr bool v = Op::kTmaDefault;
};

template <class Op>
bool launch_bsr3t(const CsrView &A, const Op &op, cudaStream_t s) {
    static const int on = [] {
        const char *e = getenv("PMGR_BSR_TMA");
        return e ? atoi(e) : 1;
    }();
    static const int tpw = [] {
        const char *e = getenv("PMGR_BSR_TPW");
        return e ? atoi(e) : 2;
    }();
    static const int stages = [] {
        const char *e = getenv("PMGR_BSR_STAGES");
        const int v = e ? atoi(e) : 2;
        return v < 2 ? 2 : v > 8 ? 8 : v;
    }();
    static const int cps = [] {
        const char *e = getenv("PMGR_BSR_CPS");
        return e ? atoi(e) : 3;
    }();
    if (!on || (on == 1 && !tma_default<Op>::v) || A.rro != nullptr || A.nbrows <= 0) return false;
    if (tpw == 1) launch_bsr3t_t<Op, 1>(A, op, stages, cps, s);
    else if (tpw == 4) launch_bsr3t_t<Op, 4>(A, op, stages, cps, s);
    else launch_bsr3t_t<Op, 2>(A, op, stages, cps, s);
    PMGR_LAUNCHED();
    return true;
}

// sliced jagged copy: block slices (role A) and consecutive scalar slices
// (role B) of one launch, restricted to the slices that meet the view's row
// range (row-distributed interior / boundary split)
template <class Op>
void launch_sj(const CsrView &A, const Op &op, cudaStream_t s) {
    const SjView &J = A.sj;
    const int64_t r0 = J.r0, r1 = J.r1 < 0 ? J.nrows : J.r1;
    int64_t bs0 = 0, bs1 = 0, cs0 = 0, cs1 = 0;
    if (J.nbslice > 0) {
        const int64_t prow = 3 * J.nbrows;
        const int64_t lo = r0 < prow ? r0 : prow, hi = r1 < prow ? r1 : prow;
        if (hi > lo) {
            bs0 = lo / 96;
            bs1 = (hi + 95) / 96;
        }
    }
    if (J.ncslice > 0 && r1 > J.row0) {
        const int64_t lo = (r0 > J.row0 ? r0 : J.row0) - J.row0, hi = r1 - J.row0;
        if (hi > lo) {
            const int64_t R = 32 >> J.lg;
            cs0 = lo / R;
            cs1 = (hi + R - 1) / R;
        }
    }
    const unsigned ga = (unsigned)((bs1 - bs0 + 3) / 4), gb = (unsigned)((cs1 - cs0 + 3) / 4);
    if (ga + gb == 0) return;
    const int trig = ga + gb <= (unsigned)(trigger_blocks_per_sm() * num_sms()) ? 1 : 0;
    static const int ub = [] {
        const char *e = getenv("PMGR_SJ_UB");
        return e ? atoi(e) : 2;  // C4 outer SpMV 1.73 ms with 3 positions per chunk, 1.53 ms with 2
    }();
    static const int uforce = [] {
        const char *e = getenv("PMGR_SJ_U");
        return e ? atoi(e) : 0;
    }();
    const int u = uforce > 0 ? uforce : J.u;
#define PMGR_SJ_GO(U_, UB_) \
    launch_pdl(k_sj<U_, UB_, Op>, dim3(ga + gb), dim3(128), 0, s, J, op, trig, ga, bs0, cs0)
    if (ga > 0 && ub == 2) {
        if (u <= 2) PMGR_SJ_GO(2, 2);
        else if (u <= 4) PMGR_SJ_GO(4, 2);
        else PMGR_SJ_GO(8, 2);
    } else if (ga > 0) {
        if (u <= 2) PMGR_SJ_GO(2, 3);
        else if (u <= 4) PMGR_SJ_GO(4, 3);
        else PMGR_SJ_GO(8, 3);
    } else {
        // PMGR_SJ_SHORT_MINB: blocks per SM the shortest-row variant (two
        // positions per chunk: prolongations, restrictions) is compiled for: their one or two chunks per row
        // are a chain of dependent round trips, so more resident warps help
        // (12 blocks = 40 registers: C4 MGR apply 15.64 -> 15.54 ms, the AMG
        // prolongation 98 -> 86 us)
        static const int short_minb = [] {
            const char *e = getenv("PMGR_SJ_SHORT_MINB");
            return e ? atoi(e) : 12;
        }();
        // (the four-position variant spills at 40 registers and measured slower:
        // it keeps six blocks per SM; a persistent grid-stride grid for the
        // short-row operators measured 15.65-15.80 ms against 15.61)
        if (u <= 2 && short_minb == 12) launch_pdl(k_sjs<2, Op, 12>, dim3(gb), dim3(128), 0, s, J, op, trig, cs0);
        else if (u <= 2 && short_minb == 10) launch_pdl(k_sjs<2, Op, 10>, dim3(gb), dim3(128), 0, s, J, op, trig, cs0);
        else if (u <= 2) launch_pdl(k_sjs<2, Op>, dim3(gb), dim3(128), 0, s, J, op, trig, cs0);
        else if (u <= 4) launch_pdl(k_sjs<4, Op>, dim3(gb), dim3(128), 0, s, J, op, trig, cs0);
        else launch_pdl(k_sjs<8, Op>, dim3(gb), dim3(128), 0, s, J, op, trig, cs0);
    }
#undef PMGR_SJ_GO
    PMGR_LAUNCHED();
}

template <class Op>
void launch(const CsrView &A, const Op &op, cudaStream_t s) {
    if (A.nrows == 0) return;
    ledger(csr_pass_bytes(A) + Op::row_bytes(op) * A.nrows + col_bytes_of<Op>::v * A.ncols);
    if (A.sj.on()) {
        launch_sj(A, op, s);
        return;
    }
    if (A.nbrows > 0 && launch_bsr3t(A, op, s)) return;
    if (A.nbrows > 0) {
        const int64_t ntrip = A.rro ? (A.nrows + 2) / 3 : A.nbrows;
        const unsigned grid = grid_for(ntrip * 32, 256);
        const int trigger = grid <= (unsigned)(trigger_blocks_per_sm() * num_sms()) ? 1 : 0;
        // PMGR_BSR_STREAM: evict-first loads for block-prefix operators with a
        // remainder (the Krylov operator A0: read once per iteration) = 1, for all = 2
        static const int bstream = [] {
            const char *e = getenv("PMGR_BSR_STREAM");
            return e ? atoi(e) : 0;
        }();
        // full occupancy (32 registers, a few spilled to L1) beats 40 registers at 75 %
        static const int minb = [] {
            const char *e = getenv("PMGR_BSR_MINB");
            return e ? atoi(e) : 8;
        }();
        // PMGR_BSR_PIPE: the software-pipelined variant with that many
        // blocks per SM (2..4; default 4), a resident grid striding over the
        // triples, for pure block operators (the level-0 F-relaxation sweeps:
        // 24.8 -> 22.3 us at C2); operators with a CSR remainder (A0) measured
        // faster on the one-triple-per-warp kernel
        static const int pipe = [] {
            const char *e = getenv("PMGR_BSR_PIPE");
            return e ? atoi(e) : 4;
        }();
        // PMGR_BSR_RMINB: blocks per SM of k_bsr3r for operators with a
        // remainder (0: the plain k_bsr3)
        static const int rminb = [] {
            const char *e = getenv("PMGR_BSR_RMINB");
            return e ? atoi(e) : 0;  // C2 +-0 %, C4 outer SpMV 2.37 -> 2.69 ms: off
        }();
        // PMGR_BSR_TAIL=0: rows past the prefix as 10-lane groups of triples
        static const int tailsplit = [] {
            const char *e = getenv("PMGR_BSR_TAIL");
            return e ? atoi(e) : 1;
        }();
        // PMGR_BSR_PIPE_A0=1: A0's block role as the pipelined kernel (resident
        // grid), its flow rows as extra blocks of the same launch
        static const int pipe_a0 = [] {
            const char *e = getenv("PMGR_BSR_PIPE_A0");
            return e ? atoi(e) : 1;
        }();
        // (latency-bound sizes only: C2 outer SpMV 37.2 -> 36.1 us, but C4's
        // 8.6 GB pass 2.01 -> 2.19 ms)
        if (A.rro != nullptr && tailsplit && A.nrows > 3 * A.nbrows && rminb == 0 && pipe_a0 &&
            csr_pass_bytes(A) <= 512.0 * 1024 * 1024) {
            const unsigned need = grid_for(A.nbrows * 32, 256);
            const int64_t want = 4 * (int64_t)num_sms();
            const unsigned gb = (unsigned)((int64_t)need < want ? (int64_t)need : want);
            const unsigned gt = grid_for((A.nrows - 3 * A.nbrows) * 8, 256);
            const int ttrig = gb + gt <= (unsigned)(trigger_blocks_per_sm() * num_sms()) ? 1 : 0;
            launch_pdl(k_bsr3p<Op, 4>, dim3(gb + gt), dim3(256), 0, s, A.nbrows, A.nbrows, A.nrows, A.bro, A.bci,
                       A.bval, A.rro, A.rci, A.rv, op, A.row_off, ttrig, gb);
        } else if (A.rro != nullptr && minb == 8 && tailsplit && A.nrows > 3 * A.nbrows && rminb == 0) {
            const unsigned gb = grid_for(A.nbrows * 32, 256);
            const unsigned gt = grid_for((A.nrows - 3 * A.nbrows) * 8, 256);
            const int ttrig = gb + gt <= (unsigned)(trigger_blocks_per_sm() * num_sms()) ? 1 : 0;
            launch_pdl(k_bsr3<Op, false, 8>, dim3(gb + gt), dim3(256), 0, s, A.nbrows, A.nbrows, A.nrows, A.bro,
                       A.bci, A.bval, A.rro, A.rci, A.rv, op, A.row_off, ttrig, gb);
        } else if (A.rro != nullptr && (rminb == 4 || rminb == 6 || rminb == 8)) {
            if (rminb == 4)
                launch_pdl(k_bsr3r<Op, 4>, dim3(grid), dim3(256), 0, s, ntrip, A.nbrows, A.nrows, A.bro, A.bci,
                           A.bval, A.rro, A.rci, A.rv, op, A.row_off, trigger);
            else if (rminb == 6)
                launch_pdl(k_bsr3r<Op, 6>, dim3(grid), dim3(256), 0, s, ntrip, A.nbrows, A.nrows, A.bro, A.bci,
                           A.bval, A.rro, A.rci, A.rv, op, A.row_off, trigger);
            else
                launch_pdl(k_bsr3r<Op, 8>, dim3(grid), dim3(256), 0, s, ntrip, A.nbrows, A.nrows, A.bro, A.bci,
                           A.bval, A.rro, A.rci, A.rv, op, A.row_off, trigger);
        } else if (pipe >= 2 && pipe <= 4 && A.rro == nullptr) {
            const int64_t want = (int64_t)pipe * num_sms();
            const unsigned pg = (unsigned)((int64_t)grid < want ? (int64_t)grid : want);
            const int ptrig = pg <= (unsigned)(trigger_blocks_per_sm() * num_sms()) ? 1 : 0;
            if (pipe == 2)
                launch_pdl(k_bsr3p<Op, 2>, dim3(pg), dim3(256), 0, s, ntrip, A.nbrows, A.nrows, A.bro, A.bci, A.bval,
                           A.rro, A.rci, A.rv, op, A.row_off, ptrig, 0xffffffffu);
            else if (pipe == 3)
                launch_pdl(k_bsr3p<Op, 3>, dim3(pg), dim3(256), 0, s, ntrip, A.nbrows, A.nrows, A.bro, A.bci, A.bval,
                           A.rro, A.rci, A.rv, op, A.row_off, ptrig, 0xffffffffu);
            else
                launch_pdl(k_bsr3p<Op, 4>, dim3(pg), dim3(256), 0, s, ntrip, A.nbrows, A.nrows, A.bro, A.bci, A.bval,
                           A.rro, A.rci, A.rv, op, A.row_off, ptrig, 0xffffffffu);
        } else if (minb == 8)
            launch_pdl(k_bsr3<Op, false, 8>, dim3(grid), dim3(256), 0, s, ntrip, A.nbrows, A.nrows, A.bro, A.bci,
                       A.bval, A.rro, A.rci, A.rv, op, A.row_off, trigger, 0xffffffffu);
        else if (bstream == 2 || (bstream == 1 && A.rro != nullptr))
            launch_pdl(k_bsr3<Op, true>, dim3(grid), dim3(256), 0, s, ntrip, A.nbrows, A.nrows, A.bro, A.bci,
                       A.bval, A.rro, A.rci, A.rv, op, A.row_off, trigger, 0xffffffffu);
        else
            launch_pdl(k_bsr3<Op>, dim3(grid), dim3(256), 0, s, ntrip, A.nbrows, A.nrows, A.bro, A.bci, A.bval,
                       A.rro, A.rci, A.rv, op, A.row_off, trigger, 0xffffffffu);
        PMGR_LAUNCHED();
        return;
    }
    // matrices far larger than L2 are streamed with evict-first loads so the
    // gathered vectors stay cached; small operators stay L2-resident
    static const double stream_mb = [] {
        const char *e = getenv("PMGR_SPMV_STREAM_MB");
        return e ? atof(e) : 1e30;
    }();
    const bool stream = 12.0 * (double)A.nnz > stream_mb * 1024 * 1024;
    switch (A.lanes > 0 ? A.lanes : spmv_lanes(A)) {
        case 2: go<2>(A, op, stream, s); break;
        case 4: go<4>(A, op, stream, s); break;
        case 8: go<8>(A, op, stream, s); break;
        case 16: go<16>(A, op, stream, s); break;
        default: go<32>(A, op, stream, s); break;
    }
    PMGR_LAUNCHED();
}

// Hybrid l1-GS over contiguous partitions (l1_gs_kernel, _kernels.py:13-44):
// one thread per partition runs Gauss-Seidel over its rows in order, reading
// the pre-sweep vector for columns outside the partition.
__global__ void k_hybrid_gs(int64_t nparts, const int64_t *__restrict__ starts,
                            const int64_t *__restrict__ ro, const int32_t *__restrict__ ci,
                            const double *__restrict__ v, const double *__restrict__ d,
                            const double *__restrict__ b, double *x, const double *__restrict__ xpre,
                            int forward) {
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= nparts) return;
    int64_t lo = starts[p], hi = starts[p + 1];
    for (int64_t t = 0; t < hi - lo; ++t) {
        int64_t i = forward ? lo + t : hi - 1 - t;
        double s = 0.0;
        for (int64_t q = ro[i]; q < ro[i + 1]; ++q) {
            int64_t j = ci[q];
            s += v[q] * ((j >= lo && j < hi) ? x[j] : xpre[j]);
        }
        x[i] += (b[i] - s) / d[i];
    }
}

// y = M x, M dense row-major with leading dimension ld (the collapsed coarse
// cycle, the coarsest inverse).  A block owns 8 rows; its warps split the
// columns, so a lane's x element is loaded once and reused for the 8 rows
// whose 8 independent matrix loads are in flight together.  PAIR: ld even,
// 16-byte loads of column pairs.
template <bool PAIR, bool STREAM = false, int RB = 8>
__global__ void __launch_bounds__(256) k_dense_matvec(const double *__restrict__ M, int64_t nrows, int64_t n, int64_t ld,
                                                      const double *__restrict__ x, double *__restrict__ y, int trigger) {
    constexpr int W = 8;
    __shared__ double red[W][RB];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r0 = (int64_t)blockIdx.x * RB;
    const int nr = (int)(nrows - r0 < RB ? nrows - r0 : RB);
    double acc[RB];
#pragma unroll
    for (int r = 0; r < RB; ++r) acc[r] = 0.0;
    if (PAIR) {
        const int64_t np = n >> 1;
        // M is constant: the first column pairs of the block's rows are
        // loaded before griddepcontrol.wait (overlapping the predecessor),
        // then each batch's loads are issued before the previous batch's FMAs
        double2 m[RB];
        int64_t p = warp * 32 + lane;
#define PMGR_DENSE_LOAD(P)                                                                                   \
    _Pragma("unroll") for (int r = 0; r < RB; ++r) m[r] =                                                     \
        (r < nr && (P) < np) ? (STREAM ? __ldcs(reinterpret_cast<const double2 *>(M + (r0 + r) * ld) + (P))   \
                                       : __ldg(reinterpret_cast<const double2 *>(M + (r0 + r) * ld) + (P)))   \
                             : make_double2(0.0, 0.0);
        PMGR_DENSE_LOAD(p)
        pdl_wait();
        if (trigger) pdl_trigger();
        for (; p < np; p += W * 32) {
            const double2 xv = make_double2(__ldg(x + 2 * p), __ldg(x + 2 * p + 1));
            double2 mc[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) mc[r] = m[r];
            PMGR_DENSE_LOAD(p + W * 32)
#pragma unroll
            for (int r = 0; r < RB; ++r) acc[r] = fma(mc[r].y, xv.y, fma(mc[r].x, xv.x, acc[r]));
        }
#undef PMGR_DENSE_LOAD
        if ((n & 1) && warp == 0 && lane == 0) {
            const double xl = __ldg(x + n - 1);
#pragma unroll
            for (int r = 0; r < RB; ++r)
                if (r < nr) acc[r] = fma(__ldg(M + (r0 + r) * ld + n - 1), xl, acc[r]);
        }
    } else {
        pdl_wait();
        if (trigger) pdl_trigger();
        for (int64_t c = warp * 32 + lane; c < n; c += W * 32) {
            const double xv = __ldg(x + c);
            double m[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) m[r] = r < nr ? __ldg(M + (r0 + r) * ld + c) : 0.0;
#pragma unroll
            for (int r = 0; r < RB; ++r) acc[r] = fma(m[r], xv, acc[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
        double t = acc[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL, t, o);
        if (lane == 0) red[warp][r] = t;
    }
    __syncthreads();
    if (threadIdx.x < nr) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < W; ++w) t += red[w][threadIdx.x];
        y[r0 + threadIdx.x] = t;
    }
}

__global__ void k_gather(const double *__restrict__ src, const int64_t *__restrict__ idx, int64_t n,
                         double *__restrict__ dst) {
    pdl_wait();
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}
__global__ void k_scale_gather(const double *__restrict__ src, const int64_t *__restrict__ idx,
                               const double *__restrict__ d, int64_t n, double *__restrict__ dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t k = i < n ? idx[i] : 0;  // constant index map: before the wait
    pdl_wait();
    if (i < n) dst[i] = d[i] * src[k];
}
__global__ void k_zero(double *x, int64_t n) {
    pdl_wait();
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) x[i] = 0.0;
}
__global__ void k_axpy(double a, const double *__restrict__ x, double *__restrict__ y, int64_t n) {
    pdl_wait();
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) y[i] += a * x[i];
}
__global__ void k_mul(const double *__restrict__ a, const double *__restrict__ b, double *__restrict__ y,
                      int64_t n) {
    pdl_wait();
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) y[i] = a[i] * b[i];
}

}  // namespace

CsrView rows_view(const CsrView &A, int64_t r0, int64_t r1) {
    CsrView v = A;
    if (A.sj.on()) {  // the copy keeps the operator's own row numbering: only the range narrows
        v.nrows = r1 - r0;
        v.sj.r0 = A.sj.r0 + r0;
        v.sj.r1 = A.sj.r0 + r1;
        return v;
    }
    v.nrows = r1 - r0;
    v.ro = A.ro + r0;
    v.row_off = A.row_off + r0;
    if (A.nbrows > 0) {  // pure block operator: ranges are whole row triples
        v.bro = A.bro + r0 / 3;
        v.nbrows = (r1 - r0) / 3;
    }
    v.long_len = 0;
    v.nlong = 0;
    v.lrows = nullptr;
    return v;
}

void spmv(const CsrView &A, const double *x, double *y, cudaStream_t s) { launch(A, OpY{x, y}, s); }

void spmv_residual(const CsrView &A, const double *x, const double *b, double *r, cudaStream_t s) {
    launch(A, OpResidual{x, b, r}, s);
}

void spmv_jacobi(const CsrView &A, const double *x, const double *b, const double *d, double *xo,
                 cudaStream_t s) {
    launch(A, OpJacobi{x, b, d, xo}, s);
}

void spmv_jacobi_bpre(const CsrView &A, const double *x, const double *b, const double *d, double *xo,
                      cudaStream_t s) {
    launch(A, OpJacobiPre{x, b, d, xo}, s);
}

void spmv_sweep0_residual(const CsrView &A, const double *b, const double *d, double *x, double *r,
                          cudaStream_t s) {
    launch(A, OpSweep0{b, d, x, r}, s);
}

void spmv_restrict_div(const CsrView &R, const double *r, const double *d, double *b, double *x,
                       cudaStream_t s) {
    launch(R, OpRestrictDiv{r, d, b, x}, s);
}

namespace {
__global__ void k_copy_div(const double *__restrict__ b, const double *__restrict__ d, int64_t n,
                           double *__restrict__ bo, double *__restrict__ xo) {
    pdl_wait();
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) {
        double v = b[i];
        bo[i] = v;
        xo[i] = v / d[i];
    }
}
}  // namespace

namespace {
__global__ void k_gather_div(const double *__restrict__ v, const int64_t *__restrict__ rows,
                             const double *__restrict__ d, int64_t n, double *__restrict__ bo,
                             double *__restrict__ xo) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t row = i < n ? rows[i] : 0;  // constant index map: before the wait
    pdl_wait();
    if (i < n) {
        const double t = v[row];
        bo[i] = t;
        xo[i] = t / d[i];
    }
}
}  // namespace

void vec_gather_div(const double *v, const int64_t *rows, const double *d, int64_t n, double *bo, double *xo,
                    cudaStream_t s) {
    if (n == 0) return;
    ledger(40.0 * n);
    launch_pdl(k_gather_div, dim3(grid_for(n, 256)), dim3(256), 0, s, v, rows, d, n, bo, xo);
    PMGR_LAUNCHED();
}

void vec_copy_div(const double *b, const double *d, int64_t n, double *bo, double *xo, cudaStream_t s) {
    if (n == 0) return;
    ledger(32.0 * n);
    launch_pdl(k_copy_div, dim3(grid_for(n, 256)), dim3(256), 0, s, b, d, n, bo, xo);
    PMGR_LAUNCHED();
}

void spmv_add_pre(const CsrView &A, const double *e, double *x, cudaStream_t s) {
    launch(A, OpAddPre{e, x}, s);
}

void spmv_add(const CsrView &A, const double *e, double *x, cudaStream_t s) {
    launch(A, OpAdd{e, x}, s);
}

void spmv_resid_rows(const CsrView &A, const double *zf, const double *v, const int64_t *rows, double *r,
                     const ResidNext &nx, cudaStream_t s) {
    launch(A, OpResidRows{zf, v, rows, r, nx.d2, nx.x2, nx.sidx, nx.sd, nx.sz}, s);
}

void spmv_prolong_combine(const CsrView &P, const double *ec, const double *zf, const int64_t *findex,
                          double *z, cudaStream_t s) {
    launch(P, OpProlong{ec, zf, findex, z}, s);
}

void hybrid_gs(const CsrView &A, int64_t nparts, const int64_t *starts, const double *d,
               const double *b, double *x, double *xpre, bool forward, cudaStream_t s) {
    PMGR_CUDA(cudaMemcpyAsync(xpre, x, sizeof(double) * A.nrows, cudaMemcpyDeviceToDevice, s));
    ledger(csr_pass_bytes(A) + 16.0 * A.nrows + 8.0 * A.ncols);  // b, d; x read twice
    k_hybrid_gs<<<grid_for(nparts, 128), 128, 0, s>>>(nparts, starts, A.ro, A.ci, A.v, d, b, x, xpre,
                                                     forward ? 1 : 0);
    PMGR_LAUNCHED();
}

void dense_matvec(const double *M, int64_t n, int64_t ld, const double *x, double *y, cudaStream_t s) {
    dense_matvec_rows(M, n, n, ld, x, y, s);
}

void dense_matvec_rows(const double *M, int64_t nrows, int64_t ncols, int64_t ld, const double *x, double *y,
                       cudaStream_t s) {
    if (nrows == 0) return;
    ledger(8.0 * nrows * ncols + 8.0 * ncols + 8.0 * nrows);
    // the collapsed operators are read once per cycle: evict-first loads keep
    // the sparse levels' operators (read again on the way up) in L2
    static const bool stream = !(getenv("PMGR_DENSE_STREAM") && getenv("PMGR_DENSE_STREAM")[0] == '0');
    static const int rb = [] {
        const char *e = getenv("PMGR_DENSE_RB");
        return e ? atoi(e) : 8;
    }();
    const unsigned blocks = (unsigned)((nrows + rb - 1) / rb);
    const int trig = (int64_t)((nrows + 7) / 8) <= (int64_t)trigger_blocks_per_sm() * num_sms() ? 1 : 0;
    if (ld % 2 == 0 && stream) {
        if (rb == 4)
            launch_pdl(k_dense_matvec<true, true, 4>, dim3(blocks), dim3(256), 0, s, M, nrows, ncols, ld, x, y, trig);
        else if (rb == 2)
            launch_pdl(k_dense_matvec<true, true, 2>, dim3(blocks), dim3(256), 0, s, M, nrows, ncols, ld, x, y, trig);
        else if (rb == 16)
            launch_pdl(k_dense_matvec<true, true, 16>, dim3(blocks), dim3(256), 0, s, M, nrows, ncols, ld, x, y, trig);
        else
            launch_pdl(k_dense_matvec<true, true, 8>, dim3(blocks), dim3(256), 0, s, M, nrows, ncols, ld, x, y, trig);
    } else if (ld % 2 == 0) {
        const unsigned b8 = (unsigned)((nrows + 7) / 8);
        launch_pdl(k_dense_matvec<true>, dim3(b8), dim3(256), 0, s, M, nrows, ncols, ld, x, y, trig);
    } else {
        const unsigned b8 = (unsigned)((nrows + 7) / 8);
        launch_pdl(k_dense_matvec<false>, dim3(b8), dim3(256), 0, s, M, nrows, ncols, ld, x, y, trig);
    }
    PMGR_LAUNCHED();
}

void vec_gather(const double *src, const int64_t *idx, int64_t n, double *dst, cudaStream_t s) {
    if (n == 0) return;
    ledger(24.0 * n);
    launch_pdl(k_gather, dim3(grid_for(n, 256)), dim3(256), 0, s, src, idx, n, dst);
    PMGR_LAUNCHED();
}

void vec_scale_gather(const double *src, const int64_t *idx, const double *d, int64_t n, double *dst,
                      cudaStream_t s) {
    if (n == 0) return;
    ledger(32.0 * n);
    launch_pdl(k_scale_gather, dim3(grid_for(n, 256)), dim3(256), 0, s, src, idx, d, n, dst);
    PMGR_LAUNCHED();
}

void vec_zero(double *x, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    ledger(8.0 * n);
    launch_pdl(k_zero, dim3(grid_for(n, 256)), dim3(256), 0, s, x, n);
    PMGR_LAUNCHED();
}

void vec_copy(const double *x, double *y, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    ledger(16.0 * n);
    PMGR_CUDA(cudaMemcpyAsync(y, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
}

void vec_axpy(double a, const double *x, double *y, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    ledger(24.0 * n);
    launch_pdl(k_axpy, dim3(grid_for(n, 256)), dim3(256), 0, s, a, x, y, n);
    PMGR_LAUNCHED();
}

void vec_mul(const double *a, const double *b, double *y, int64_t n, cudaStream_t s) {
    if (n == 0) return;
    ledger(24.0 * n);
    launch_pdl(k_mul, dim3(grid_for(n, 256)), dim3(256), 0, s, a, b, y, n);
    PMGR_LAUNCHED();
}

}  // namespace pmgr
