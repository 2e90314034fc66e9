// collapse.cu -- the coarse end of the AMG V-cycle as one dense operator.
//
// With a zero initial guess and l1-Jacobi smoothing, the V(1,1) cycle from
// level t downwards (amg.py:220-231) is a fixed LINEAR map b_t -> x_t:
//   M_l = (I - D_l^-1 A_l) (D_l^-1 + P_l M_{l+1} R_l (I - A_l D_l^-1)) + D_l^-1,
//   M_coarsest = A_c^-1.
// On the elasticity hierarchies the levels below ~2000 rows are many (the
// coarsening stagnates next to the Dirichlet-coupled dense rows) and tiny,
// so running them costs dozens of latency-bound launches per cycle.  Setup
// evaluates the cycle on all n_t unit vectors at once (the same six steps as
// the solve, as sparse x dense products) and keeps M_t (n_t^2 doubles, L2
// sized); the solve then replaces the whole tail by ONE bandwidth-bound
// dense matrix-vector product.  Same operator, different summation order:
// the apply parity bar (1e-10) is unaffected.
#include <cstdlib>

#include "hier.cuh"

namespace pmgr {

namespace {

constexpr int MM_BLOCK = 256;

// Y[i, c] = epilogue(i, c, sum_q a_iq X[ci_q, c]) for row-major n x k blocks
enum MmOp { MM_RESID = 0, MM_ASSIGN = 1, MM_ADD = 2, MM_SWEEP = 3 };

template <int OP>
__global__ void __launch_bounds__(MM_BLOCK) k_spmm(int64_t n, int64_t k, const int64_t *__restrict__ ro,
                                                    const int32_t *__restrict__ ci, const double *__restrict__ v,
                                                    const double *__restrict__ X, const double *__restrict__ B,
                                                    const double *__restrict__ d, double *Y) {
    const int64_t i = blockIdx.y;
    const int64_t c = blockIdx.x * (int64_t)MM_BLOCK + threadIdx.x;
    if (c >= k) return;
    double s = 0.0;
    for (int64_t q = ro[i]; q < ro[i + 1]; ++q) s = fma(v[q], X[(int64_t)ci[q] * k + c], s);
    const int64_t o = i * k + c;
    if (OP == MM_RESID) Y[o] = B[o] - s;                        // Y = B - A X
    if (OP == MM_ASSIGN) Y[o] = s;                              // Y = A X
    if (OP == MM_ADD) Y[o] += s;                                // Y += A X
    if (OP == MM_SWEEP) Y[o] = X[o] + (B[o] - s) / d[i];        // Y = X + (B - A X) / d
}

__global__ void k_rowdiv(int64_t n, int64_t k, const double *B, const double *d, double *X) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n * k) X[t] = B[t] / d[t / k];
}

__global__ void k_eye(int64_t n, double *X) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n * n) X[t] = (t / n == t % n) ? 1.0 : 0.0;
}

// Y (m x k) = C (m x m, row-major) * B (m x k)
__global__ void k_dense_mm(int64_t m, int64_t k, const double *C, const double *B, double *Y) {
    const int64_t i = blockIdx.y;
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= k) return;
    double s = 0.0;
    for (int64_t j = 0; j < m; ++j) s = fma(C[i * m + j], B[j * k + c], s);
    Y[i * k + c] = s;
}

template <int OP>
void spmm(const CsrView &A, int64_t k, const double *X, const double *B, const double *d, double *Y,
          cudaStream_t s) {
    if (A.nrows == 0 || k == 0) return;
    dim3 grid((unsigned)((k + MM_BLOCK - 1) / MM_BLOCK), (unsigned)A.nrows);
    k_spmm<OP><<<grid, MM_BLOCK, 0, s>>>(A.nrows, k, A.ro, A.ci, A.v, X, B, d, Y);
    PMGR_LAUNCHED();
}

// batched V-cycle from zero on k right-hand sides: XO = M_l B
void cycle_block(pmgr_amg &h, size_t l, int64_t k, const double *B, double *XO, cudaStream_t s) {
    if (l == h.levels.size()) {
        const int64_t nc = h.coarse->nrows;
        dim3 grid((unsigned)((k + 255) / 256), (unsigned)nc);
        if (nc) {
            k_dense_mm<<<grid, 256, 0, s>>>(nc, k, h.coarse_inv.p, B, XO);
            PMGR_LAUNCHED();
        }
        return;
    }
    AmgLevel &L = h.levels[l];
    const CsrView A = L.A->view();
    const int64_t n = A.nrows, nn = L.P.ncols;
    TBuf<double> X(n * k, s), Rm(n * k, s), Bn(nn * k, s), XOn(nn * k, s);
    k_rowdiv<<<grid_for(n * k, 256), 256, 0, s>>>(n, k, B, L.dtilde.p, X.p);    // first sweep from zero
    PMGR_LAUNCHED();
    spmm<MM_RESID>(A, k, X.p, B, nullptr, Rm.p, s);                             // r = b - A x
    spmm<MM_ASSIGN>(L.R.view(), k, Rm.p, nullptr, nullptr, Bn.p, s);            // b_c = R r
    cycle_block(h, l + 1, k, Bn.p, XOn.p, s);                                   // e = M_{l+1} b_c
    spmm<MM_ADD>(L.P.view(), k, XOn.p, nullptr, nullptr, X.p, s);               // x += P e
    spmm<MM_SWEEP>(A, k, X.p, B, L.dtilde.p, XO, s);                            // post-sweep
}

}  // namespace

int64_t collapse_limit() {
    static const int64_t limit = [] {
        const char *e = getenv("PMGR_COLLAPSE_ROWS");
        const int64_t v = e ? atoll(e) : (int64_t)3584;  // <= ~100 MB dense, read once per cycle
        return v < 65535 ? v : (int64_t)65535;
    }();
    return limit;
}

void collapse_tail(pmgr_amg &h, cudaStream_t s) {
    const int64_t limit = collapse_limit();
    if (limit <= 0 || h.levels.empty()) return;
    // deepest contiguous run of l1-Jacobi levels, starting at the first level
    // small enough for a dense operator
    int from = (int)h.levels.size();
    for (int l = (int)h.levels.size() - 1; l >= 0; --l) {
        if (!h.levels[l].jacobi || h.levels[l].A->nrows > limit) break;
        from = l;
    }
    if (from == (int)h.levels.size()) return;
    const int64_t k = h.levels[from].A->nrows;
    TBuf<double> B(k * k, s);
    k_eye<<<grid_for(k * k, 256), 256, 0, s>>>(k, B.p);
    PMGR_LAUNCHED();
    TBuf<double> Mt(k * k, s);
    cycle_block(h, (size_t)from, k, B.p, Mt.p, s);
    // rows padded to 256 bytes for the paired loads of the solve-phase matvec
    h.collapsed_ld = (k + 31) / 32 * 32;
    h.collapsed.alloc(k * h.collapsed_ld);
    PMGR_CUDA(cudaMemcpy2DAsync(h.collapsed.p, sizeof(double) * h.collapsed_ld, Mt.p, sizeof(double) * k,
                                sizeof(double) * k, k, cudaMemcpyDeviceToDevice, s));
    PMGR_CUDA(cudaStreamSynchronize(s));
    h.collapse_from = from;
}

}  // namespace pmgr
