// common.cuh -- shared infrastructure of libpmgr (B200 / sm_100a).
//
// Error model, device buffers, device CSR, launch bookkeeping and the warp
// primitives every kernel uses.  The setup kernels need bitwise-reproducible
// arithmetic: they use the explicit round-to-nearest
// intrinsics (__dadd_rn / __dmul_rn / __ddiv_rn), which nvcc never contracts
// into FMAs, and keep every per-entry sum in the reference's sequential order.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <string>
#include <utility>
#include <array>
#include <vector>

#include "../../include/pmgr.h"

namespace pmgr {

constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------

struct Error {
    pmgr_status code;
    std::string msg;
    int64_t index;
};

[[noreturn]] inline void fail(pmgr_status code, const std::string &msg, int64_t index = -1) {
    throw Error{code, msg, index};
}

[[noreturn]] inline void fail_cuda(cudaError_t e, const char *what, const char *file, int line) {
    char buf[512];
    snprintf(buf, sizeof(buf), "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
             cudaGetErrorString(e), file, line, what);
    fail(e == cudaErrorMemoryAllocation ? PMGR_ERR_OOM : PMGR_ERR_CUDA, buf);
}

#define PMGR_CUDA(x)                                                        \
    do {                                                                    \
        cudaError_t e_ = (x);                                               \
        if (e_ != cudaSuccess) ::pmgr::fail_cuda(e_, #x, __FILE__, __LINE__); \
    } while (0)

extern std::atomic<int64_t> g_launches;
// while a graph is being captured, launches are counted into the graph's
// kernel count instead (and charged to g_launches per replay)
extern thread_local int64_t *g_capture_count;

// Count + check a kernel launch issued just before.
// algorithmic-byte ledger: while set (a dry capture of one MGR application,
// pmgr_mgr_apply_bytes), every streaming launch adds the bytes it must move
extern thread_local double *g_byte_ledger;
inline void ledger(double bytes) {
    if (g_byte_ledger) *g_byte_ledger += bytes;
}

#define PMGR_LAUNCHED()                                                                \
    do {                                                                               \
        if (::pmgr::g_capture_count) ++*::pmgr::g_capture_count;                       \
        else ::pmgr::g_launches.fetch_add(1, std::memory_order_relaxed);              \
        cudaError_t e_ = cudaPeekAtLastError();                                        \
        if (e_ != cudaSuccess) ::pmgr::fail_cuda(e_, "kernel launch", __FILE__, __LINE__); \
    } while (0)

int num_sms();

// Programmatic dependent launch (Hopper+): a kernel launched with
// launch_pdl() may start while its predecessor drains; it must call
// pdl_wait() before touching anything the predecessor writes.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

// PMGR_SETUP_TRACE=1: synchronise and print the wall time of each setup
// phase to stderr (diagnostics only; off by default)
void setup_trace(const char *what, int64_t level, cudaStream_t s);
// host-side accounting under PMGR_SETUP_TRACE: seconds spent in cudaMalloc,
// cudaFree, pool allocations and blocking scalar reads (kind 0..3)
bool host_trace_on();
void host_trace_add(int kind, double seconds, double bytes);
void host_trace_report(const char *what);
struct HostTimer {
    int kind;
    double bytes;
    bool on;
    double t0;
    HostTimer(int k, double b);
    ~HostTimer();
};

template <class... KArgs, class... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
    if (e != cudaSuccess) fail_cuda(e, "cudaLaunchKernelEx", __FILE__, __LINE__);
}

inline unsigned grid_for(int64_t threads_needed, int block) {
    int64_t g = (threads_needed + block - 1) / block;
    if (g < 1) g = 1;
    if (g > 2147483647LL) g = 2147483647LL;
    return (unsigned)g;
}

// ---------------------------------------------------------------------------
// device buffers
// ---------------------------------------------------------------------------

// Persistent device buffers go through a block cache (prims.cu): cudaMalloc /
// cudaFree of the setup's ~900 operator arrays (62 GB at C4) cost 0.2-0.6 s
// per setup and varied box to box; freed blocks are kept (after a device
// synchronisation -- what cudaFree did implicitly) and handed to the next
// request of about that size, so a repeated setup allocates nothing.  The
// cache is capped (PMGR_DBUF_CACHE_GB, default 45 % of the device) and is
// returned to the driver when an allocation fails.  PMGR_DBUF_CACHE=0: off.
void *dbuf_alloc(size_t bytes);
void dbuf_free(void *p, size_t bytes);
void dbuf_trim();  // return the cached blocks to the driver

// Persistent device buffer: owned by long-lived handles.
template <class T>
struct DBuf {
    T *p = nullptr;
    int64_t n = 0;
    DBuf() = default;
    explicit DBuf(int64_t count) { alloc(count); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf &operator=(DBuf &&o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(int64_t count) {
        release();
        n = count;
        size_t bytes = sizeof(T) * (size_t)(count > 0 ? count : 1);
        p = static_cast<T *>(dbuf_alloc(bytes));
    }
    void release() {
        if (p) dbuf_free(p, sizeof(T) * (size_t)(n > 0 ? n : 1));
        p = nullptr;
        n = 0;
    }
    T *get() const { return p; }
};

// The device's default memory pool keeps what scratch buffers free (release
// threshold = unlimited) instead of returning it to the driver at every
// synchronisation: setup allocates and frees tens of GB of scratch at C4,
// and re-mapping it cost hundreds of ms per setup.  Called once per device.
void keep_pool_memory();

// Stream-ordered scratch buffer (cudaMallocAsync / cudaFreeAsync).
template <class T>
struct TBuf {
    T *p = nullptr;
    int64_t n = 0;
    cudaStream_t s = nullptr;
    TBuf() = default;
    TBuf(int64_t count, cudaStream_t st) { alloc(count, st); }
    TBuf(const TBuf &) = delete;
    TBuf &operator=(const TBuf &) = delete;
    TBuf(TBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    TBuf &operator=(TBuf &&o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            s = o.s;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~TBuf() { release(); }
    void alloc(int64_t count, cudaStream_t st) {
        release();
        s = st;
        n = count;
        size_t bytes = sizeof(T) * (size_t)(count > 0 ? count : 1);
        keep_pool_memory();
        HostTimer ht(2, (double)bytes);
        cudaError_t e = cudaMallocAsync((void **)&p, bytes, s);
        if (e == cudaErrorMemoryAllocation) {  // give the persistent buffers' cached blocks back and retry
            cudaGetLastError();
            dbuf_trim();
            e = cudaMallocAsync((void **)&p, bytes, s);
        }
        if (e != cudaSuccess) fail_cuda(e, "cudaMallocAsync", __FILE__, __LINE__);
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    T *get() const { return p; }
};

template <class T>
inline T read_scalar(const T *dev, cudaStream_t s) {
    T h;
    HostTimer ht(3, 0.0);
    PMGR_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, s));
    PMGR_CUDA(cudaStreamSynchronize(s));
    return h;
}

// ---------------------------------------------------------------------------
// device CSR
// ---------------------------------------------------------------------------

// Sliced jagged copy of an operator for the solve phase (sj.cu, spmv.cu): rows
// (or row triples of 3x3 blocks) in slices of 32, one lane per row; a slice
// stores position t of all its rows that have one contiguously (rows shorter
// than t simply drop out: no padding), so thread-per-row loads are coalesced
// and no cross-lane reduction is needed.  Scalar slices come first in
// "triple mode" (3 per block slice: rows 3 I + g of its triples, the entries
// outside the blocks), then over consecutive rows from row0.
struct SjView {
    int64_t nrows = 0;                        // rows of the whole operator
    int64_t nbslice = 0, nbrows = 0;          // block slices / row triples
    int64_t ntslice = 0, ncslice = 0, row0 = 0;
    const int64_t *bptr = nullptr;            // per block slice: first block
    const int32_t *blen = nullptr, *bci = nullptr;
    const double *bval = nullptr;             // per position: 9 planes of k doubles
    const int64_t *sptr = nullptr;            // per scalar slice: first entry
    const int32_t *slen = nullptr, *sci = nullptr;
    const double *sv = nullptr;
    int64_t nblocks = 0, nent = 0;
    int64_t r0 = 0, r1 = -1;                  // output row range (r1 < 0: all)
    int64_t row_off = 0;
    int u = 0;                                // positions per chunk of the scalar slices
    int lg = 0;                               // consecutive slices: 2^lg lanes per row
    bool on() const { return bptr != nullptr || sptr != nullptr; }
};

struct CsrView {
    int64_t nrows, ncols, nnz;
    const int64_t *ro;
    const int32_t *ci;
    const double *v;
    int64_t maxrow = -1;  // longest row (-1: unknown); picks the SpMV lane group
    // row-distributed operators (dist.cu): output row i is written at i + row_off
    // of the output vector; lanes force the global operator's lane group
    int64_t row_off = 0;
    int lanes = 0;
    const uint16_t *ci16 = nullptr;  // 16-bit copy of ci (ncols <= 65536), solve phase
    // optional solve-phase copy: the leading 3*nbrows rows/columns as 3x3
    // blocks (node-blocked displacement; blocks column-major, zero-filled),
    // every other entry as a remainder CSR over all rows (rro null: none)
    int64_t nbrows = 0, nblocks = 0, nrem = 0;
    const int64_t *bro = nullptr;
    const int32_t *bci = nullptr;
    const double *bval = nullptr;
    const int64_t *rro = nullptr;
    const int32_t *rci = nullptr;
    const double *rv = nullptr;
    // rows longer than long_len (> 0) are summed by a whole block each (the
    // nlong rows listed in lrows); the lane group then fits the other rows
    int64_t long_len = 0, nlong = 0;
    const int32_t *lrows = nullptr;
    int lanes_u = 0;  // entries per lane in flight (2 / 4; 0: from this operator's mean)
    SjView sj;        // sliced jagged solve copy (takes precedence when present)
};

struct Sj {
    int64_t nbslice = 0, nbrows = 0, ntslice = 0, ncslice = 0, row0 = 0, nblocks = 0, nent = 0;
    DBuf<int64_t> bptr, sptr;
    DBuf<int32_t> blen, bci, slen, sci;
    DBuf<double> bval, sv;
    std::shared_ptr<const Sj> blk_src;  // block piece borrowed from another operator (A0 <- A_uu)
    int u = 0, lg = 0;
};

struct Csr {
    int64_t nrows = 0, ncols = 0, nnz = 0;
    DBuf<int64_t> ro;
    DBuf<int32_t> ci;
    DBuf<double> v;
    void alloc(int64_t r, int64_t c, int64_t z) {
        nrows = r;
        ncols = c;
        nnz = z;
        ro.alloc(r + 1);
        ci.alloc(z);
        v.alloc(z);
    }
    int64_t maxrow = -1;
    int64_t row_off = 0;
    int lanes = 0;
    DBuf<uint16_t> ci16;
    int64_t nbrows = 0, nblocks = 0, nrem = 0;
    DBuf<int64_t> bro, rro;
    DBuf<int32_t> bci, rci;
    DBuf<double> bval, rv;
    int64_t long_len = 0, nlong = 0;
    DBuf<int32_t> lrows;
    int lanes_u = 0;
    // blocks shared with another operator whose blocks are this one's block
    // prefix (A0 and its level-0 A_FF = A_uu: one copy of the displacement
    // blocks, so the Krylov SpMV re-reads what the last F-relaxation sweep
    // left in L2)
    std::shared_ptr<const Csr> blk_src;
    // row-distributed operators: contiguous local row ranges that read no
    // ghost column (inner) and the rest (outer); the interior rows run while
    // the halo exchange is in flight (with_halo, hier.cuh).  Empty: no split.
    std::vector<std::array<int64_t, 2>> inner, outer;
    std::shared_ptr<Sj> sj;  // sliced jagged solve copy (large operators)
    bool sj_want = false;    // the (global) operator is large enough for it
    bool sj_tried = false;   // a caller's matrix: the lazy build ran (capi.cu)
    // the GLOBAL operator's rows / entries when this is a rank's slice or a
    // partial (owned-rows) operator (0: its own): the lanes-per-row choice of
    // the sliced jagged copy fixes the summation order, so slices follow it
    int64_t g_rows = 0, g_nnz = 0;
    CsrView view() const {
        const Csr &b = blk_src ? *blk_src : *this;
        CsrView V{nrows,  ncols,  nnz,     ro.p,    ci.p,    v.p,      maxrow, row_off,  lanes, ci16.p,
                  nbrows, nblocks, nrem,   b.bro.p, b.bci.p, b.bval.p, rro.p,  rci.p,    rv.p,  long_len,
                  nlong,  lrows.p, lanes_u};
        if (sj) {
            const Sj &bs = sj->blk_src ? *sj->blk_src : *sj;
            SjView &J = V.sj;
            J.nrows = nrows;
            J.nbslice = bs.nbslice;
            J.nbrows = bs.nbrows;
            J.ntslice = sj->ntslice;
            J.ncslice = sj->ncslice;
            J.row0 = sj->row0;
            J.bptr = bs.bptr.p;
            J.blen = bs.blen.p;
            J.bci = bs.bci.p;
            J.bval = bs.bval.p;
            J.sptr = sj->sptr.p;
            J.slen = sj->slen.p;
            J.sci = sj->sci.p;
            J.sv = sj->sv.p;
            J.nblocks = bs.nblocks;
            J.nent = sj->nent;
            J.row_off = row_off;
            J.u = sj->u;
            J.lg = sj->lg;
        }
        return V;
    }
};

// build the block-prefix solve copy of an operator whose leading prow rows
// and pcol columns are node-blocked by 3 (prow = nrows, pcol = ncols: pure
// BSR3); keeps the plain CSR when the blocks would be too sparse (unless force)
struct DistSetup;
void csr_make_bsr3(Csr &A, int64_t prow, int64_t pcol, cudaStream_t s, bool force = false,
                   const DistSetup *dist = nullptr);
// the block-prefix copy of A reusing src's blocks (src: a pure BSR3 operator
// equal to A's leading prefix x prefix block); builds only A's remainder
void csr_make_bsr3_shared(Csr &A, int64_t prefix, std::shared_ptr<const Csr> src, cudaStream_t s);
// sliced jagged solve copy of an operator of at least PMGR_SJ_MIN_NNZ entries
// (built from its block-prefix copy when it has one); blk: the operator whose
// blocks are this one's block prefix and already has its own copy
void csr_make_sj(Csr &A, cudaStream_t s, bool force = false);
// B = P A P^T (row i of B = row perm[i] of A), columns re-sorted
std::shared_ptr<Csr> csr_permute(const Csr &A, const int64_t *perm_host, cudaStream_t s);

// record the longest row of a finished operator (setup time, synchronises)
// build_sj = false: only note whether the operator wants the sliced jagged
// copy (sj_want); the caller builds it later (csr_make_sj) or never
void csr_finalize(Csr &A, cudaStream_t s, bool build_sj = true);
bool sj_wanted(int64_t nrows, int64_t nnz);  // PMGR_SJ_MIN_NNZ / PMGR_SJ_MIN_ROWS
// list the rows longer than A.long_len (0: none) for the block-per-row path
void csr_long_rows(Csr &A, cudaStream_t s);

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------

// Sequential left-to-right sum of a chunk of up to 32 values held one per
// lane (lane k holds element k), continued from s.  Every lane returns the
// same, order-exact result: (((s + x0) + x1) + ...).
__device__ __forceinline__ double warp_seq_sum(double s, double x, int cnt) {
    for (int k = 0; k < cnt; ++k) s = __dadd_rn(s, __shfl_sync(FULL, x, k));
    return s;
}

__device__ __forceinline__ double warp_max(double x) {
    for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(FULL, x, o));
    return x;
}

__device__ __forceinline__ int64_t warp_sum_i64(int64_t x) {
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    return x;
}

// ---------------------------------------------------------------------------
// live kernel timing (pmgr_prof_*): CUDA events around selected launches on
// the launching stream, with the algorithmic bytes each one must move.
// ---------------------------------------------------------------------------

enum ProfKind {
    PROF_OUTER_SPMV = 0,    // y = A z in the GMRES loop
    PROF_FRELAX_SWEEP0 = 1, // level-0 fused first sweep + residual of the F-relax AMG
    PROF_FRELAX_JACOBI = 2, // level-0 post-sweep of the F-relax AMG
    PROF_MGR_APPLY = 3,     // whole preconditioner application
    PROF_ORTHO = 4,         // CGS2 projections + normalisation of one Arnoldi step
    PROF_KINDS = 5
};

struct ProfRec {
    int kind;
    double bytes;
    cudaEvent_t a, b;
};
bool prof_on();
void prof_capture_begin(std::vector<ProfRec> *recs);
void prof_capture_end();
void prof_collect(std::vector<ProfRec> &graph_recs);
void prof_release(std::vector<ProfRec> &graph_recs);
void prof_enable(bool on);
void prof_query(int kind, int64_t *count, double *ms, double *bytes);
void prof_begin(int kind, double bytes, cudaStream_t s);
void prof_end(int kind, cudaStream_t s);

struct ProfScope {
    int kind;
    cudaStream_t s;
    bool on;
    ProfScope(int k, double bytes, cudaStream_t st) : kind(k), s(st), on(k < PROF_KINDS && prof_on()) {
        if (on) prof_begin(k, bytes, st);
    }
    ~ProfScope() {
        if (on) prof_end(kind, s);
    }
};

// algorithmic bytes of one CSR pass (int64 offsets, int32 columns, fp64
// values; x gathered once, y written once)
inline double csr_pass_bytes(int64_t nrows, int64_t ncols, int64_t nnz) {
    return 12.0 * nnz + 8.0 * (nrows + 1) + 8.0 * ncols + 8.0 * nrows;
}
// one pass over the format the solve actually streams (BSR3 copy if present)
inline double csr_pass_bytes(const CsrView &A) {
    if (A.sj.on())  // blocks + entries + 4-byte lengths per lane + 8-byte slice starts
        return 76.0 * A.sj.nblocks + 12.0 * A.sj.nent +
               (4.0 * 32 + 8.0) * (A.sj.nbslice + A.sj.ntslice + A.sj.ncslice) + 8.0 * A.ncols + 8.0 * A.nrows;
    if (A.nbrows > 0)
        return 76.0 * A.nblocks + 8.0 * (A.nbrows + 1) + 12.0 * A.nrem + (A.rro ? 8.0 * (A.nrows + 1) : 0.0) +
               8.0 * A.ncols + 8.0 * A.nrows;
    return csr_pass_bytes(A.nrows, A.ncols, A.nnz) - (A.ci16 ? 2.0 * A.nnz : 0.0);
}

// ---------------------------------------------------------------------------
// host-side primitives implemented in prims.cu (CUB based)
// ---------------------------------------------------------------------------

// out[0] = 0, out[i+1] = sum_{k<=i} in[k]; returns the total (synchronises).
int64_t exclusive_scan_total(const int64_t *in, int64_t *out, int64_t n, cudaStream_t s);
int64_t exclusive_scan_total_i32(const int32_t *in, int64_t *out, int64_t n, cudaStream_t s);
// Sort (keys, vals) pairs within each CSR row segment by key (ascending).
// the same over an explicit list of [sbeg[i], send[i]) segments
void segmented_sort_pairs_list(int32_t *keys, double *vals, int64_t nnz, const int64_t *sbeg, const int64_t *send,
                               int64_t nseg, cudaStream_t s);
void segmented_sort_pairs(int32_t *keys, double *vals, int64_t nnz, const int64_t *ro,
                          int64_t nrows, cudaStream_t s);
double device_max_abs(const double *x, int64_t n, cudaStream_t s);

// CSR utilities (csr.cu)
void csr_transpose(const CsrView &A, Csr &T, cudaStream_t s);
// mode 0: drop exact zeros (scipy product); mode 1: structural pattern kept,
// zero sums stored as +0.0 (reference spgemm).
void spgemm(const CsrView &X, const CsrView &Y, int mode, Csr &C, cudaStream_t s);
void csr_subtract(const CsrView &A, const CsrView &B, Csr &C, cudaStream_t s);
void csr_sparsify(const CsrView &M, const int32_t *entity, int64_t n_max, Csr &K,
                  cudaStream_t s);
void csr_copy(const CsrView &A, Csr &B, cudaStream_t s);
void csr_diagonal(const CsrView &A, double *d, cudaStream_t s);
// d = 1/diag; returns the first row whose diagonal is zero or missing (-1 if none).
int64_t csr_diag_inverse(const CsrView &A, double *dinv, cudaStream_t s);
void csr_validate(const CsrView &A, cudaStream_t s);

// SpMV family (spmv.cu)
void spmv(const CsrView &A, const double *x, double *y, cudaStream_t s);
void spmv_residual(const CsrView &A, const double *x, const double *b, double *r, cudaStream_t s);
void spmv_jacobi(const CsrView &A, const double *x, const double *b, const double *d,
                 double *xo, cudaStream_t s);
// the same when the predecessor kernel does not write b
void spmv_jacobi_bpre(const CsrView &A, const double *x, const double *b, const double *d,
                 double *xo, cudaStream_t s);
void spmv_sweep0_residual(const CsrView &A, const double *b, const double *d, double *x,
                          double *r, cudaStream_t s);
void spmv_add(const CsrView &A, const double *e, double *x, cudaStream_t s);
// the same, for call sites whose predecessor kernel does not write x
void spmv_add_pre(const CsrView &A, const double *e, double *x, cudaStream_t s);
void spmv_restrict_div(const CsrView &R, const double *r, const double *d, double *b, double *x,
                       cudaStream_t s);
void vec_copy_div(const double *b, const double *d, int64_t n, double *bo, double *xo, cudaStream_t s);
// bo = v[rows], xo = bo / d (gathered right-hand side + first l1-Jacobi sweep)
void vec_gather_div(const double *v, const int64_t *rows, const double *d, int64_t n, double *bo, double *xo,
                    cudaStream_t s);
// optional fused first step of the level consuming a C residual
struct ResidNext {
    const double *d2 = nullptr;  // l1-Jacobi entry of an AMG: x2 = r / d2
    double *x2 = nullptr;
    const int64_t *sidx = nullptr;  // Jacobi F-relaxation of an MGR level: sz[sidx[k]] = sd[..] r[k]
    const double *sd = nullptr;
    double *sz = nullptr;
};
void spmv_resid_rows(const CsrView &A, const double *zf, const double *v, const int64_t *rows, double *r,
                     const ResidNext &nx, cudaStream_t s);
void spmv_prolong_combine(const CsrView &P, const double *ec, const double *zf,
                          const int64_t *findex, double *z, cudaStream_t s);
void hybrid_gs(const CsrView &A, int64_t nparts, const int64_t *starts, const double *d,
               const double *b, double *x, double *xpre, bool forward, cudaStream_t s);
int spmv_lanes(const CsrView &A);
// lane group per row for a mean row length (no skew correction)
int spmv_lanes_mean(double mean);
// entries per lane the CSR kernel keeps in flight for lane group G (4 when
// rows average more than two entries per lane); row-distributed copies
// inherit the global operator's choice (lanes_u) so their sums stay bitwise
int spmv_u_for(int64_t nnz, int64_t nrows, int G);
// y[0:nrows) = M[0:nrows, 0:ncols) x (row-distributed collapsed operators)
void dense_matvec_rows(const double *M, int64_t nrows, int64_t ncols, int64_t ld, const double *x, double *y,
                       cudaStream_t s);
void dense_matvec(const double *M, int64_t n, int64_t ld, const double *x, double *y, cudaStream_t s);

// elementwise (spmv.cu)
void vec_gather(const double *src, const int64_t *idx, int64_t n, double *dst, cudaStream_t s);
void vec_scale_gather(const double *src, const int64_t *idx, const double *d, int64_t n,
                      double *dst, cudaStream_t s);
void vec_zero(double *x, int64_t n, cudaStream_t s);
void vec_copy(const double *x, double *y, int64_t n, cudaStream_t s);
void vec_axpy(double a, const double *x, double *y, int64_t n, cudaStream_t s);
void vec_mul(const double *a, const double *b, double *y, int64_t n, cudaStream_t s);

}  // namespace pmgr
