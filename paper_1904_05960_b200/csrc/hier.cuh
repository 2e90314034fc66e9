// hier.cuh -- device-resident AMG and MGR hierarchies.
#pragma once

#include <functional>
#include <memory>
#include <vector>

#include "common.cuh"

struct pmgr_csr {
    std::shared_ptr<pmgr::Csr> m;
};

namespace pmgr {

// ---- row distribution (dist.cu) --------------------------------
// Every vector space of a row-distributed hierarchy is owned in contiguous
// global ranges, rank after rank (the level-0 numbering is rank-major and C
// points keep their order).  A rank stores a space as an "ext" vector: its
// owned range plus the ghost entries its operators read, in global order, so
// local rows sum their columns in the global stored order.
struct Transport;
struct Halo {  // ghost exchange of one space on one rank
    Transport *tr = nullptr;
    int64_t n_ext = 0, off = 0, n_own = 0;  // owned entries sit at [off, off + n_own)
    std::vector<int> rpeer, speer;          // peers I receive from / send to
    std::vector<int64_t> roff, rcnt;        // per receive peer: its contiguous ghost segment
    std::vector<int64_t> soff, scnt;        // per send peer: its segment of send_idx
    DBuf<int64_t> send_idx;                 // owned-local indices, peer after peer
    DBuf<double> sbuf;                      // packed send values
    int id = -1;                            // space id (matches across ranks)
};
struct Gather {  // all-gather of one space into its full global-order vector
    Transport *tr = nullptr;
    int64_t n_full = 0;
    std::vector<int64_t> start;  // per rank global range start (nranks + 1)
    int id = -1;
};
void halo_exchange(Halo *h, double *ext, cudaStream_t s);

// Interior / boundary overlap of a row-distributed operator: halo_fork starts
// the exchange of x's ghosts on a side stream (forked from s) when A has a
// row split and the halo has a transport, returning false otherwise;
// halo_join makes s wait for it.  with_halo runs `launch` on A's interior row
// ranges while the exchange is in flight, then on the boundary ranges.  Every
// row keeps its lane group and summation order, so the results are bitwise
// those of exchange-then-launch.
bool halo_fork(const Csr &A, Halo *h, double *x, cudaStream_t s);
void halo_join(cudaStream_t s);
CsrView rows_view(const CsrView &A, int64_t r0, int64_t r1);
template <class F>
inline void with_halo(const Csr &A, Halo *h, double *x, cudaStream_t s, F &&launch) {
    if (!halo_fork(A, h, x, s)) {
        halo_exchange(h, x, s);
        launch(A.view());
        return;
    }
    const CsrView V = A.view();
    for (const auto &r : A.inner) launch(rows_view(V, r[0], r[1]));
    halo_join(s);
    for (const auto &r : A.outer) launch(rows_view(V, r[0], r[1]));
}
void gather_full(Gather *g, const double *own, double *full, cudaStream_t s);

// One classical-AMG level (reference amg.py:51-57).
struct AmgLevel {
    std::shared_ptr<const Csr> A;  // level operator (level 0 may be shared with MGR)
    Csr P;                         // interpolation n_l x n_{l+1}
    Csr R;                         // explicit P^T (restriction)
    DBuf<int8_t> is_c;             // C/F split
    DBuf<double> dtilde;           // l1 diagonal
    DBuf<int64_t> starts;          // partition boundaries (hybrid GS only)
    int64_t nparts = 0;
    bool jacobi = true;            // one row per partition
    // solve workspace
    DBuf<double> b, x, r, xo, xpre;
    // row distribution: owned rows start at ext position off; halo of this space
    int64_t off = 0;
    std::shared_ptr<Halo> halo;
};

// coarse end of the V-cycle as one dense operator (collapse.cu)
void collapse_tail(pmgr_amg &h, cudaStream_t s);
// largest level the collapse densifies (PMGR_COLLAPSE_ROWS, default 3584)
int64_t collapse_limit();

}  // namespace pmgr

struct pmgr_amg {
    pmgr_amg_cfg cfg;
    std::vector<pmgr::AmgLevel> levels;
    std::shared_ptr<const pmgr::Csr> coarse;  // coarsest operator
    pmgr::DBuf<double> coarse_inv;            // dense inverse, row-major
    pmgr::DBuf<double> cb, cx, ctmp;          // coarsest workspace
    int64_t flagged = 0;
    bool prof_tag = false;  // time level-0 smoother kernels (F-relax AMG of MGR level 0)
    int collapse_from = -1;          // levels >= this run as one dense operator (-1: none)
    pmgr::DBuf<double> collapsed;    // that operator, row-major n x collapsed_ld
    int64_t collapsed_ld = 0;
    // row distribution: the collapsed operator holds the owned rows only and
    // reads the full right-hand side gathered from every rank
    std::shared_ptr<pmgr::Gather> gather;
    pmgr::DBuf<double> full;
};

namespace pmgr {

struct DistSetup;
// dist: distributed setup of a partial operator (dsetup.cuh), null on one GPU
std::unique_ptr<pmgr_amg> amg_build(std::shared_ptr<const Csr> A, const pmgr_amg_cfg &cfg,
                                    cudaStream_t s, const DistSetup *dist = nullptr);
// out = V-cycle(h, b, x); x may be null (zero initial guess).  b/out are
// length n_0 device vectors; out may alias neither b nor x.
void amg_cycle(pmgr_amg &h, const double *b, const double *x, double *out, cudaStream_t s);
// zero-guess cycle on the right-hand side v[rows] (gather fused into the
// first sweep); false when the hierarchy cannot take that path
bool amg_cycle_rows(pmgr_amg &h, const double *v, const int64_t *rows, double *out, cudaStream_t s);
// l1-Jacobi entry of a hierarchy whose first step a producer fuses: the
// right-hand side goes to *b, b / dtilde to *x (false: not such a hierarchy)
bool amg_entry(pmgr_amg &h, double **b, double **x, const double **dtilde);
// V-cycle from zero once amg_entry's buffers are filled
void amg_cycle_prefilled(pmgr_amg &h, double *out, cudaStream_t s);

// on-device assembly of the synthetic Jacobian (assemble.cu)
std::shared_ptr<Csr> assemble_poromech(const pmgr_assembly &a, cudaStream_t s);

// Level-2 global smoother (smooth.cu; reference mgr.py:275-292)
struct GlobalSmoother {
    int kind = 0;  // PMGR_SMOOTHER_ILU / _HBGS
    int64_t n = 0, nparts = 1;
    DBuf<int64_t> starts;               // partition boundaries (align 2)
    Csr lu;                             // ILU(k): combined L\U, unit lower implicit
    DBuf<int64_t> dpos;                 // diagonal position per row
    bool leveled = false;               // substitutions by level schedule
    DBuf<int32_t> frows, brows;         // rows grouped by forward / backward level
    std::vector<int64_t> fptr, bptr;    // level boundaries
    std::shared_ptr<const Csr> A;       // HBGS: the level operator
    DBuf<double> add, xpre;             // off-partition |a| row sums, sweep copy
    DBuf<int64_t> cstart, cs, cp;       // cells per partition: s / p rows
    int nsweeps = 0;
};
std::unique_ptr<GlobalSmoother> smoother_build(std::shared_ptr<const Csr> A, int kind, int ilu_fill, int hbgs_sweeps,
                                               int64_t npartitions, bool interleaved, const int8_t *field_of,
                                               const int32_t *entity_of, cudaStream_t s);
void smoother_apply(GlobalSmoother &g, const double *v, double *z, cudaStream_t s);
// the smoother of the rows [lo, hi) of g's level for a rank that owns them:
// ILU(k) with one thread per partition only, and only when the partition
// boundaries fall on lo and hi (every partition then lives on one rank, the
// factors are the global ones row for row and the application is local)
std::unique_ptr<GlobalSmoother> smoother_slice(const GlobalSmoother &g, int64_t lo, int64_t hi, cudaStream_t s);

// One MGR reduction level (reference mgr.py:300-311).
struct MgrLevel {
    std::shared_ptr<const Csr> A;  // level operator
    int64_t n = 0, nc = 0, nf = 0;
    DBuf<int8_t> is_c;
    DBuf<int64_t> c_rows, f_rows;  // level-local row ids of C / F points
    DBuf<int64_t> f_index;         // row -> F index or -1
    Csr A_cf;                      // C rows x F cols (residual restriction)
    Csr P;                         // [W_p ; I] in level order
    DBuf<double> dinv_ff;          // 1 / diag(A_FF)
    int32_t f_relax = PMGR_FRELAX_NONE;
    int32_t f_relax_sweeps = 1;
    std::shared_ptr<const Csr> A_ff;  // for Jacobi sweeps > 1
    std::unique_ptr<pmgr_amg> amg;    // F-relaxation AMG
    std::unique_ptr<GlobalSmoother> smoother;  // optional global smoother
    Csr A_c;                          // C rows of A (residual after a global smoother)
    DBuf<double> zs, rr;              // smoother workspace
    // workspace
    DBuf<double> vf, zf, rc, zc, tmpf;
    // row distribution: owned offsets of the level (M), F and C spaces; halos
    // of the F space (read by A_CF) and of the C space (read by P)
    int64_t off = 0, off_f = 0, off_c = 0;
    std::shared_ptr<Halo> halo_f, halo_c;
    std::shared_ptr<Halo> halo_m;  // of the level space itself (read by A and A_c behind a global smoother)
};

}  // namespace pmgr

namespace pmgr {
// One instantiated CUDA graph of a full preconditioner application, keyed by
// its input/output buffers (GMRES always uses the same pair).
struct ApplyGraph {
    const double *v = nullptr;
    double *z = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool prof = false;               // captured with timing events
    bool pending = false;            // launched, events not yet collected
    std::vector<ProfRec> recs;
    uint64_t last_use = 0;
    int64_t kernels = 0;             // kernels per replay
};
}  // namespace pmgr

struct pmgr_mgr {
    ~pmgr_mgr();
    std::vector<pmgr::ApplyGraph> graphs;
    cudaStream_t cap_stream = nullptr;
    bool use_graphs = true;
    uint64_t tick = 0;
    std::vector<pmgr::MgrLevel> levels;
    std::shared_ptr<const pmgr::Csr> terminal_A;
    std::unique_ptr<pmgr_amg> terminal;
    int32_t terminal_cycles = 1;
    int32_t f_relax_post = 0;
    int64_t n = 0;
    int64_t block_prefix = 0;  // level-0 F rows: a node-blocked prefix of A0 (0: none)
    std::shared_ptr<const pmgr::Csr> block_src;  // level-0 A_FF with its BSR3 blocks
    bool dist = false;         // a rank's row slice of a hierarchy (dist.cu)
    pmgr::DBuf<double> tz;  // terminal scratch
};

namespace pmgr {
std::unique_ptr<pmgr_mgr> mgr_build(std::shared_ptr<const Csr> A, const int8_t *field_of_host,
                                    const int32_t *entity_of_host, const pmgr_level_spec *specs,
                                    int nlevels, const pmgr_mgr_cfg &cfg, cudaStream_t s,
                                    const DistSetup *dist = nullptr);
void mgr_apply(pmgr_mgr &h, const double *v, double *z, cudaStream_t s);
void mgr_collect(pmgr_mgr &h);  // fold finished graph timing events into the totals
void mgr_apply_direct(pmgr_mgr &h, const double *v, double *z, cudaStream_t s);  // no graph (for capture)
void mgr_apply_bytes(pmgr_mgr &h, double *bytes, int64_t *kernels);
}  // namespace pmgr

namespace pmgr {
void gmres_forget(const void *obj);  // drop cached solve workspaces of a matrix / hierarchy
void gmres_device(const pmgr_csr *A, pmgr_mgr *M, const double *b, double *x, int nonzero_x0,
                  const pmgr_gmres_cfg &cfg, pmgr_gmres_stats &stats, double *history,
                  int32_t history_cap, cudaStream_t s);
// GMRES over row-distributed vectors: the caller provides w = A M vin for
// the owned slices (halo exchanges inside), the owned-slice operators for the
// restart update and the cross-rank all-reduce (dist.cu)
struct SplitWs;  // persistent GMRES workspace + captured step (krylov.cu)
struct SplitOps {
    std::shared_ptr<SplitWs> *cache = nullptr;  // caller-owned slot, reused across solves
    int64_t n = 0;          // owned rows
    double *vin = nullptr;  // owned slice the preconditioner reads
    double *w = nullptr;    // owned slice the operator writes
    bool capturable = false;
    std::function<void(cudaStream_t)> step;
    std::function<void(const double *, double *, cudaStream_t)> spmv, apply;
    std::function<void(double *, int64_t, cudaStream_t)> allreduce;
};
void gmres_split(SplitOps &ops, const double *b, double *x, int nonzero_x0, const pmgr_gmres_cfg &cfg,
                 pmgr_gmres_stats &stats, double *history, int32_t history_cap, cudaStream_t s);
void multidot(const double *V, int64_t n, int32_t nvec, const double *w, double *h, cudaStream_t s);
void multiaxpy(const double *V, int64_t n, int32_t nvec, const double *h, double *w, cudaStream_t s);
double vec_norm2(const double *x, int64_t n, cudaStream_t s);
void vec_axpby(double a, const double *x, double b, double *y, int64_t n, cudaStream_t s);
void vec_combine(const double *V, int64_t n, int64_t ldv, int32_t nvec, const double *y, double *u, cudaStream_t s);
}  // namespace pmgr
