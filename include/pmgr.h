/*
 * pmgr.h -- C ABI of libpmgr.so, the B200-native (sm_100a) MGR-preconditioned
 * GMRES hot path of arxiv/paper_1904_05960 (reference package `poromgr`).
 *
 * The reference has no FFI: its surface is the in-process Python API of
 * /root/reference/pkg/src/poromgr.  Each entry point below replaces one of
 * those Python functions (cited per declaration); the Python package
 * paper_1904_05960_b200 binds them through ctypes and reproduces the
 * reference signatures, exceptions and messages on top.
 *
 * Conventions
 *  - Plain pointers and sizes only.  `stream` is a cudaStream_t passed as
 *    void* (NULL = legacy default stream).  Pointers named *_dev are device
 *    pointers; *_host are host pointers.
 *  - Every call returns a pmgr_status.  On error, pmgr_last_error() gives a
 *    thread-local message and pmgr_last_error_index() the offending row (or
 *    -1); the Python layer maps codes to the reference exception types.
 *  - CSR: int64 row offsets, int32 column indices (strictly increasing per
 *    row), fp64 values -- the reference CsrMatrix dtypes (sparse.py:81-83).
 *  - Handles own device memory; apply/solve calls are asynchronous on the
 *    given stream and read-only over the hierarchy (one workspace per
 *    handle; use one handle per concurrent caller).
 */
#ifndef PMGR_H
#define PMGR_H

#include <stdint.h>

#if defined(__GNUC__)
#define PMGR_API __attribute__((visibility("default")))
#else
#define PMGR_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PMGR_OK = 0,
    PMGR_ERR_INVALID = 1,           /* ValueError (dimension, config, pattern)          */
    PMGR_ERR_SINGULAR_DIAG = 2,     /* ValueError "singular diagonal: zero or missing entry at row N" (sparse.py:407) */
    PMGR_ERR_L1_VANISHES = 3,       /* ValueError "l1 diagonal vanishes at row N" (smoothers.py:105) */
    PMGR_ERR_DENSE_CAP = 4,         /* RuntimeError coarsest level too large (amg.py:208-209) */
    PMGR_ERR_CUDA = 5,              /* RuntimeError from the CUDA runtime               */
    PMGR_ERR_NOT_SUPPORTED = 6,     /* NotImplementedError (option outside the hot path) */
    PMGR_ERR_OOM = 7,               /* MemoryError                                       */
    PMGR_ERR_INTERP_DIAG = 8,       /* ValueError "direct interpolation requires nonzero diagonals" (amg.py:137-138) */
    PMGR_ERR_FIELDS = 9,            /* ValueError level spec fields vs present fields (mgr.py:338-344) */
    PMGR_ERR_ZERO_PIVOT = 10        /* ZeroPivotError "zero pivot at row N" (smoothers.py:38)           */
} pmgr_status;

typedef struct pmgr_csr pmgr_csr;     /* device CSR matrix              (CsrMatrix, sparse.py:65)      */
typedef struct pmgr_amg pmgr_amg;     /* classical AMG hierarchy        (AmgHierarchy, amg.py:60)      */
typedef struct pmgr_mgr pmgr_mgr;     /* MGR hierarchy                  (MgrHierarchy, mgr.py:313)     */

/* ---- library ---------------------------------------------------------- */
PMGR_API int pmgr_version(void);
PMGR_API const char *pmgr_last_error(void);
PMGR_API int64_t pmgr_last_error_index(void);
/* Number of kernel launches issued by this library so far (bench evidence). */
PMGR_API int64_t pmgr_launch_count(void);
/* Device memory of destroyed matrices / hierarchies is kept in a block cache
 * and reused by the next setup (a repeated setup then allocates nothing);
 * this returns the cached blocks to the driver.  The reference has no
 * counterpart (NumPy arrays are freed by the garbage collector). */
PMGR_API int pmgr_release_cached_memory(void);

/* ---- sparse core (sparse.py) ------------------------------------------- */
/* Copy a CSR matrix (host or device arrays) into library-owned device memory.
 * Validates like CsrMatrix._validate (sparse.py:86-101) when validate != 0.
 * Replaces CsrMatrix(...) construction + to_scipy(). */
PMGR_API int pmgr_csr_create(int64_t nrows, int64_t ncols, int64_t nnz, const int64_t *row_offsets,
                    const int32_t *col_indices, const double *values, int on_device,
                    int validate, void *stream, pmgr_csr **out);
PMGR_API int pmgr_csr_destroy(pmgr_csr *A);
PMGR_API int pmgr_csr_info(const pmgr_csr *A, int64_t *nrows, int64_t *ncols, int64_t *nnz);
/* Copy the three CSR arrays out (host or device destination pointers). */
PMGR_API int pmgr_csr_download(const pmgr_csr *A, int64_t *row_offsets, int32_t *col_indices,
                      double *values, int to_device, void *stream);
/* y = A x, replaces sparse.matvec (sparse.py:261-266). */
/* B = P A P^T for a host permutation (row i of B = row perm[i] of A, columns
 * renumbered and sorted): problems.rank_major on the device. */
/* Rows [lo, hi) of A in A's row space (every other row empty): one rank's
 * slice for pmgr_dist_setup. */
PMGR_API int pmgr_csr_rows(const pmgr_csr *A, int64_t lo, int64_t hi, void *stream, pmgr_csr **out);
PMGR_API int pmgr_csr_permute(const pmgr_csr *A, const int64_t *perm_host, void *stream, pmgr_csr **out);
PMGR_API int pmgr_spmv(const pmgr_csr *A, const double *x_dev, double *y_dev, void *stream);

/* ---- classical AMG (amg.py) -------------------------------------------- */
typedef struct {
    double strength_threshold;   /* AmgConfig.strength_threshold (amg.py:37)  */
    int32_t max_levels;          /* AmgConfig.max_levels                      */
    int32_t coarse_size_cutoff;  /* AmgConfig.coarse_size_cutoff              */
    int32_t num_functions;       /* AmgConfig.num_functions                   */
    int32_t cycles;              /* AmgConfig.cycles                          */
    int64_t npartitions;         /* AmgConfig.npartitions (>= n: l1-Jacobi)   */
} pmgr_amg_cfg;

/* Replaces amg_setup (amg.py:184-211). */
PMGR_API int pmgr_amg_setup(const pmgr_csr *A, const pmgr_amg_cfg *cfg, void *stream, pmgr_amg **out);
PMGR_API int pmgr_amg_destroy(pmgr_amg *h);
/* Level count L (fine levels) ; sizes has L+1 entries (AmgHierarchy.level_sizes). */
PMGR_API int pmgr_amg_num_levels(const pmgr_amg *h, int32_t *nlevels);
PMGR_API int pmgr_amg_level_sizes(const pmgr_amg *h, int64_t *sizes);
PMGR_API int pmgr_amg_flagged_rows(const pmgr_amg *h, int64_t *flagged);
/* out = amg_vcycle(h, b, x) (amg.py:214-231); x_dev may be NULL for x = 0. */
PMGR_API int pmgr_amg_vcycle(pmgr_amg *h, const double *b_dev, const double *x_dev, double *out_dev,
                    void *stream);
/* Parity export of level `level`: what = 0 A_l, 1 P_l, 2 coarsest A.  Returns
 * a new pmgr_csr handle owned by the caller. */
PMGR_API int pmgr_amg_export_csr(const pmgr_amg *h, int32_t level, int32_t what, void *stream,
                        pmgr_csr **out);
/* what = 0: is_c (int8, n_l), 1: dtilde (fp64, n_l); host destination. */
PMGR_API int pmgr_amg_export_vec(const pmgr_amg *h, int32_t level, int32_t what, void *host_out,
                        void *stream);

/* ---- MGR (mgr.py) ------------------------------------------------------ */
enum { PMGR_INTERP_INJECTION_ONLY = 0, PMGR_INTERP_INJECTION_JACOBI = 1, PMGR_INTERP_IDEAL = 2 };
enum { PMGR_RESTRICT_INJECTION = 0, PMGR_RESTRICT_JACOBI = 1, PMGR_RESTRICT_IDEAL = 2 };
enum { PMGR_FRELAX_NONE = 0, PMGR_FRELAX_JACOBI = 1, PMGR_FRELAX_AMG = 2, PMGR_FRELAX_EXACT = 3 };
enum { PMGR_SMOOTHER_NONE = 0, PMGR_SMOOTHER_HBGS = 1, PMGR_SMOOTHER_ILU = 2 };

typedef struct {                 /* MgrLevelSpec (mgr.py:53-83)                 */
    uint64_t f_mask;             /* bit t set: field tag t is F on this level     */
    uint64_t c_mask;             /* bit t set: field tag t is C on this level     */
    int32_t interp;              /* PMGR_INTERP_*                                 */
    int32_t restrict_;           /* PMGR_RESTRICT_*                               */
    int32_t f_relax;             /* PMGR_FRELAX_*                                 */
    int32_t f_relax_sweeps;
    int32_t global_smoother;     /* PMGR_SMOOTHER_* (mgr.py:388-396)               */
    int32_t n_max;               /* < 0: no dropping (n_max=None)                 */
    int32_t quasi_impes;
    int32_t amg_num_functions;   /* F-relax AMG functions (3 when F = {U})        */
    int32_t ilu_fill;            /* MgrLevelSpec.ilu_fill (ILU(k) level of fill)   */
    int32_t hbgs_sweeps;         /* MgrLevelSpec.hbgs_sweeps                       */
} pmgr_level_spec;

typedef struct {                 /* MgrConfig (mgr.py:86-123)                     */
    int32_t terminal_cycles;
    int32_t f_relax_post;        /* 0: "pre", 1: "post"                           */
    pmgr_amg_cfg amg_f_relax;
    pmgr_amg_cfg amg_terminal;
    int64_t npartitions;         /* MgrConfig.npartitions (global smoothers)       */
    int32_t flow_interleaved;    /* FieldLayout.ordering == FLOW_INTERLEAVED       */
} pmgr_mgr_cfg;

/* Replaces mgr_setup (mgr.py:329-371).  field_of (int8) / entity_of (int32)
 * are host arrays of length n (FieldLayout, sparse.py:167-216). */
PMGR_API int pmgr_mgr_setup(const pmgr_csr *A, const int8_t *field_of, const int32_t *entity_of,
                   const pmgr_level_spec *levels, int32_t nlevels, const pmgr_mgr_cfg *cfg,
                   void *stream, pmgr_mgr **out);
PMGR_API int pmgr_mgr_destroy(pmgr_mgr *h);
/* MgrHierarchy.level_sizes (mgr.py:325): nlevels_built + 1 sizes. */
PMGR_API int pmgr_mgr_num_levels(const pmgr_mgr *h, int32_t *nlevels);
PMGR_API int pmgr_mgr_level_sizes(const pmgr_mgr *h, int64_t *sizes);
/* Algorithmic HBM bytes (SURVEY.md §8(d) per-pass rules, summed over every
 * operator pass, vector pass and dense collapsed product) and kernel count of
 * one mgr_apply; computed from a dry capture, nothing executes. */
PMGR_API int pmgr_mgr_apply_bytes(pmgr_mgr *h, double *bytes, int64_t *kernels);
/* z = mgr_apply(h, v) (mgr.py:399-429), device vectors. */
PMGR_API int pmgr_mgr_apply(pmgr_mgr *h, const double *v_dev, double *z_dev, void *stream);
/* Parity export: what = 0 P_l, 1 next coarse operator, 2 the level's ILU(k)
 * factors (combined L\U, IluFactors.lu); returns a new handle. */
PMGR_API int pmgr_mgr_export_csr(const pmgr_mgr *h, int32_t level, int32_t what, void *stream,
                        pmgr_csr **out);
/* what = 0: is_c (int8) of level `level` into host memory. */
PMGR_API int pmgr_mgr_export_vec(const pmgr_mgr *h, int32_t level, int32_t what, void *host_out,
                        void *stream);
/* AMG hierarchy used by level `level` (-1: terminal); borrowed pointer. */
PMGR_API int pmgr_mgr_amg(const pmgr_mgr *h, int32_t level, const pmgr_amg **out);

/* ---- Krylov (krylov.py) ------------------------------------------------ */
typedef struct {                 /* GmresConfig (krylov.py:18-29)                 */
    int32_t restart;
    int32_t max_iters;
    double rtol;
    double atol;
} pmgr_gmres_cfg;

typedef struct {                 /* SolveStats (krylov.py:32-36)                  */
    int32_t iterations;
    int32_t converged;
    int32_t history_len;         /* entries written to `history`                  */
    int32_t restarts;
} pmgr_gmres_stats;

/* Right-preconditioned restarted GMRES (krylov.py:39-117) with A and M both
 * library objects: the whole solve runs on the device.  M may be NULL
 * (identity).  x_dev holds x0 on entry (nonzero_x0 != 0) and the solution
 * on exit.  history_host receives residual_history (capacity history_cap). */
PMGR_API int pmgr_gmres(const pmgr_csr *A, pmgr_mgr *M, const double *b_dev, double *x_dev,
               int nonzero_x0, const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats,
               double *history_host, int32_t history_cap, void *stream);
/* Same solve with HOST b / x buffers: the host<->device copies are part of
 * the call (the end-to-end entry point a reference-side binding would use). */
PMGR_API int pmgr_gmres_host(const pmgr_csr *A, pmgr_mgr *M, const double *b_host, double *x_host,
                    int nonzero_x0, const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats,
                    double *history_host, int32_t history_cap, void *stream);

/* ---- live kernel timing ------------------------------------------------- */
/* Record CUDA events around selected launches (0 outer SpMV, 1 level-0
 * F-relax first sweep + residual, 2 level-0 F-relax post-sweep, 3 MGR apply,
 * 4 CGS2 step); enabling resets the record.  query returns the launch count,
 * summed device milliseconds and summed algorithmic bytes of one kind. */
PMGR_API int pmgr_prof_enable(int on);
PMGR_API int pmgr_prof_query(int32_t kind, int64_t *count, double *ms, double *bytes);

/* Device BLAS-1 helpers used by the generic (Python-callable) GMRES path:
 * h[k] = V_k . w for k < nvec (V row-major nvec x n); w -= sum_k h[k] V_k. */
PMGR_API int pmgr_multidot(const double *V_dev, int64_t n, int32_t nvec, const double *w_dev,
                  double *h_dev, void *stream);
PMGR_API int pmgr_multiaxpy(const double *V_dev, int64_t n, int32_t nvec, const double *h_dev,
                   double *w_dev, void *stream);
/* ||x||_2 of a device vector, returned on the host (synchronises the stream);
 * y = a x + b y (b = 0: y = a x, y's old contents ignored); u = sum_k y_k V_k
 * over nvec rows of V (leading dimension ldv, y on the device).  These replace
 * the reference's numpy vector algebra in krylov.py:52-117 on the generic
 * (Python-callable) GMRES path. */
PMGR_API int pmgr_vec_norm2(const double *x_dev, int64_t n, double *out_host, void *stream);
PMGR_API int pmgr_vec_axpby(double a, const double *x_dev, double b, double *y_dev, int64_t n, void *stream);
PMGR_API int pmgr_combine(const double *V_dev, int64_t n, int64_t ldv, int32_t nvec, const double *y_dev,
                          double *u_dev, void *stream);

/* ---- on-device assembly ---------------------------
 * The synthetic poromechanics Jacobian of paper_1904_05960_b200/problems.py
 * (Q1 elasticity, TPFA flow with upwinded Corey / Stone-I mobilities, Biot
 * coupling, bottom Dirichlet rows) assembled directly into device CSR from
 * host per-cell fields (arrays of nz*ny*nx, x fastest; sats nsat x cells)
 * and the 24x24 unit-E element stiffness / Biot vector; bitwise the host
 * generator's matrix. */
typedef struct {
    int32_t nx, ny, nz;
    int32_t phases;              /* 1 single, 2 two (s, p), 3 three (s, s2, p)   */
    double h, V;                 /* cell size and volume h**3 (host-rounded)     */
    double phi, ct, dt, biot;
    double mu[3];                /* phase viscosities                            */
    const double *E, *kx, *ky, *kz, *sats, *pstate;
    const double *K0;            /* 24 x 24 row-major */
    const double *bvec;          /* 24 */
} pmgr_assembly;
PMGR_API int pmgr_assemble_poromech(const pmgr_assembly *a, void *stream, pmgr_csr **out);

/* ---- row distribution (the reference is single-process) ---
 * Every rank builds the global A / MGR hierarchy on its own GPU (replicated
 * setup), then pmgr_dist_create keeps its rows of every operator.  `bounds`
 * (nranks + 1 entries) are the ranks' contiguous row ranges of a rank-major
 * numbered A (problems.rank_major); all coarser spaces inherit contiguous
 * ranges.  Exchange steps: halo exchange before each operator that reads
 * other ranks' entries, an all-gather of the collapsed coarse right-hand
 * side, all-reduces of the Krylov projections.  A distributed application is
 * bitwise identical to the single-GPU one. */
typedef struct { char internal[128]; } pmgr_nccl_id;   /* ncclUniqueId */
typedef struct pmgr_transport pmgr_transport;
typedef struct pmgr_dist pmgr_dist;
PMGR_API int pmgr_nccl_get_id(pmgr_nccl_id *out);
/* NCCL communicator over the process's libnccl (one GPU per rank). */
PMGR_API int pmgr_transport_nccl_create(const pmgr_nccl_id *id, int32_t rank, int32_t nranks,
                                        pmgr_transport **out);
/* Host-staged transport over caller-supplied collectives on HOST memory (for
 * example torch.distributed gloo): a personalised all-to-all (sptr[p] /
 * sbytes[p] to peer p, rptr[p] / rbytes[p] from peer p; self entries are 0)
 * and an in-place double all-reduce (sum, the same result on every rank).
 * Each callback returns 0 on success.  Every exchange synchronises the
 * stream -- slow by design: several processes can share one GPU. */
typedef int (*pmgr_alltoallv_fn)(void *ctx, const void *const *sptr, const int64_t *sbytes, void *const *rptr,
                                 const int64_t *rbytes);
typedef int (*pmgr_allreduce_fn)(void *ctx, double *buf, int64_t n);
PMGR_API int pmgr_transport_host_create(int32_t rank, int32_t nranks, pmgr_alltoallv_fn alltoallv,
                                        pmgr_allreduce_fn allreduce, void *ctx, pmgr_transport **out);
PMGR_API int pmgr_transport_destroy(pmgr_transport *t);
PMGR_API int pmgr_dist_create(const pmgr_csr *A, pmgr_mgr *M, const int64_t *bounds, int32_t rank,
                              int32_t nranks, pmgr_transport *t, void *stream, pmgr_dist **out);
/* Distributed setup (replaces mgr_setup, mgr.py:329-371, when the rows are
 * spread over ranks): A_rows is this rank's rows [bounds[rank],
 * bounds[rank+1]) of the rank-major global matrix, in the GLOBAL row space
 * (every other row empty); field_of / entity_of are the global layout.
 * Every rank calls it.  Each rank sets up the owned rows of every operator
 * (bitwise equal to the single-GPU rows: strength, MIS rounds with status
 * exchanges, interpolation, Galerkin products over fetched ghost rows) and
 * the coarse levels below PMGR_DIST_REPLICATE_ROWS (20000) redundantly. */
PMGR_API int pmgr_dist_setup(const pmgr_csr *A_rows, const int8_t *field_of, const int32_t *entity_of,
                             const pmgr_level_spec *levels, int32_t nlevels, const pmgr_mgr_cfg *cfg,
                             const int64_t *bounds, int32_t rank, int32_t nranks, pmgr_transport *t, void *stream,
                             pmgr_dist **out);
/* global index of the first owned row and the number of owned rows */
PMGR_API int pmgr_dist_info(const pmgr_dist *d, int64_t *lo, int64_t *n_own);
/* owned slices (n_own doubles) in and out */
PMGR_API int pmgr_dist_apply(pmgr_dist *d, const double *v_own_dev, double *z_own_dev, void *stream);
PMGR_API int pmgr_dist_spmv(pmgr_dist *d, const double *x_own_dev, double *y_own_dev, void *stream);
PMGR_API int pmgr_dist_gmres(pmgr_dist *d, const double *b_own_dev, double *x_own_dev, int nonzero_x0,
                             const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats, double *history_host,
                             int32_t history_cap, void *stream);
PMGR_API int pmgr_dist_destroy(pmgr_dist *d);
/* Test harness: nranks ranks emulated on this GPU (in-process loopback
 * transport, one host thread per rank).  what = 0: z = M v; what = 1: GMRES
 * from x0 = 0 (stats filled).  in / out are global device vectors. */
PMGR_API int pmgr_dist_emulate(const pmgr_csr *A, pmgr_mgr *M, const int64_t *bounds, int32_t nranks,
                               int32_t what, const double *in_dev, double *out_dev,
                               const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats, void *stream);
/* Same, with the distributed setup (pmgr_dist_setup) run by the emulated
 * ranks from their row slices of the global A. */
PMGR_API int pmgr_dist_setup_emulate(const pmgr_csr *A, const int8_t *field_of, const int32_t *entity_of,
                                     const pmgr_level_spec *levels, int32_t nlevels, const pmgr_mgr_cfg *mcfg,
                                     const int64_t *bounds, int32_t nranks, int32_t what, const double *in_dev,
                                     double *out_dev, const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats,
                                     void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PMGR_H */
