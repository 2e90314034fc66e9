// dist.cuh -- row-distributed solve phase (dist.cu).
#pragma once

#include <memory>
#include <vector>

#include "hier.cuh"

namespace pmgr {

// point-to-point halo exchange, all-gather and all-reduce of one rank
struct Transport {
    int rank = 0, nranks = 1;
    virtual ~Transport() {}
    virtual void exchange(Halo &h, double *ext, cudaStream_t s) = 0;
    virtual void gather(Gather &g, const double *own, double *full, cudaStream_t s) = 0;
    virtual void allreduce(double *buf, int64_t n, cudaStream_t s) = 0;
    virtual bool capturable() const { return false; }  // may be recorded into a CUDA graph
};

std::unique_ptr<Transport> make_nccl_transport(const pmgr_nccl_id &id, int rank, int nranks);
void nccl_unique_id(pmgr_nccl_id *out);

// one rank's slice of a global (A, MGR) pair
struct DistSolver {
    int rank = 0, nranks = 1;
    Transport *tr = nullptr;
    std::unique_ptr<Transport> own_tr;  // when the solver owns its transport
    int64_t n_global = 0, lo = 0, n_own = 0, off = 0, n_ext = 0;
    Csr A;                              // owned rows of A, ext columns
    std::shared_ptr<Halo> halo0;
    std::unique_ptr<pmgr_mgr> M;        // owned rows of every level
    std::vector<std::shared_ptr<Halo>> halos;
    std::vector<int> spaces;
    DBuf<double> ve, ze, we;            // ext workspaces of the level-0 space
    std::shared_ptr<SplitWs> gws;       // GMRES workspace / captured step
    void ensure_work();
};

std::unique_ptr<DistSolver> dist_build(const pmgr_csr *A, pmgr_mgr *M, const int64_t *bounds, int rank, int nranks,
                                       Transport *tr, cudaStream_t s);
void dist_apply(DistSolver &D, const double *v_own, double *z_own, cudaStream_t s);
void dist_gmres(DistSolver &D, const double *b, double *x, int nonzero_x0, const pmgr_gmres_cfg &cfg,
                pmgr_gmres_stats &st, double *history, int32_t history_cap, cudaStream_t s);
// N ranks emulated on this GPU (loopback transport, one host thread per
// rank): what 0 = one MGR application, 1 = a GMRES solve; in/out are global
void dist_emulate(const pmgr_csr *A, pmgr_mgr *M, const int64_t *bounds, int nranks, int what, const double *in,
                  double *out, const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats, cudaStream_t s);

}  // namespace pmgr
