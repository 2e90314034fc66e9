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
    // setup-phase collectives (synchronising): one int64 to / from every rank,
    // and a personalised exchange of device byte ranges (peer p's send to me
    // lands in rptr[p]; sizes must match the peers' counts)
    virtual void alltoall_counts(const std::vector<int64_t> &send, std::vector<int64_t> &recv, cudaStream_t s) = 0;
    virtual void alltoallv(const std::vector<const void *> &sptr, const std::vector<int64_t> &sbytes,
                           const std::vector<void *> &rptr, const std::vector<int64_t> &rbytes, cudaStream_t s) = 0;
};

std::unique_ptr<Transport> make_nccl_transport(const pmgr_nccl_id &id, int rank, int nranks);
void nccl_unique_id(pmgr_nccl_id *out);
std::unique_ptr<Transport> make_callback_transport(int rank, int nranks, pmgr_alltoallv_fn a2a,
                                                   pmgr_allreduce_fn ared, void *ctx);

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
// distributed setup: A holds this rank's rows (global row space, the rest
// empty); field_of / entity_of are global (replicated); every rank calls
std::unique_ptr<DistSolver> dist_setup(const pmgr_csr *A, const int8_t *field_of, const int32_t *entity_of,
                                       const pmgr_level_spec *levels, int nlevels, const pmgr_mgr_cfg &cfg,
                                       const int64_t *bounds, int rank, int nranks, Transport *tr, cudaStream_t s);
// N ranks emulated on this GPU, distributed setup included (threads meet at
// every collective); what 0 = one MGR application, 1 = a GMRES solve
void dist_setup_emulate(const pmgr_csr *A, const int8_t *field_of, const int32_t *entity_of,
                        const pmgr_level_spec *levels, int nlevels, const pmgr_mgr_cfg &mcfg, const int64_t *bounds,
                        int nranks, int what, const double *in, double *out, const pmgr_gmres_cfg *cfg,
                        pmgr_gmres_stats *stats, cudaStream_t s);
void dist_apply(DistSolver &D, const double *v_own, double *z_own, cudaStream_t s);
void dist_gmres(DistSolver &D, const double *b, double *x, int nonzero_x0, const pmgr_gmres_cfg &cfg,
                pmgr_gmres_stats &st, double *history, int32_t history_cap, cudaStream_t s);
// N ranks emulated on this GPU (loopback transport, one host thread per
// rank): what 0 = one MGR application, 1 = a GMRES solve; in/out are global
void dist_emulate(const pmgr_csr *A, pmgr_mgr *M, const int64_t *bounds, int nranks, int what, const double *in,
                  double *out, const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats, cudaStream_t s);

}  // namespace pmgr
