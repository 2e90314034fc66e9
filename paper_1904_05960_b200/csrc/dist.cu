// dist.cu -- row-distributed solve phase.
//
// One process per GPU.  Every rank builds the global hierarchy (replicated
// setup: same kernels, same bits), then keeps only its rows of every operator:
//
// * numbering: level 0 is rank-major (problems.rank_major), so each rank owns
//   one contiguous global range of every space -- F/C splits and AMG C points
//   keep their relative order, so the ranges survive coarsening;
// * a rank stores a space as an "ext" vector: owned range plus the ghost
//   entries its local operators read, in global order.  Local rows therefore
//   sum their columns in the global stored order with the global operator's
//   lane group (and block layout), so a distributed application is bitwise
//   identical to the single-GPU one;
// * exchange steps: a halo exchange before every operator that reads ghosts
//   (point-to-point, only the neighbours that share entries), an all-gather
//   of the collapsed coarse right-hand side (a few thousand doubles), and the
//   all-reduces of the Krylov projections and norms.
//
// Transports: NCCL (loaded at run time, one GPU per rank) and an in-process
// loopback hub that emulates N ranks on one GPU for the parity tests (host
// threads meet at every exchange; the copies are ordinary stream-ordered
// kernels, no kernel ever waits on another rank).
#include <dlfcn.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>

#include <thrust/copy.h>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sort.h>
#include <thrust/unique.h>

#include "dist.cuh"
#include "dsetup.cuh"

namespace pmgr {

// =========================================================== transports

namespace {

__global__ void k_pull(double *__restrict__ dst, const double *__restrict__ src, const int64_t *__restrict__ idx,
                       int64_t n) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n) dst[t] = src[idx[t]];
}

constexpr int MAX_RANKS = 64;
struct PtrPack {
    double *p[MAX_RANKS];
};

__global__ void k_sum_ranks(PtrPack bufs, int nranks, int64_t n) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += bufs.p[r][t];  // rank order on every rank
    for (int r = 0; r < nranks; ++r) bufs.p[r][t] = s;
}

}  // namespace

// ---- loopback: N ranks of one process on one GPU and one stream ---------
struct LoopbackHub {
    int n;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool failed = false;
    std::string why;
    enum Kind { EXCHANGE, GATHER, ALLREDUCE, COUNTS, ALLTOALLV };
    struct Post {
        Kind kind;
        Halo *h = nullptr;
        Gather *g = nullptr;
        double *p = nullptr;
        const double *cp = nullptr;
        int64_t cnt = 0;
        const std::vector<int64_t> *csend = nullptr, *sbytes = nullptr, *rbytes = nullptr;
        std::vector<int64_t> *crecv = nullptr;
        const std::vector<const void *> *sptr = nullptr;
        const std::vector<void *> *rptr = nullptr;
    };
    std::vector<Post> posts;
    explicit LoopbackHub(int nr) : n(nr), posts(nr) {}

    void execute(cudaStream_t s) {
        const Kind k = posts[0].kind;
        for (auto &p : posts)
            if (p.kind != k) fail(PMGR_ERR_INVALID, "loopback ranks diverged (different collective order)");
        if (k == EXCHANGE) {
            for (int r = 0; r < n; ++r) {
                Halo &hr = *posts[r].h;
                for (size_t i = 0; i < hr.rpeer.size(); ++i) {
                    const int p = hr.rpeer[i];
                    Halo &hp = *posts[p].h;
                    auto it = std::find(hp.speer.begin(), hp.speer.end(), r);
                    if (it == hp.speer.end()) fail(PMGR_ERR_INVALID, "halo plans disagree");
                    const size_t j = (size_t)(it - hp.speer.begin());
                    if (hp.scnt[j] != hr.rcnt[i]) fail(PMGR_ERR_INVALID, "halo segment sizes disagree");
                    if (hr.rcnt[i] == 0) continue;
                    k_pull<<<grid_for(hr.rcnt[i], 256), 256, 0, s>>>(posts[r].p + hr.roff[i], posts[p].p + hp.off,
                                                                      hp.send_idx.p + hp.soff[j], hr.rcnt[i]);
                    PMGR_LAUNCHED();
                }
            }
        } else if (k == GATHER) {
            for (int r = 0; r < n; ++r) {
                Gather &g = *posts[r].g;
                for (int p = 0; p < n; ++p) {
                    const int64_t c = g.start[p + 1] - g.start[p];
                    if (c > 0)
                        PMGR_CUDA(cudaMemcpyAsync(posts[r].p + g.start[p], posts[p].cp, sizeof(double) * c,
                                                  cudaMemcpyDeviceToDevice, s));
                }
            }
        } else if (k == COUNTS) {
            for (int r = 0; r < n; ++r) {
                posts[r].crecv->assign(n, 0);
                for (int p = 0; p < n; ++p) (*posts[r].crecv)[p] = (*posts[p].csend)[r];
            }
        } else if (k == ALLTOALLV) {
            for (int r = 0; r < n; ++r)
                for (int p = 0; p < n; ++p) {
                    const int64_t b = (*posts[p].sbytes)[r];
                    if (b != (*posts[r].rbytes)[p]) fail(PMGR_ERR_INVALID, "loopback all-to-all sizes disagree");
                    if (b > 0)
                        PMGR_CUDA(cudaMemcpyAsync((*posts[r].rptr)[p], (*posts[p].sptr)[r], (size_t)b,
                                                  cudaMemcpyDeviceToDevice, s));
                }
        } else {
            if (n > MAX_RANKS) fail(PMGR_ERR_NOT_SUPPORTED, "loopback all-reduce: too many ranks");
            PtrPack pk;
            for (int r = 0; r < n; ++r) pk.p[r] = posts[r].p;
            const int64_t cnt = posts[0].cnt;
            if (cnt > 0) {
                k_sum_ranks<<<grid_for(cnt, 128), 128, 0, s>>>(pk, n, cnt);
                PMGR_LAUNCHED();
            }
        }
    }

    void arrive(int rank, const Post &p, cudaStream_t s) {
        std::unique_lock<std::mutex> lk(m);
        if (failed) fail(PMGR_ERR_CUDA, "loopback peer failed: " + why);
        posts[rank] = p;
        const uint64_t my = gen;
        if (++arrived == n) {
            try {
                execute(s);
                if (p.kind == EXCHANGE) PMGR_CUDA(cudaStreamSynchronize(s));  // see LoopbackTransport::exchange
            } catch (const Error &e) {
                failed = true;
                why = e.msg;
            }
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != my || failed; });
        }
        if (failed) fail(PMGR_ERR_CUDA, "loopback exchange failed: " + why);
    }

    void abort(const std::string &w) {
        std::lock_guard<std::mutex> lk(m);
        if (!failed) {
            failed = true;
            why = w;
        }
        cv.notify_all();
    }
};

struct LoopbackTransport : Transport {
    LoopbackHub *hub;
    LoopbackTransport(LoopbackHub *h, int r) : hub(h) {
        rank = r;
        nranks = h->n;
    }
    void exchange(Halo &h, double *ext, cudaStream_t s) override {
        // s may be a rank's side stream (with_halo): every rank's producers
        // must be done before the last arriver copies, and the copies done
        // before any rank proceeds (the emulated ranks share one main stream)
        PMGR_CUDA(cudaStreamSynchronize(s));
        LoopbackHub::Post p;
        p.kind = LoopbackHub::EXCHANGE;
        p.h = &h;
        p.p = ext;
        hub->arrive(rank, p, s);
        PMGR_CUDA(cudaStreamSynchronize(s));
    }
    void gather(Gather &g, const double *own, double *full, cudaStream_t s) override {
        LoopbackHub::Post p;
        p.kind = LoopbackHub::GATHER;
        p.g = &g;
        p.cp = own;
        p.p = full;
        hub->arrive(rank, p, s);
    }
    void allreduce(double *buf, int64_t n, cudaStream_t s) override {
        LoopbackHub::Post p;
        p.kind = LoopbackHub::ALLREDUCE;
        p.p = buf;
        p.cnt = n;
        hub->arrive(rank, p, s);
    }
    void alltoall_counts(const std::vector<int64_t> &send, std::vector<int64_t> &recv, cudaStream_t s) override {
        LoopbackHub::Post p;
        p.kind = LoopbackHub::COUNTS;
        p.csend = &send;
        p.crecv = &recv;
        hub->arrive(rank, p, s);
    }
    void alltoallv(const std::vector<const void *> &sptr, const std::vector<int64_t> &sbytes,
                   const std::vector<void *> &rptr, const std::vector<int64_t> &rbytes, cudaStream_t s) override {
        LoopbackHub::Post p;
        p.kind = LoopbackHub::ALLTOALLV;
        p.sptr = &sptr;
        p.sbytes = &sbytes;
        p.rptr = &rptr;
        p.rbytes = &rbytes;
        hub->arrive(rank, p, s);
        PMGR_CUDA(cudaStreamSynchronize(s));
    }
};

// ---- NCCL, resolved at run time (the process's libnccl, e.g. torch's) ----
namespace {
typedef int nres_t;  // ncclResult_t
struct NcclApi {
    void *h = nullptr;
    nres_t (*GetUniqueId)(void *) = nullptr;
    nres_t (*CommInitRank)(void **, int, pmgr_nccl_id, int) = nullptr;
    nres_t (*CommDestroy)(void *) = nullptr;
    nres_t (*GroupStart)() = nullptr;
    nres_t (*GroupEnd)() = nullptr;
    nres_t (*Send)(const void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    nres_t (*Recv)(void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    nres_t (*AllReduce)(const void *, void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(nres_t) = nullptr;
};
constexpr int NCCL_FLOAT64 = 8;  // ncclFloat64 / ncclDouble
constexpr int NCCL_INT8 = 0;     // ncclInt8 / ncclChar
constexpr int NCCL_SUM = 0;      // ncclSum

NcclApi &nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *nm : names) {
            api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
            if (!api.h) api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) return;
        api.GetUniqueId = (nres_t(*)(void *))dlsym(api.h, "ncclGetUniqueId");
        api.CommInitRank = (nres_t(*)(void **, int, pmgr_nccl_id, int))dlsym(api.h, "ncclCommInitRank");
        api.CommDestroy = (nres_t(*)(void *))dlsym(api.h, "ncclCommDestroy");
        api.GroupStart = (nres_t(*)())dlsym(api.h, "ncclGroupStart");
        api.GroupEnd = (nres_t(*)())dlsym(api.h, "ncclGroupEnd");
        api.Send = (nres_t(*)(const void *, size_t, int, int, void *, cudaStream_t))dlsym(api.h, "ncclSend");
        api.Recv = (nres_t(*)(void *, size_t, int, int, void *, cudaStream_t))dlsym(api.h, "ncclRecv");
        api.AllReduce =
            (nres_t(*)(const void *, void *, size_t, int, int, void *, cudaStream_t))dlsym(api.h, "ncclAllReduce");
        api.GetErrorString = (const char *(*)(nres_t))dlsym(api.h, "ncclGetErrorString");
    });
    if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.AllReduce)
        fail(PMGR_ERR_NOT_SUPPORTED, "NCCL is not loadable in this process (libnccl.so.2)");
    return api;
}

void nccl_check(nres_t r, const char *what) {
    if (r != 0) {
        const char *msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
        fail(PMGR_ERR_CUDA, std::string(what) + ": " + msg);
    }
}

__global__ void k_pack(double *__restrict__ dst, const double *__restrict__ src, const int64_t *__restrict__ idx,
                       int64_t n) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n) dst[t] = src[idx[t]];
}
}  // namespace

void nccl_unique_id(pmgr_nccl_id *out) { nccl_check(nccl().GetUniqueId(out), "ncclGetUniqueId"); }

struct NcclTransport : Transport {
    void *comm = nullptr;
    NcclTransport(const pmgr_nccl_id &id, int r, int nr) {
        rank = r;
        nranks = nr;
        nccl_check(nccl().CommInitRank(&comm, nr, id, r), "ncclCommInitRank");
    }
    ~NcclTransport() override {
        if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
    }
    void exchange(Halo &h, double *ext, cudaStream_t s) override {
        const int64_t ns = h.send_idx.n;
        if (ns > 0) {
            k_pack<<<grid_for(ns, 256), 256, 0, s>>>(h.sbuf.p, ext + h.off, h.send_idx.p, ns);
            PMGR_LAUNCHED();
        }
        NcclApi &a = nccl();
        nccl_check(a.GroupStart(), "ncclGroupStart");
        for (size_t i = 0; i < h.speer.size(); ++i)
            if (h.scnt[i] > 0)
                nccl_check(a.Send(h.sbuf.p + h.soff[i], (size_t)h.scnt[i], NCCL_FLOAT64, h.speer[i], comm, s),
                           "ncclSend");
        for (size_t i = 0; i < h.rpeer.size(); ++i)
            if (h.rcnt[i] > 0)
                nccl_check(a.Recv(ext + h.roff[i], (size_t)h.rcnt[i], NCCL_FLOAT64, h.rpeer[i], comm, s),
                           "ncclRecv");
        nccl_check(a.GroupEnd(), "ncclGroupEnd");
    }
    void gather(Gather &g, const double *own, double *full, cudaStream_t s) override {
        const int64_t mine = g.start[rank + 1] - g.start[rank];
        if (mine > 0)
            PMGR_CUDA(cudaMemcpyAsync(full + g.start[rank], own, sizeof(double) * mine, cudaMemcpyDeviceToDevice, s));
        NcclApi &a = nccl();
        nccl_check(a.GroupStart(), "ncclGroupStart");
        for (int p = 0; p < nranks; ++p) {
            if (p == rank) continue;
            const int64_t c = g.start[p + 1] - g.start[p];
            if (mine > 0) nccl_check(a.Send(own, (size_t)mine, NCCL_FLOAT64, p, comm, s), "ncclSend");
            if (c > 0) nccl_check(a.Recv(full + g.start[p], (size_t)c, NCCL_FLOAT64, p, comm, s), "ncclRecv");
        }
        nccl_check(a.GroupEnd(), "ncclGroupEnd");
    }
    void allreduce(double *buf, int64_t n, cudaStream_t s) override {
        if (n <= 0) return;
        nccl_check(nccl().AllReduce(buf, buf, (size_t)n, NCCL_FLOAT64, NCCL_SUM, comm, s), "ncclAllReduce");
    }
    bool capturable() const override { return true; }
    void alltoall_counts(const std::vector<int64_t> &send, std::vector<int64_t> &recv, cudaStream_t s) override {
        TBuf<int64_t> sb(nranks, s), rb(nranks, s);
        PMGR_CUDA(cudaMemcpyAsync(sb.p, send.data(), sizeof(int64_t) * nranks, cudaMemcpyHostToDevice, s));
        std::vector<const void *> sp(nranks);
        std::vector<void *> rp(nranks);
        std::vector<int64_t> by(nranks, 8);
        for (int p = 0; p < nranks; ++p) {
            sp[p] = sb.p + p;
            rp[p] = rb.p + p;
        }
        alltoallv(sp, by, rp, by, s);
        recv.assign(nranks, 0);
        PMGR_CUDA(cudaMemcpyAsync(recv.data(), rb.p, sizeof(int64_t) * nranks, cudaMemcpyDeviceToHost, s));
        PMGR_CUDA(cudaStreamSynchronize(s));
    }
    void alltoallv(const std::vector<const void *> &sptr, const std::vector<int64_t> &sbytes,
                   const std::vector<void *> &rptr, const std::vector<int64_t> &rbytes, cudaStream_t s) override {
        if (sbytes[rank] != rbytes[rank]) fail(PMGR_ERR_INVALID, "all-to-all self sizes disagree");
        if (sbytes[rank] > 0)
            PMGR_CUDA(cudaMemcpyAsync(rptr[rank], sptr[rank], (size_t)sbytes[rank], cudaMemcpyDeviceToDevice, s));
        NcclApi &a = nccl();
        nccl_check(a.GroupStart(), "ncclGroupStart");
        for (int p = 0; p < nranks; ++p) {
            if (p == rank) continue;
            if (sbytes[p] > 0) nccl_check(a.Send(sptr[p], (size_t)sbytes[p], NCCL_INT8, p, comm, s), "ncclSend");
            if (rbytes[p] > 0) nccl_check(a.Recv(rptr[p], (size_t)rbytes[p], NCCL_INT8, p, comm, s), "ncclRecv");
        }
        nccl_check(a.GroupEnd(), "ncclGroupEnd");
        PMGR_CUDA(cudaStreamSynchronize(s));
    }
};

std::unique_ptr<Transport> make_nccl_transport(const pmgr_nccl_id &id, int rank, int nranks) {
    return std::unique_ptr<Transport>(new NcclTransport(id, rank, nranks));
}

// ---- host-staged transport over caller-supplied collectives --------------
// (e.g. torch.distributed gloo on CPU tensors): every exchange packs on the
// device, copies to pinned host buffers, synchronises the stream, runs the
// caller's personalised all-to-all / all-reduce on host memory and copies the
// received data back.  Synchronous and slow by design -- it lets several
// processes share one GPU (no kernel ever waits on another process) and
// exercises the multi-process setup and solve end to end without NCCL.
struct CallbackTransport : Transport {
    pmgr_alltoallv_fn a2a;
    pmgr_allreduce_fn ared;
    void *ctx;
    std::vector<char> hs, hr;  // host staging (pageable: cudaMemcpy synchronous)
    CallbackTransport(int r, int nr, pmgr_alltoallv_fn f, pmgr_allreduce_fn g, void *c) : a2a(f), ared(g), ctx(c) {
        rank = r;
        nranks = nr;
    }
    // host all-to-all: sbytes[p] from hsend + soff[p] to peer p, rbytes[p] into hrecv + roff[p]
    void host_a2a(const std::vector<int64_t> &sbytes, const std::vector<int64_t> &rbytes, char *hsend, char *hrecv) {
        std::vector<const void *> sp(nranks);
        std::vector<void *> rp(nranks);
        int64_t so = 0, ro = 0;
        for (int p = 0; p < nranks; ++p) {
            sp[p] = hsend + so;
            rp[p] = hrecv + ro;
            so += sbytes[p];
            ro += rbytes[p];
        }
        if (sbytes[rank] != rbytes[rank]) fail(PMGR_ERR_INVALID, "host transport: self sizes disagree");
        if (sbytes[rank] > 0) std::memcpy(rp[rank], sp[rank], (size_t)sbytes[rank]);  // the callback skips self
        if (a2a(ctx, sp.data(), sbytes.data(), rp.data(), rbytes.data()) != 0)
            fail(PMGR_ERR_CUDA, "host transport: all-to-all callback failed");
    }
    void exchange(Halo &h, double *ext, cudaStream_t s) override {
        const int64_t ns = h.send_idx.n;
        if (ns > 0) {
            k_pack<<<grid_for(ns, 256), 256, 0, s>>>(h.sbuf.p, ext + h.off, h.send_idx.p, ns);
            PMGR_LAUNCHED();
        }
        std::vector<int64_t> sb(nranks, 0), rb(nranks, 0), so(nranks, 0), ro(nranks, 0);
        for (size_t i = 0; i < h.speer.size(); ++i) {
            sb[h.speer[i]] = 8 * h.scnt[i];
            so[h.speer[i]] = h.soff[i];
        }
        for (size_t i = 0; i < h.rpeer.size(); ++i) {
            rb[h.rpeer[i]] = 8 * h.rcnt[i];
            ro[h.rpeer[i]] = h.roff[i];
        }
        int64_t st = 0, rt = 0;
        for (int p = 0; p < nranks; ++p) {
            st += sb[p];
            rt += rb[p];
        }
        hs.resize(st > 0 ? st : 1);
        hr.resize(rt > 0 ? rt : 1);
        int64_t o = 0;
        for (int p = 0; p < nranks; ++p) {  // device send buffer -> host, peer order
            if (sb[p]) PMGR_CUDA(cudaMemcpyAsync(hs.data() + o, h.sbuf.p + so[p], sb[p], cudaMemcpyDeviceToHost, s));
            o += sb[p];
        }
        PMGR_CUDA(cudaStreamSynchronize(s));
        host_a2a(sb, rb, hs.data(), hr.data());
        o = 0;
        for (int p = 0; p < nranks; ++p) {
            if (rb[p]) PMGR_CUDA(cudaMemcpyAsync(ext + ro[p], hr.data() + o, rb[p], cudaMemcpyHostToDevice, s));
            o += rb[p];
        }
        PMGR_CUDA(cudaStreamSynchronize(s));
    }
    void gather(Gather &g, const double *own, double *full, cudaStream_t s) override {
        const int64_t mine = g.start[rank + 1] - g.start[rank];
        std::vector<int64_t> sb(nranks), rb(nranks);
        for (int p = 0; p < nranks; ++p) {
            sb[p] = p == rank ? 0 : 8 * mine;
            rb[p] = p == rank ? 0 : 8 * (g.start[p + 1] - g.start[p]);
        }
        hs.resize(8 * mine * (nranks - 1) + 1);
        hr.resize(8 * (g.n_full - mine) + 1);
        if (mine > 0) {
            PMGR_CUDA(cudaMemcpyAsync(full + g.start[rank], own, 8 * mine, cudaMemcpyDeviceToDevice, s));
            PMGR_CUDA(cudaMemcpyAsync(hs.data(), own, 8 * mine, cudaMemcpyDeviceToHost, s));
        }
        PMGR_CUDA(cudaStreamSynchronize(s));
        for (int c = 1; c < nranks - 1; ++c) std::memcpy(hs.data() + 8 * mine * c, hs.data(), 8 * mine);
        host_a2a(sb, rb, hs.data(), hr.data());
        int64_t o = 0;
        for (int p = 0; p < nranks; ++p) {
            if (rb[p]) PMGR_CUDA(cudaMemcpyAsync(full + g.start[p], hr.data() + o, rb[p], cudaMemcpyHostToDevice, s));
            o += rb[p];
        }
        PMGR_CUDA(cudaStreamSynchronize(s));
    }
    void allreduce(double *buf, int64_t n, cudaStream_t s) override {
        if (n <= 0) return;
        std::vector<double> hb(n);
        PMGR_CUDA(cudaMemcpyAsync(hb.data(), buf, 8 * n, cudaMemcpyDeviceToHost, s));
        PMGR_CUDA(cudaStreamSynchronize(s));
        if (ared(ctx, hb.data(), n) != 0) fail(PMGR_ERR_CUDA, "host transport: all-reduce callback failed");
        PMGR_CUDA(cudaMemcpyAsync(buf, hb.data(), 8 * n, cudaMemcpyHostToDevice, s));
        PMGR_CUDA(cudaStreamSynchronize(s));
    }
    void alltoall_counts(const std::vector<int64_t> &send, std::vector<int64_t> &recv, cudaStream_t) override {
        std::vector<int64_t> by(nranks, 8);
        recv.assign(nranks, 0);
        host_a2a(by, by, (char *)send.data(), (char *)recv.data());
    }
    void alltoallv(const std::vector<const void *> &sptr, const std::vector<int64_t> &sbytes,
                   const std::vector<void *> &rptr, const std::vector<int64_t> &rbytes, cudaStream_t s) override {
        int64_t st = 0, rt = 0;
        for (int p = 0; p < nranks; ++p) {
            st += sbytes[p];
            rt += rbytes[p];
        }
        std::vector<char> sh(st > 0 ? st : 1), rh(rt > 0 ? rt : 1);
        int64_t o = 0;
        for (int p = 0; p < nranks; ++p) {
            if (sbytes[p]) PMGR_CUDA(cudaMemcpyAsync(sh.data() + o, sptr[p], sbytes[p], cudaMemcpyDeviceToHost, s));
            o += sbytes[p];
        }
        PMGR_CUDA(cudaStreamSynchronize(s));
        host_a2a(sbytes, rbytes, sh.data(), rh.data());
        o = 0;
        for (int p = 0; p < nranks; ++p) {
            if (rbytes[p]) PMGR_CUDA(cudaMemcpyAsync(rptr[p], rh.data() + o, rbytes[p], cudaMemcpyHostToDevice, s));
            o += rbytes[p];
        }
        PMGR_CUDA(cudaStreamSynchronize(s));
    }
};

std::unique_ptr<Transport> make_callback_transport(int rank, int nranks, pmgr_alltoallv_fn a2a,
                                                   pmgr_allreduce_fn ared, void *ctx) {
    return std::unique_ptr<Transport>(new CallbackTransport(rank, nranks, a2a, ared, ctx));
}

void halo_exchange(Halo *h, double *ext, cudaStream_t s) {
    if (h && h->tr) h->tr->exchange(*h, ext, s);
}

namespace {
struct OverlapCtx {  // per thread (one rank per thread in the emulation) and device
    int dev = -1;
    cudaStream_t cs = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
thread_local OverlapCtx g_ov;

bool overlap_enabled() {
    static const bool on = !(getenv("PMGR_OVERLAP") && getenv("PMGR_OVERLAP")[0] == '0');
    return on;
}
}  // namespace

bool halo_fork(const Csr &A, Halo *h, double *x, cudaStream_t s) {
    if (!h || !h->tr || A.inner.empty() || !overlap_enabled()) return false;
    int dev = 0;
    PMGR_CUDA(cudaGetDevice(&dev));
    if (g_ov.dev != dev) {
        PMGR_CUDA(cudaStreamCreateWithFlags(&g_ov.cs, cudaStreamNonBlocking));
        PMGR_CUDA(cudaEventCreateWithFlags(&g_ov.fork, cudaEventDisableTiming));
        PMGR_CUDA(cudaEventCreateWithFlags(&g_ov.join, cudaEventDisableTiming));
        g_ov.dev = dev;
    }
    PMGR_CUDA(cudaEventRecord(g_ov.fork, s));
    PMGR_CUDA(cudaStreamWaitEvent(g_ov.cs, g_ov.fork, 0));
    h->tr->exchange(*h, x, g_ov.cs);
    PMGR_CUDA(cudaEventRecord(g_ov.join, g_ov.cs));
    return true;
}

void halo_join(cudaStream_t s) { PMGR_CUDA(cudaStreamWaitEvent(s, g_ov.join, 0)); }

namespace {
__global__ void k_row_ghost(int64_t n, const int64_t *__restrict__ ro, const int32_t *__restrict__ ci, int64_t lo,
                            int64_t hi, int8_t *flag) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    int g = 0;
    for (int64_t q = ro[i] + lane; q < ro[i + 1]; q += 32) g |= (ci[q] < lo || ci[q] >= hi);
    g = __any_sync(FULL, g);
    if (lane == 0) flag[i] = (int8_t)g;
}
}  // namespace

// split a localized operator's rows into contiguous interior / boundary
// ranges (row triples for block operators); operators whose rows interleave
// too finely, or that route long rows through per-row blocks, keep no split
void classify_overlap(Csr &A, int64_t col_lo, int64_t col_hi, cudaStream_t s) {
    A.inner.clear();
    A.outer.clear();
    const int64_t n = A.nrows;
    if (n == 0 || (A.long_len > 0 && A.nlong > 0)) return;
    const bool blocks = A.nbrows > 0;
    if (blocks && (A.nbrows * 3 != n || A.rro.p)) return;
    TBuf<int8_t> f(n, s);
    k_row_ghost<<<grid_for(n * 32, 256), 256, 0, s>>>(n, A.ro.p, A.ci.p, col_lo, col_hi, f.p);
    PMGR_LAUNCHED();
    std::vector<int8_t> h(n);
    PMGR_CUDA(cudaMemcpyAsync(h.data(), f.p, n, cudaMemcpyDeviceToHost, s));
    PMGR_CUDA(cudaStreamSynchronize(s));
    const int64_t step = blocks ? 3 : 1;
    std::vector<std::array<int64_t, 2>> in, out;
    for (int64_t r = 0; r < n;) {
        int g = 0;
        for (int64_t k = 0; k < step; ++k) g |= h[r + k];
        int64_t e = r + step;
        while (e < n) {
            int ge = 0;
            for (int64_t k = 0; k < step; ++k) ge |= h[e + k];
            if (ge != g) break;
            e += step;
        }
        (g ? out : in).push_back({r, e});
        r = e;
    }
    if (in.empty() || in.size() + out.size() > 16) return;
    static const bool stats = getenv("PMGR_HIER_STATS") && getenv("PMGR_HIER_STATS")[0] != '0';
    if (stats) {
        int64_t ri = 0, ro_ = 0;
        for (auto &r : in) ri += r[1] - r[0];
        for (auto &r : out) ro_ += r[1] - r[0];
        fprintf(stderr, "[pmgr] overlap split %lld rows: inner %lld in %zu ranges, outer %lld in %zu ranges\n",
                (long long)n, (long long)ri, in.size(), (long long)ro_, out.size());
    }
    A.inner = std::move(in);
    A.outer = std::move(out);
}

void gather_full(Gather *g, const double *own, double *full, cudaStream_t s) {
    if (g->tr) {
        g->tr->gather(*g, own, full, s);
    } else {
        const int64_t c = g->n_full;
        if (c > 0) PMGR_CUDA(cudaMemcpyAsync(full, own, sizeof(double) * c, cudaMemcpyDeviceToDevice, s));
    }
}

// ===================================================== local hierarchy

namespace {

// a vector space of the global hierarchy as seen by one rank
struct Space {
    int id = -1;
    int64_t n = 0;                 // global size
    std::vector<int64_t> start;    // nranks + 1 global range starts
    std::vector<std::vector<int64_t>> ghosts;  // per rank, sorted global ids
    bool triples = false;          // close ghost sets under node triples (BSR operators)
    DBuf<int64_t> gdev;            // my ghosts on the device
    int64_t lo = 0, hi = 0, nlow = 0;
    int64_t pad = 0;               // gap before the owned range: off() is a multiple of 96
    int64_t off() const { return nlow + pad; }
    std::shared_ptr<Halo> halo;
    int64_t n_own() const { return hi - lo; }
    int64_t n_ext() const { return (int64_t)ghosts_me->size() + pad + n_own(); }
    const std::vector<int64_t> *ghosts_me = nullptr;
};

struct Reader {
    const Csr *Y;
    Space *rows;
};

__global__ void k_mark_outside(int64_t n, const int64_t *ro, int64_t r0, const int32_t *ci, int64_t c0, int64_t c1,
                               int64_t *out, int64_t *cnt) {
    // collect columns outside [c0, c1) of rows [r0, r0 + n)
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int64_t q = ro[r0 + i]; q < ro[r0 + i + 1]; ++q) {
        const int64_t c = ci[q];
        if (c < c0 || c >= c1) out[atomicAdd((unsigned long long *)cnt, 1ull)] = c;
    }
}

__global__ void k_localize(int64_t n, const int64_t *ro, int64_t r0, const int32_t *ci, const double *v, int64_t c0,
                           int64_t c1, int64_t nlow, int64_t pad, const int64_t *ghosts, int64_t ng, int64_t *lro,
                           int32_t *lci,
                           double *lv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    const int64_t base = ro[r0];
    lro[i] = ro[r0 + i] - base;
    if (i == n) return;
    for (int64_t q = ro[r0 + i]; q < ro[r0 + i + 1]; ++q) {
        const int64_t c = ci[q];
        int64_t pos;
        if (c >= c0 && c < c1) {
            pos = nlow + pad + (c - c0);
        } else {
            int64_t a = 0, b = ng;  // lower_bound in the sorted ghost list
            while (a < b) {
                const int64_t m = (a + b) >> 1;
                if (ghosts[m] < c) a = m + 1;
                else b = m;
            }
            pos = a < nlow ? a : a + pad + (c1 - c0);
        }
        lci[q - base] = (int32_t)pos;
        lv[q - base] = v[q];
    }
}

// level-local index maps: out[off_o + t] = map(in[g_lo + t]) for the owned entries
__global__ void k_map_owned(int64_t n, const int64_t *in, int64_t g_lo, int64_t in_lo, int64_t in_off, int64_t *out,
                            int64_t off_o, int keep_negative) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int64_t g = in[g_lo + t];
    out[off_o + t] = (keep_negative && g < 0) ? -1 : in_off + (g - in_lo);
}

__global__ void k_count_sel(int64_t n, const int8_t *is_c, int want, int64_t *o) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) o[i] = (is_c[i] != 0) == (want != 0) ? 1 : 0;
}

}  // namespace

struct Builder {
    int rank, nranks;
    Transport *tr;
    cudaStream_t s;
    std::vector<std::unique_ptr<Space>> spaces;
    std::vector<std::vector<Reader>> readers;  // per space id

    // partial: the operators hold this rank's rows only (distributed setup);
    // ghost lists then travel to their owners instead of being derived from
    // every rank's rows
    bool partial = false;

    Builder(int r, int nr, Transport *t, cudaStream_t st) : rank(r), nranks(nr), tr(t), s(st) {}

    Space *root(int64_t n, const int64_t *bounds) {
        auto sp = std::make_unique<Space>();
        sp->id = (int)spaces.size();
        sp->n = n;
        sp->start.assign(bounds, bounds + nranks + 1);
        if (sp->start[0] != 0 || sp->start[nranks] != n)
            fail(PMGR_ERR_INVALID, "rank bounds must cover [0, n)");
        for (int r = 0; r < nranks; ++r)
            if (sp->start[r + 1] < sp->start[r]) fail(PMGR_ERR_INVALID, "rank bounds must be non-decreasing");
        spaces.push_back(std::move(sp));
        readers.emplace_back();
        return spaces.back().get();
    }

    // entries of `parent` with (is_c != 0) == want, in order
    Space *derive(const Space *parent, const int8_t *is_c, bool want) {
        const int64_t n = parent->n;
        TBuf<int64_t> sel(n > 0 ? n : 1, s), sc(n + 1, s);
        if (n > 0) {
            k_count_sel<<<grid_for(n, 256), 256, 0, s>>>(n, is_c, want ? 1 : 0, sel.p);
            PMGR_LAUNCHED();
        }
        const int64_t tot = exclusive_scan_total(sel.p, sc.p, n, s);
        std::vector<int64_t> hsc(n + 1);
        PMGR_CUDA(cudaMemcpyAsync(hsc.data(), sc.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
        PMGR_CUDA(cudaStreamSynchronize(s));
        hsc[n] = tot;
        auto sp = std::make_unique<Space>();
        sp->id = (int)spaces.size();
        sp->n = tot;
        sp->start.resize(nranks + 1);
        for (int r = 0; r <= nranks; ++r) sp->start[r] = hsc[parent->start[r]];
        spaces.push_back(std::move(sp));
        readers.emplace_back();
        return spaces.back().get();
    }

    void read(Space *cols, const Csr *Y, Space *rows) { readers[cols->id].push_back({Y, rows}); }

    // partial mode: every rank learns which of its entries each peer reads
    // (ghosts[q] keeps the part of q's ghost list this rank owns)
    void exchange_ghosts(Space *sp) {
        const std::vector<int64_t> mine = sp->ghosts[rank];
        std::vector<int64_t> scnt(nranks), soff(nranks + 1, 0), rcnt;
        for (int q = 0; q < nranks; ++q) {
            const auto a = std::lower_bound(mine.begin(), mine.end(), sp->start[q]);
            const auto b = std::lower_bound(mine.begin(), mine.end(), sp->start[q + 1]);
            soff[q] = a - mine.begin();
            scnt[q] = b - a;
        }
        tr->alltoall_counts(scnt, rcnt, s);
        std::vector<int64_t> roff(nranks + 1, 0);
        for (int q = 0; q < nranks; ++q) roff[q + 1] = roff[q] + rcnt[q];
        TBuf<int64_t> sd((int64_t)mine.size() > 0 ? (int64_t)mine.size() : 1, s), rd(roff[nranks] > 0 ? roff[nranks] : 1, s);
        if (!mine.empty())
            PMGR_CUDA(cudaMemcpyAsync(sd.p, mine.data(), sizeof(int64_t) * mine.size(), cudaMemcpyHostToDevice, s));
        std::vector<const void *> sp_(nranks);
        std::vector<void *> rp(nranks);
        std::vector<int64_t> sb(nranks), rb(nranks);
        for (int q = 0; q < nranks; ++q) {
            const bool self = q == rank;
            sp_[q] = sd.p + soff[q];
            sb[q] = self ? 0 : 8 * scnt[q];
            rp[q] = rd.p + roff[q];
            rb[q] = self ? 0 : 8 * rcnt[q];
        }
        tr->alltoallv(sp_, sb, rp, rb, s);
        std::vector<int64_t> all(roff[nranks]);
        if (!all.empty())
            PMGR_CUDA(cudaMemcpyAsync(all.data(), rd.p, sizeof(int64_t) * all.size(), cudaMemcpyDeviceToHost, s));
        PMGR_CUDA(cudaStreamSynchronize(s));
        for (int q = 0; q < nranks; ++q)
            if (q != rank) sp->ghosts[q].assign(all.begin() + roff[q], all.begin() + roff[q + 1]);
    }

    // ghost sets of every rank, my halo plan
    void finalize(Space *sp) {
        sp->ghosts.assign(nranks, {});
        for (int q = 0; q < nranks; ++q) {
            if (partial && q != rank) continue;
            std::vector<int64_t> all;
            for (const Reader &rd : readers[sp->id]) {
                const int64_t r0 = rd.rows->start[q], r1 = rd.rows->start[q + 1];
                if (r1 <= r0) continue;
                int64_t e0, e1;
                PMGR_CUDA(cudaMemcpyAsync(&e0, rd.Y->ro.p + r0, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
                PMGR_CUDA(cudaMemcpyAsync(&e1, rd.Y->ro.p + r1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
                PMGR_CUDA(cudaStreamSynchronize(s));
                if (e1 <= e0) continue;
                TBuf<int64_t> buf(e1 - e0, s), cnt(1, s);
                PMGR_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int64_t), s));
                k_mark_outside<<<grid_for(r1 - r0, 128), 128, 0, s>>>(r1 - r0, rd.Y->ro.p, r0, rd.Y->ci.p,
                                                                      sp->start[q], sp->start[q + 1], buf.p, cnt.p);
                PMGR_LAUNCHED();
                const int64_t c = read_scalar(cnt.p, s);
                if (c == 0) continue;
                thrust::device_ptr<int64_t> b(buf.p);
                thrust::sort(thrust::cuda::par.on(s), b, b + c);
                const int64_t u = thrust::unique(thrust::cuda::par.on(s), b, b + c) - b;
                const size_t old = all.size();
                all.resize(old + u);
                PMGR_CUDA(cudaMemcpyAsync(all.data() + old, buf.p, sizeof(int64_t) * u, cudaMemcpyDeviceToHost, s));
                PMGR_CUDA(cudaStreamSynchronize(s));
            }
            if (sp->triples) {
                const size_t m = all.size();
                for (size_t i = 0; i < m; ++i)
                    for (int c = 0; c < 3; ++c) all.push_back(3 * (all[i] / 3) + c);
            }
            std::sort(all.begin(), all.end());
            all.erase(std::unique(all.begin(), all.end()), all.end());
            // closure may pull in owned entries: drop them
            all.erase(std::remove_if(all.begin(), all.end(),
                                     [&](int64_t g) { return g >= sp->start[q] && g < sp->start[q + 1]; }),
                      all.end());
            sp->ghosts[q] = std::move(all);
        }
        if (partial) exchange_ghosts(sp);
        sp->lo = sp->start[rank];
        sp->hi = sp->start[rank + 1];
        sp->ghosts_me = &sp->ghosts[rank];
        const auto &gm = sp->ghosts[rank];
        sp->nlow = std::lower_bound(gm.begin(), gm.end(), sp->lo) - gm.begin();
        // owned range 768-byte aligned (16-byte vector loads; node triples stay aligned)
        sp->pad = (96 - sp->nlow % 96) % 96;
        sp->gdev.alloc((int64_t)gm.size());
        if (!gm.empty())
            PMGR_CUDA(cudaMemcpyAsync(sp->gdev.p, gm.data(), sizeof(int64_t) * gm.size(), cudaMemcpyHostToDevice, s));
        // halo plan
        auto h = std::make_shared<Halo>();
        h->tr = tr;
        h->id = sp->id;
        h->n_own = sp->n_own();
        h->off = sp->off();
        h->n_ext = sp->n_ext();
        for (int p = 0; p < nranks; ++p) {
            if (p == rank) continue;
            const int64_t a = std::lower_bound(gm.begin(), gm.end(), sp->start[p]) - gm.begin();
            const int64_t b = std::lower_bound(gm.begin(), gm.end(), sp->start[p + 1]) - gm.begin();
            if (b > a) {
                h->rpeer.push_back(p);
                h->roff.push_back(a < sp->nlow ? a : a + sp->pad + sp->n_own());
                h->rcnt.push_back(b - a);
            }
        }
        std::vector<int64_t> sidx;
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            const auto &gq = sp->ghosts[q];
            const int64_t a = std::lower_bound(gq.begin(), gq.end(), sp->lo) - gq.begin();
            const int64_t b = std::lower_bound(gq.begin(), gq.end(), sp->hi) - gq.begin();
            if (b > a) {
                h->speer.push_back(q);
                h->soff.push_back((int64_t)sidx.size());
                h->scnt.push_back(b - a);
                for (int64_t t = a; t < b; ++t) sidx.push_back(gq[t] - sp->lo);
            }
        }
        h->send_idx.alloc((int64_t)sidx.size());
        h->sbuf.alloc((int64_t)sidx.size());
        if (!sidx.empty())
            PMGR_CUDA(cudaMemcpyAsync(h->send_idx.p, sidx.data(), sizeof(int64_t) * sidx.size(),
                                      cudaMemcpyHostToDevice, s));
        PMGR_CUDA(cudaStreamSynchronize(s));
        sp->halo = h;
    }

    // my rows of Y (rows space R) with columns at their ext positions in C
    void localize(const Csr &Y, const Space *R, const Space *C, Csr &out) {
        const int64_t r0 = R->lo, n = R->n_own();
        int64_t e0 = 0, e1 = 0;
        PMGR_CUDA(cudaMemcpyAsync(&e0, Y.ro.p + r0, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        PMGR_CUDA(cudaMemcpyAsync(&e1, Y.ro.p + r0 + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        PMGR_CUDA(cudaStreamSynchronize(s));
        out.nrows = n;
        out.ncols = C->n_ext();
        out.nnz = e1 - e0;
        out.ro.alloc(n + 1);
        out.ci.alloc(out.nnz);
        out.v.alloc(out.nnz);
        k_localize<<<grid_for(n + 1, 128), 128, 0, s>>>(n, Y.ro.p, r0, Y.ci.p, Y.v.p, C->lo, C->hi, C->nlow, C->pad,
                                                        C->gdev.p, (int64_t)C->ghosts_me->size(), out.ro.p,
                                                        out.ci.p, out.v.p);
        PMGR_LAUNCHED();
        csr_finalize(out, s, false);
        out.sj_want = Y.sj_want;
        out.g_rows = Y.g_rows > 0 ? Y.g_rows : Y.nrows;
        out.g_nnz = Y.g_nnz > 0 ? Y.g_nnz : Y.nnz;
        out.row_off = R->off();
        out.lanes = Y.lanes > 0 ? Y.lanes : spmv_lanes(Y.view());
        out.lanes_u = Y.lanes_u > 0 ? Y.lanes_u : spmv_u_for(Y.nnz, Y.nrows, out.lanes);
        // the same rows take the block-per-row path as in the global operator
        out.long_len = Y.long_len;
        csr_long_rows(out, s);
        // a pure block operator keeps its blocks (same blocks, same order as the
        // global copy); a block-prefix operator (A0 on the original layout)
        // is sliced as CSR
        if (Y.nbrows > 0 && Y.nbrows * 3 == Y.nrows && !Y.rro.p) {
            csr_make_bsr3(out, out.nrows, out.ncols, s, true);
            if (out.nbrows * 3 != out.nrows) fail(PMGR_ERR_INVALID, "local block copy failed");
        } else {
            csr_make_sj(out, s);
        }
        if (nranks > 1) classify_overlap(out, C->off(), C->off() + C->n_own(), s);
    }

    // owned values of a global per-entry array into an ext-length buffer
    void own_values(const double *glob, const Space *sp, DBuf<double> &ext) {
        ext.alloc(sp->n_ext());
        PMGR_CUDA(cudaMemsetAsync(ext.p, 0, sizeof(double) * (size_t)(ext.n > 0 ? ext.n : 1), s));
        if (sp->n_own() > 0)
            PMGR_CUDA(cudaMemcpyAsync(ext.p + sp->off(), glob + sp->lo, sizeof(double) * sp->n_own(),
                                      cudaMemcpyDeviceToDevice, s));
    }
    void ext_buffer(const Space *sp, DBuf<double> &ext) {
        ext.alloc(sp->n_ext());
        PMGR_CUDA(cudaMemsetAsync(ext.p, 0, sizeof(double) * (size_t)(ext.n > 0 ? ext.n : 1), s));
    }
    // index map over the owned entries of `over`: global ids in space `to`
    // (owned by this rank as well) -> ext positions of `to`
    void own_map(const int64_t *glob, const Space *over, const Space *to, DBuf<int64_t> &ext, bool keep_negative) {
        ext.alloc(over->n_ext());
        PMGR_CUDA(cudaMemsetAsync(ext.p, 0xff, sizeof(int64_t) * (size_t)(ext.n > 0 ? ext.n : 1), s));
        if (over->n_own() > 0) {
            k_map_owned<<<grid_for(over->n_own(), 256), 256, 0, s>>>(over->n_own(), glob, over->lo, to->lo, to->off(),
                                                                      ext.p, over->off(), keep_negative ? 1 : 0);
            PMGR_LAUNCHED();
        }
    }
};

namespace {

// AMG hierarchy over space S0: register spaces and readers (phase 1)
struct AmgPlan {
    const pmgr_amg *G;
    std::vector<Space *> sp;  // per level (up to collapse_from inclusive)
};

void plan_amg(Builder &B, const pmgr_amg &G, Space *S0, AmgPlan &P) {
    P.G = &G;
    if (G.levels.empty() || G.collapse_from < 0)
        fail(PMGR_ERR_NOT_SUPPORTED,
             "row distribution needs the collapsed coarse cycle (PMGR_COLLAPSE_ROWS > 0, at least one AMG level)");
    for (const AmgLevel &L : G.levels)
        if (!L.jacobi) fail(PMGR_ERR_NOT_SUPPORTED, "row distribution needs l1-Jacobi AMG levels (npartitions >= n)");
    P.sp.push_back(S0);
    for (int l = 0; l < G.collapse_from; ++l) P.sp.push_back(B.derive(P.sp[l], G.levels[l].is_c.p, true));
    for (int l = 0; l < G.collapse_from; ++l) {
        const AmgLevel &L = G.levels[l];
        B.read(P.sp[l], L.A.get(), P.sp[l]);
        B.read(P.sp[l], &L.R, P.sp[l + 1]);
        B.read(P.sp[l + 1], &L.P, P.sp[l]);
    }
    // a wholly collapsed hierarchy still applies its operator once per cycle
    // from a nonzero guess (multi-cycle F-relaxation: x + M_t (b - A x))
    if (G.collapse_from == 0) B.read(P.sp[0], G.levels[0].A.get(), P.sp[0]);
    if (G.levels[0].A->nbrows > 0) S0->triples = true;
}

std::unique_ptr<pmgr_amg> build_amg(Builder &B, const AmgPlan &P) {
    const pmgr_amg &G = *P.G;
    auto h = std::make_unique<pmgr_amg>();
    h->cfg = G.cfg;
    h->collapse_from = G.collapse_from;
    h->levels.resize(G.collapse_from + 1);
    for (int l = 0; l <= G.collapse_from; ++l) {
        const AmgLevel &GL = G.levels[l];
        AmgLevel &L = h->levels[l];
        Space *S = P.sp[l];
        L.jacobi = true;
        L.off = S->off();
        L.halo = S->halo;
        auto A = std::make_shared<Csr>();
        if (l < G.collapse_from) {
            B.localize(*GL.A, S, S, *A);
            B.localize(GL.P, S, P.sp[l + 1], L.P);
            B.localize(GL.R, P.sp[l + 1], S, L.R);
        } else if (l == 0) {
            B.localize(*GL.A, S, S, *A);
        } else {
            A->nrows = S->n_own();  // the collapsed level only needs its row count
            A->ncols = S->n_ext();
        }
        L.A = A;
        B.own_values(GL.dtilde.p, S, L.dtilde);
        B.ext_buffer(S, L.b);
        B.ext_buffer(S, L.x);
        B.ext_buffer(S, L.r);
        B.ext_buffer(S, L.xo);
    }
    // collapsed operator: my rows, full width
    Space *Sc = P.sp[G.collapse_from];
    h->collapsed_ld = G.collapsed_ld;
    h->collapsed.alloc(Sc->n_own() * G.collapsed_ld);
    if (Sc->n_own() > 0)
        PMGR_CUDA(cudaMemcpyAsync(h->collapsed.p, G.collapsed.p + Sc->lo * G.collapsed_ld,
                                  sizeof(double) * Sc->n_own() * G.collapsed_ld, cudaMemcpyDeviceToDevice, B.s));
    h->gather = std::make_shared<Gather>();
    h->gather->tr = B.tr;
    h->gather->n_full = Sc->n;
    h->gather->start = Sc->start;
    h->gather->id = Sc->id;
    h->full.alloc(Sc->n > 0 ? Sc->n : 1);
    return h;
}

}  // namespace

namespace {
std::unique_ptr<DistSolver> dist_build_impl(const pmgr_csr *A, pmgr_mgr *M, const int64_t *bounds, int rank,
                                            int nranks, Transport *tr, cudaStream_t s, bool partial);
}

std::unique_ptr<DistSolver> dist_build(const pmgr_csr *A, pmgr_mgr *M, const int64_t *bounds, int rank, int nranks,
                                       Transport *tr, cudaStream_t s) {
    return dist_build_impl(A, M, bounds, rank, nranks, tr, s, false);
}

std::unique_ptr<DistSolver> dist_setup(const pmgr_csr *A, const int8_t *field_of, const int32_t *entity_of,
                                       const pmgr_level_spec *levels, int nlevels, const pmgr_mgr_cfg &cfg,
                                       const int64_t *bounds, int rank, int nranks, Transport *tr, cudaStream_t s) {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(PMGR_ERR_INVALID, "bad rank / nranks");
    if (nranks > 1 && (!tr || tr->rank != rank || tr->nranks != nranks))
        fail(PMGR_ERR_INVALID, "transport rank mismatch");
    DistSetup d;
    d.tr = tr;
    d.rank = rank;
    d.nranks = nranks;
    d.start.assign(bounds, bounds + nranks + 1);
    // small levels are set up redundantly on every rank; the collapsed coarse
    // cycle needs its levels whole
    const char *e = getenv("PMGR_DIST_REPLICATE_ROWS");
    d.replicate_below = std::max(e ? (int64_t)atoll(e) : (int64_t)20000, collapse_limit());
    if (nranks > 1) ds_finalize(&d, *A->m, s);  // the global operator's lane group
    std::unique_ptr<pmgr_mgr> M = mgr_build(A->m, field_of, entity_of, levels, nlevels, cfg, s, &d);
    return dist_build_impl(A, M.get(), bounds, rank, nranks, tr, s, nranks > 1);
}

namespace {
std::unique_ptr<DistSolver> dist_build_impl(const pmgr_csr *A, pmgr_mgr *M, const int64_t *bounds, int rank,
                                            int nranks, Transport *tr, cudaStream_t s, bool partial) {
    if (!M || M->dist) fail(PMGR_ERR_INVALID, "row distribution needs a global hierarchy");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(PMGR_ERR_INVALID, "bad rank / nranks");
    if (tr && (tr->rank != rank || tr->nranks != nranks)) fail(PMGR_ERR_INVALID, "transport rank mismatch");
    const Csr &A0 = *A->m;
    if (A0.nrows != M->n) fail(PMGR_ERR_INVALID, "matrix and hierarchy sizes differ");
    if (M->f_relax_post || M->terminal_cycles != 1)
        fail(PMGR_ERR_NOT_SUPPORTED, "row distribution supports pre F-relaxation and one terminal cycle");
    for (const MgrLevel &L : M->levels) {
        if (L.smoother && partial)
            fail(PMGR_ERR_NOT_SUPPORTED, "distributed setup of a level with a global smoother");
        if (L.f_relax == PMGR_FRELAX_NONE || (L.f_relax_sweeps != 1 && L.f_relax != PMGR_FRELAX_AMG))
            fail(PMGR_ERR_NOT_SUPPORTED,
                 "row distribution supports AMG F-relaxation (any number of cycles) or single-sweep Jacobi");
    }
    if (!M->terminal) fail(PMGR_ERR_NOT_SUPPORTED, "row distribution needs a terminal AMG");
    Builder B(rank, nranks, tr, s);
    B.partial = partial;
    // ---- phase 1: spaces and who reads them
    Space *M0 = B.root(A0.nrows, bounds);
    B.read(M0, &A0, M0);
    const size_t nl = M->levels.size();
    std::vector<Space *> Ms{M0}, Fs;
    std::vector<AmgPlan> fplans(nl);
    for (size_t l = 0; l < nl; ++l) {
        const MgrLevel &L = M->levels[l];
        Space *F = B.derive(Ms[l], L.is_c.p, false);
        Space *C = B.derive(Ms[l], L.is_c.p, true);
        Fs.push_back(F);
        Ms.push_back(C);
        B.read(F, &L.A_cf, C);
        B.read(C, &L.P, Ms[l]);
        if (L.smoother) {  // the smoothed iterate is read by the level operator and its C rows
            B.read(Ms[l], L.A.get(), Ms[l]);
            B.read(Ms[l], &L.A_c, C);
        }
        if (L.f_relax == PMGR_FRELAX_AMG) plan_amg(B, *L.amg, F, fplans[l]);
    }
    AmgPlan tplan;
    plan_amg(B, *M->terminal, Ms[nl], tplan);
    for (auto &sp : B.spaces) B.finalize(sp.get());
    // ---- phase 2: local operators and workspaces
    auto D = std::make_unique<DistSolver>();
    D->rank = rank;
    D->nranks = nranks;
    D->tr = tr;
    D->n_global = A0.nrows;
    D->lo = M0->lo;
    D->n_own = M0->n_own();
    D->off = M0->off();
    D->n_ext = M0->n_ext();
    D->halo0 = M0->halo;
    B.localize(A0, M0, M0, D->A);
    auto h = std::make_unique<pmgr_mgr>();
    h->dist = true;
    h->use_graphs = false;
    h->terminal_cycles = 1;
    h->f_relax_post = 0;
    h->n = M0->n_own();
    h->levels.resize(nl);
    for (size_t l = 0; l < nl; ++l) {
        const MgrLevel &G = M->levels[l];
        MgrLevel &L = h->levels[l];
        Space *Mi = Ms[l], *F = Fs[l], *C = Ms[l + 1];
        L.n = Mi->n_own();
        L.nf = F->n_own();
        L.nc = C->n_own();
        L.off = Mi->off();
        L.off_f = F->off();
        L.off_c = C->off();
        L.halo_f = F->halo;
        L.halo_c = C->halo;
        L.f_relax = G.f_relax;
        L.f_relax_sweeps = G.f_relax_sweeps;
        B.localize(G.A_cf, C, F, L.A_cf);
        B.localize(G.P, Mi, C, L.P);
        B.own_map(G.f_rows.p, F, Mi, L.f_rows, false);
        B.own_map(G.c_rows.p, C, Mi, L.c_rows, false);
        B.own_map(G.f_index.p, Mi, F, L.f_index, true);
        if (G.dinv_ff.p) B.own_values(G.dinv_ff.p, F, L.dinv_ff);
        B.ext_buffer(F, L.zf);
        if (L.f_relax_sweeps > 1) {  // multi-cycle F-relaxation: gathered rhs and the previous iterate
            B.ext_buffer(F, L.vf);
            B.ext_buffer(F, L.tmpf);
        }
        B.ext_buffer(C, L.rc);
        B.ext_buffer(C, L.zc);
        if (G.f_relax == PMGR_FRELAX_AMG) L.amg = build_amg(B, fplans[l]);
        if (G.smoother) {
            // ILU partitions live whole on their ranks: the rank's factors are
            // rows of the global ones, the level operator and its C rows are
            // localised like every other operator
            L.smoother = smoother_slice(*G.smoother, Mi->lo, Mi->hi, s);
            L.halo_m = Mi->halo;
            auto Al = std::make_shared<Csr>();
            B.localize(*G.A, Mi, Mi, *Al);
            L.A = Al;
            B.localize(G.A_c, C, Mi, L.A_c);
            B.ext_buffer(Mi, L.zs);
            B.ext_buffer(Mi, L.rr);
        }
    }
    h->terminal = build_amg(B, tplan);
    PMGR_CUDA(cudaStreamSynchronize(s));
    D->M = std::move(h);
    D->spaces.reserve(B.spaces.size());
    for (auto &sp : B.spaces) D->halos.push_back(sp->halo);
    return D;
}
}  // namespace

// ========================================================= apply, GMRES

void dist_apply(DistSolver &D, const double *v_own, double *z_own, cudaStream_t s) {
    D.ensure_work();
    if (D.n_own > 0)
        PMGR_CUDA(cudaMemcpyAsync(D.ve.p + D.off, v_own, sizeof(double) * D.n_own, cudaMemcpyDeviceToDevice, s));
    mgr_apply_direct(*D.M, D.ve.p, D.ze.p, s);
    if (D.n_own > 0)
        PMGR_CUDA(cudaMemcpyAsync(z_own, D.ze.p + D.off, sizeof(double) * D.n_own, cudaMemcpyDeviceToDevice, s));
}

void DistSolver::ensure_work() {
    if (ve.p) return;
    ve.alloc(n_ext > 0 ? n_ext : 1);
    ze.alloc(n_ext > 0 ? n_ext : 1);
    we.alloc(n_ext > 0 ? n_ext : 1);
    PMGR_CUDA(cudaMemset(ve.p, 0, sizeof(double) * ve.n));
    PMGR_CUDA(cudaMemset(ze.p, 0, sizeof(double) * ze.n));
    PMGR_CUDA(cudaMemset(we.p, 0, sizeof(double) * we.n));
}


// y = A x for an owned x (halo exchange into the ext buffer first)
static void dist_spmv(DistSolver &D, const double *x_own, double *y_own, cudaStream_t s) {
    D.ensure_work();
    if (D.n_own > 0)
        PMGR_CUDA(cudaMemcpyAsync(D.ze.p + D.off, x_own, sizeof(double) * D.n_own, cudaMemcpyDeviceToDevice, s));
    with_halo(D.A, D.halo0.get(), D.ze.p, s, [&](const CsrView &V) { spmv(V, D.ze.p, D.we.p, s); });
    if (D.n_own > 0)
        PMGR_CUDA(cudaMemcpyAsync(y_own, D.we.p + D.off, sizeof(double) * D.n_own, cudaMemcpyDeviceToDevice, s));
}

// Right-preconditioned restarted GMRES (krylov.py:39-117) on row-distributed
// vectors: the single-GPU Arnoldi kernels in split mode (krylov.cu), with the
// projections (2(m+1) doubles) and the squared norm all-reduced across ranks;
// the Hessenberg / Givens state is replicated (identical all-reduced inputs,
// identical control flow on every rank).  With NCCL one step is a captured
// CUDA graph (apply with its halo exchanges, SpMV, Arnoldi, all-reduces).
void dist_gmres(DistSolver &D, const double *b, double *x, int nonzero_x0, const pmgr_gmres_cfg &cfg,
                pmgr_gmres_stats &st, double *history, int32_t history_cap, cudaStream_t s) {
    D.ensure_work();
    SplitOps ops;
    ops.cache = &D.gws;
    ops.n = D.n_own;
    ops.vin = D.ve.p + D.off;
    ops.w = D.we.p + D.off;
    ops.capturable = D.tr && D.tr->capturable();
    ops.step = [&](cudaStream_t q) {
        mgr_apply_direct(*D.M, D.ve.p, D.ze.p, q);
        with_halo(D.A, D.halo0.get(), D.ze.p, q, [&](const CsrView &V) { spmv(V, D.ze.p, D.we.p, q); });
    };
    ops.spmv = [&](const double *xo, double *yo, cudaStream_t q) { dist_spmv(D, xo, yo, q); };
    ops.apply = [&](const double *uo, double *zo, cudaStream_t q) { dist_apply(D, uo, zo, q); };
    ops.allreduce = [&](double *buf, int64_t cnt, cudaStream_t q) {
        if (D.tr) D.tr->allreduce(buf, cnt, q);
    };
    gmres_split(ops, b, x, nonzero_x0, cfg, st, history, history_cap, s);
}

// ====================================================== one-GPU emulation

void dist_setup_emulate(const pmgr_csr *A, const int8_t *field_of, const int32_t *entity_of,
                        const pmgr_level_spec *levels, int nlevels, const pmgr_mgr_cfg &mcfg, const int64_t *bounds,
                        int nranks, int what, const double *in, double *out, const pmgr_gmres_cfg *cfg,
                        pmgr_gmres_stats *stats, cudaStream_t s) {
    LoopbackHub hub(nranks);
    std::vector<std::unique_ptr<LoopbackTransport>> trs;
    std::vector<pmgr_csr> parts(nranks);
    for (int r = 0; r < nranks; ++r) {
        trs.emplace_back(new LoopbackTransport(&hub, r));
        parts[r].m = std::make_shared<Csr>();
        ds_partial_rows(*A->m, bounds[r], bounds[r + 1], *parts[r].m, s);
    }
    PMGR_CUDA(cudaStreamSynchronize(s));
    int dev = 0;
    PMGR_CUDA(cudaGetDevice(&dev));
    std::vector<std::string> errs(nranks);
    std::vector<pmgr_gmres_stats> st(nranks);
    std::vector<std::thread> th;
    for (int r = 0; r < nranks; ++r) {
        th.emplace_back([&, r] {
            try {
                PMGR_CUDA(cudaSetDevice(dev));
                auto D = dist_setup(&parts[r], field_of, entity_of, levels, nlevels, mcfg, bounds, r, nranks,
                                    trs[r].get(), s);
                if (what == 0) {
                    dist_apply(*D, in + D->lo, out + D->lo, s);
                } else {
                    pmgr_gmres_stats z = {};
                    dist_gmres(*D, in + D->lo, out + D->lo, 0, *cfg, z, nullptr, 0, s);
                    st[r] = z;
                }
                PMGR_CUDA(cudaStreamSynchronize(s));
            } catch (const Error &e) {
                errs[r] = e.msg.empty() ? "error" : e.msg;
                hub.abort(errs[r]);
            } catch (const std::exception &e) {
                errs[r] = e.what();
                hub.abort(e.what());
            }
        });
    }
    for (auto &t : th) t.join();
    PMGR_CUDA(cudaStreamSynchronize(s));
    for (int r = 0; r < nranks; ++r)
        if (!errs[r].empty() && errs[r].find("loopback peer failed") == std::string::npos &&
            errs[r].find("loopback exchange failed") == std::string::npos)
            fail(PMGR_ERR_CUDA, "rank " + std::to_string(r) + ": " + errs[r]);
    for (int r = 0; r < nranks; ++r)
        if (!errs[r].empty()) fail(PMGR_ERR_CUDA, "rank " + std::to_string(r) + ": " + errs[r]);
    if (stats && what == 1) {
        *stats = st[0];
        for (int r = 1; r < nranks; ++r)
            if (st[r].iterations != st[0].iterations)
                fail(PMGR_ERR_INVALID, "emulated ranks disagree on the iteration count");
    }
}

void dist_emulate(const pmgr_csr *A, pmgr_mgr *M, const int64_t *bounds, int nranks, int what, const double *in,
                  double *out, const pmgr_gmres_cfg *cfg, pmgr_gmres_stats *stats, cudaStream_t s) {
    LoopbackHub hub(nranks);
    std::vector<std::unique_ptr<LoopbackTransport>> trs;
    std::vector<std::unique_ptr<DistSolver>> ds;
    for (int r = 0; r < nranks; ++r) {
        trs.emplace_back(new LoopbackTransport(&hub, r));
        ds.push_back(dist_build(A, M, bounds, r, nranks, trs.back().get(), s));
    }
    int dev = 0;
    PMGR_CUDA(cudaGetDevice(&dev));
    std::vector<std::string> errs(nranks);
    std::vector<pmgr_gmres_stats> st(nranks);
    std::vector<std::thread> th;
    for (int r = 0; r < nranks; ++r) {
        th.emplace_back([&, r] {
            try {
                PMGR_CUDA(cudaSetDevice(dev));
                DistSolver &D = *ds[r];
                if (what == 0) {
                    dist_apply(D, in + D.lo, out + D.lo, s);
                } else {
                    pmgr_gmres_stats z = {};
                    dist_gmres(D, in + D.lo, out + D.lo, 0, *cfg, z, nullptr, 0, s);
                    st[r] = z;
                }
            } catch (const Error &e) {
                errs[r] = e.msg.empty() ? "error" : e.msg;
                hub.abort(errs[r]);
            } catch (const std::exception &e) {
                errs[r] = e.what();
                hub.abort(e.what());
            }
        });
    }
    for (auto &t : th) t.join();
    PMGR_CUDA(cudaStreamSynchronize(s));
    for (int r = 0; r < nranks; ++r)
        if (!errs[r].empty()) fail(PMGR_ERR_CUDA, "rank " + std::to_string(r) + ": " + errs[r]);
    if (stats && what == 1) {
        *stats = st[0];
        for (int r = 1; r < nranks; ++r)
            if (st[r].iterations != st[0].iterations)
                fail(PMGR_ERR_INVALID, "emulated ranks disagree on the iteration count");
    }
}

}  // namespace pmgr
