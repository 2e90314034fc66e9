// prims.cu -- scans, segmented sorts and reductions (CUB device primitives).
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <map>
#include <mutex>

#include "common.cuh"

namespace pmgr {

std::atomic<int64_t> g_launches{0};
thread_local int64_t *g_capture_count = nullptr;
thread_local double *g_byte_ledger = nullptr;

namespace {
bool g_prof = false;
std::vector<ProfRec> g_recs;  // event pool for direct (non-graph) launches
size_t g_used = 0;
std::vector<std::pair<std::vector<ProfRec> *, size_t>> g_open[PROF_KINDS];
std::vector<ProfRec> *g_capture = nullptr;  // records of the graph being captured
int64_t g_count[PROF_KINDS];
double g_ms[PROF_KINDS], g_bytes[PROF_KINDS];

void accumulate(const ProfRec &r) {
    PMGR_CUDA(cudaEventSynchronize(r.b));
    float e = 0.f;
    PMGR_CUDA(cudaEventElapsedTime(&e, r.a, r.b));
    g_count[r.kind] += 1;
    g_ms[r.kind] += e;
    g_bytes[r.kind] += r.bytes;
}

void flush_direct() {
    for (size_t i = 0; i < g_used; ++i) accumulate(g_recs[i]);
    g_used = 0;
}
}  // namespace

bool prof_on() { return g_prof; }

void prof_capture_begin(std::vector<ProfRec> *recs) { g_capture = recs; }
void prof_capture_end() { g_capture = nullptr; }

void prof_begin(int kind, double bytes, cudaStream_t s) {
    ProfRec r{};
    r.kind = kind;
    r.bytes = bytes;
    if (g_capture) {
        // inside stream capture: the events become graph nodes
        PMGR_CUDA(cudaEventCreate(&r.a));
        PMGR_CUDA(cudaEventCreate(&r.b));
        PMGR_CUDA(cudaEventRecordWithFlags(r.a, s, cudaEventRecordExternal));
        g_capture->push_back(r);
        g_open[kind].push_back({g_capture, g_capture->size() - 1});
        return;
    }
    if (g_used == g_recs.size()) {  // the pool only grows; scopes may still be open
        PMGR_CUDA(cudaEventCreate(&r.a));
        PMGR_CUDA(cudaEventCreate(&r.b));
        g_recs.push_back(r);
    }
    ProfRec &q = g_recs[g_used];
    q.kind = kind;
    q.bytes = bytes;
    PMGR_CUDA(cudaEventRecord(q.a, s));
    g_open[kind].push_back({&g_recs, g_used});
    ++g_used;
}

void prof_end(int kind, cudaStream_t s) {
    auto top = g_open[kind].back();
    g_open[kind].pop_back();
    ProfRec &r = (*top.first)[top.second];
    if (top.first != &g_recs)
        PMGR_CUDA(cudaEventRecordWithFlags(r.b, s, cudaEventRecordExternal));
    else
        PMGR_CUDA(cudaEventRecord(r.b, s));
}

void prof_collect(std::vector<ProfRec> &graph_recs) {
    for (const ProfRec &r : graph_recs) accumulate(r);
}

void prof_release(std::vector<ProfRec> &graph_recs) {
    for (ProfRec &r : graph_recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    graph_recs.clear();
}

void prof_enable(bool on) {
    if (g_prof) flush_direct();
    g_prof = on;
    g_used = 0;
    for (auto &v : g_open) v.clear();
    for (int k = 0; k < PROF_KINDS; ++k) {
        g_count[k] = 0;
        g_ms[k] = g_bytes[k] = 0.0;
    }
}

void prof_query(int kind, int64_t *count, double *ms, double *bytes) {
    flush_direct();
    *count = g_count[kind];
    *ms = g_ms[kind];
    *bytes = g_bytes[kind];
}

void setup_trace(const char *what, int64_t level, cudaStream_t s) {
    static const bool on = [] {
        const char *e = getenv("PMGR_SETUP_TRACE");
        return e && e[0] != '0';
    }();
    if (!on) return;
    static std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[pmgr setup] %-28s level %3lld  %9.3f ms\n", what, (long long)level,
            std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

namespace {
double g_ht_sec[4] = {0, 0, 0, 0}, g_ht_bytes[4] = {0, 0, 0, 0};
int64_t g_ht_cnt[4] = {0, 0, 0, 0};
double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

bool host_trace_on() {
    static const bool on = [] {
        const char *e = getenv("PMGR_SETUP_TRACE");
        return e && e[0] != '0';
    }();
    return on;
}
void host_trace_add(int kind, double seconds, double bytes) {
    g_ht_sec[kind] += seconds;
    g_ht_bytes[kind] += bytes;
    ++g_ht_cnt[kind];
}
void host_trace_report(const char *what) {
    if (!host_trace_on()) return;
    static const char *names[4] = {"cudaMalloc", "cudaFree", "cudaMallocAsync", "blocking scalar reads"};
    for (int k = 0; k < 4; ++k) {
        fprintf(stderr, "[pmgr host] %-12s %-22s %6lld calls %9.3f ms %9.2f GB\n", what, names[k],
                (long long)g_ht_cnt[k], 1e3 * g_ht_sec[k], g_ht_bytes[k] / 1e9);
        g_ht_sec[k] = g_ht_bytes[k] = 0;
        g_ht_cnt[k] = 0;
    }
}
HostTimer::HostTimer(int k, double b) : kind(k), bytes(b), on(host_trace_on()), t0(on ? now_s() : 0.0) {}
HostTimer::~HostTimer() {
    if (on) host_trace_add(kind, now_s() - t0, bytes);
}

namespace {
// Block cache behind the persistent buffers (DBuf): a freed block is kept
// (per device, keyed by size) and handed to the next request of about that
// size, so a repeated setup -- the second build of a benchmark, every Newton
// step of a simulation -- finds its ~900 operator arrays without a single
// cudaMalloc.  Blocks are cached only after a device synchronisation, so no
// stream can still be using one when it is handed out again.
struct BlockCache {
    std::mutex mu;
    std::multimap<std::pair<int, size_t>, void *> free_blocks;
    std::map<void *, std::pair<int, size_t>> live;  // handed out: device, block size
    size_t cached = 0;
    size_t cap() {
        static const size_t c = [] {
            if (const char *e = getenv("PMGR_DBUF_CACHE_GB")) return (size_t)(atof(e) * 1e9);
            size_t fr = 0, tot = 0;
            if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) tot = (size_t)64 << 30;
            return (size_t)(0.45 * (double)tot);
        }();
        return c;
    }
    // return every cached block to the driver (out of memory, or on request)
    void trim() {
        std::lock_guard<std::mutex> lock(mu);
        for (auto &kv : free_blocks) cudaFree(kv.second);
        free_blocks.clear();
        cached = 0;
    }
};
BlockCache &block_cache() {
    static BlockCache *c = new BlockCache;  // never destroyed: buffers may outlive static teardown
    return *c;
}
}  // namespace

void dbuf_trim() { block_cache().trim(); }

void *dbuf_alloc(size_t bytes) {
    HostTimer ht(0, (double)bytes);
    BlockCache &C = block_cache();
    const size_t want = (bytes + 511) & ~(size_t)511;
    int dev = 0;
    PMGR_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lock(C.mu);
        auto it = C.free_blocks.lower_bound({dev, want});
        if (it != C.free_blocks.end() && it->first.first == dev &&
            it->first.second <= want + want / 8 + (64 << 10)) {
            void *p = it->second;
            C.live[p] = it->first;
            C.cached -= it->first.second;
            C.free_blocks.erase(it);
            return p;
        }
    }
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        C.trim();
        e = cudaMalloc(&p, want);
    }
    if (e != cudaSuccess) fail_cuda(e, "cudaMalloc", __FILE__, __LINE__);
    std::lock_guard<std::mutex> lock(C.mu);
    C.live[p] = {dev, want};
    return p;
}

void dbuf_free(void *p, size_t bytes) {
    HostTimer ht(1, (double)bytes);
    BlockCache &C = block_cache();
    std::pair<int, size_t> key{-1, 0};
    {
        std::lock_guard<std::mutex> lock(C.mu);
        auto it = C.live.find(p);
        if (it != C.live.end()) {
            key = it->second;
            C.live.erase(it);
        }
    }
    static const bool cache_on = !(getenv("PMGR_DBUF_CACHE") && getenv("PMGR_DBUF_CACHE")[0] == '0');
    if (key.first < 0 || !cache_on || cudaDeviceSynchronize() != cudaSuccess) {
        cudaGetLastError();
        cudaFree(p);  // unknown block, cache off, or the context is shutting down
        return;
    }
    std::lock_guard<std::mutex> lock(C.mu);
    if (C.cached + key.second > C.cap()) {
        cudaFree(p);
        return;
    }
    C.free_blocks.emplace(key, p);
    C.cached += key.second;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("PMGR_NO_PDL");
        return !(e && e[0] != '0');
    }();
    return on;
}

void keep_pool_memory() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    static const bool keep_on = !(getenv("PMGR_POOL_KEEP") && getenv("PMGR_POOL_KEEP")[0] == '0');
    cudaMemPool_t pool;
    if (keep_on && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done_dev = dev;
}

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        PMGR_CUDA(cudaGetDevice(&dev));
        PMGR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return sms;
}

namespace {
__global__ void k_set_zero_i64(int64_t *p) { *p = 0; }

template <class T>
__global__ void k_widen(const T *in, int64_t *out, int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = (int64_t)in[i];
}

// max |x|: non-negative doubles order like their bit patterns
__global__ void k_max_abs(const double *x, int64_t n, unsigned long long *out) {
    double m = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs(x[i]));
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}
}  // namespace

int64_t exclusive_scan_total(const int64_t *in, int64_t *out, int64_t n, cudaStream_t s) {
    // out has n+1 entries: inclusive scan written at out+1, out[0] = 0.
    k_set_zero_i64<<<1, 1, 0, s>>>(out);
    PMGR_LAUNCHED();
    if (n > 0) {
        size_t tmp = 0;
        PMGR_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, in, out + 1, n, s));
        TBuf<char> t((int64_t)tmp, s);
        PMGR_CUDA(cub::DeviceScan::InclusiveSum(t.p, tmp, in, out + 1, n, s));
        g_launches.fetch_add(1, std::memory_order_relaxed);
    }
    return read_scalar(out + n, s);
}

int64_t exclusive_scan_total_i32(const int32_t *in, int64_t *out, int64_t n, cudaStream_t s) {
    TBuf<int64_t> w(n, s);
    if (n > 0) {
        k_widen<<<grid_for(n, 256), 256, 0, s>>>(in, w.p, n);
        PMGR_LAUNCHED();
    }
    return exclusive_scan_total(w.p, out, n, s);
}

void segmented_sort_pairs(int32_t *keys, double *vals, int64_t nnz, const int64_t *ro,
                          int64_t nrows, cudaStream_t s) {
    if (nnz <= 1 || nrows == 0) return;
    TBuf<int32_t> k2(nnz, s);
    TBuf<double> v2(nnz, s);
    size_t tmp = 0;
    PMGR_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, tmp, keys, k2.p, vals, v2.p, nnz,
                                                  nrows, ro, ro + 1, s));
    TBuf<char> t((int64_t)tmp, s);
    PMGR_CUDA(cub::DeviceSegmentedSort::SortPairs(t.p, tmp, keys, k2.p, vals, v2.p, nnz, nrows,
                                                  ro, ro + 1, s));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    PMGR_CUDA(cudaMemcpyAsync(keys, k2.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, s));
    PMGR_CUDA(cudaMemcpyAsync(vals, v2.p, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, s));
}

void segmented_sort_pairs_list(int32_t *keys, double *vals, int64_t nnz, const int64_t *sbeg, const int64_t *send,
                               int64_t nseg, cudaStream_t s) {
    if (nnz <= 1 || nseg == 0) return;
    // the listed segments are sorted into a copy of the whole arrays (the
    // other entries are already in place) and copied back
    TBuf<int32_t> k2(nnz, s);
    TBuf<double> v2(nnz, s);
    PMGR_CUDA(cudaMemcpyAsync(k2.p, keys, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, s));
    PMGR_CUDA(cudaMemcpyAsync(v2.p, vals, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, s));
    size_t tmp = 0;
    PMGR_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, tmp, keys, k2.p, vals, v2.p, nnz, nseg, sbeg, send, s));
    TBuf<char> t((int64_t)tmp, s);
    PMGR_CUDA(cub::DeviceSegmentedSort::SortPairs(t.p, tmp, keys, k2.p, vals, v2.p, nnz, nseg, sbeg, send, s));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    PMGR_CUDA(cudaMemcpyAsync(keys, k2.p, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, s));
    PMGR_CUDA(cudaMemcpyAsync(vals, v2.p, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, s));
}

double device_max_abs(const double *x, int64_t n, cudaStream_t s) {
    if (n == 0) return 0.0;
    TBuf<unsigned long long> out(1, s);
    PMGR_CUDA(cudaMemsetAsync(out.p, 0, sizeof(unsigned long long), s));
    k_max_abs<<<grid_for(n, 256) < 4096 ? grid_for(n, 256) : 4096, 256, 0, s>>>(x, n, out.p);
    PMGR_LAUNCHED();
    unsigned long long bits = read_scalar(out.p, s);
    double r;
    memcpy(&r, &bits, sizeof(r));
    return r;
}

}  // namespace pmgr
