// Host engine: see engine.h. Control flow restates the reference estimator
// (proj/src/{kernel,spectrum,poly,hutchpp,entropy,measures}.cpp); all O(n^2)
// and O(n·s) work runs in the sm_100a kernels, only O(s^2) scalars and the
// per-pass trace partials come back to the host.
#include "engine.h"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>

namespace rb {

// Row pitch (elements) of a stored kernel matrix: a multiple of 64 so every row starts on a
// 128-byte line in the fp16 planes (and on a 512-byte boundary in fp64). With the former
// round_up(n, 8) pitch, n = 100000 put odd rows 64 bytes into a line, so each 128-byte TMA row
// touched two L2 lines (twice the requests, partial-line DRAM traffic).
static inline int64_t matrix_pitch(int64_t n) { return ((n + 63) / 64) * 64; }

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    (void)cudaGetLastError();
    if (e == cudaErrorMemoryAllocation) fail(kOutOfMemory, std::string(what) + ": out of device memory");
    fail(kCudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

void h2d(Context& ctx, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx.stream()), "host->device copy");
    ctx.h2d_bytes += static_cast<long long>(bytes);
}
void d2h(Context& ctx, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx.stream()), "device->host copy");
    ctx.d2h_bytes += static_cast<long long>(bytes);
}
void h2d_2d(Context& ctx, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height) {
    if (width == 0 || height == 0) return;
    cuda_check(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice, ctx.stream()),
               "host->device copy");
    ctx.h2d_bytes += static_cast<long long>(width * height);
}
void d2h_2d(Context& ctx, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height) {
    if (width == 0 || height == 0) return;
    cuda_check(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToHost, ctx.stream()),
               "device->host copy");
    ctx.d2h_bytes += static_cast<long long>(width * height);
}

namespace {
// Host inputs usually sit in pageable memory (numpy arrays, a file read into a string). Large ones go through
// two page-locked 32 MB slots per device: several host threads fill one slot while the DMA engine
// drains the other, instead of the driver's single-threaded pageable staging.
struct PinnedStaging {
    static constexpr size_t kSlot = size_t(32) << 20;
    void* slot[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    std::mutex mu;  // one staged upload at a time per device
};

PinnedStaging* staging_for(int device) {
    static std::mutex mu;
    static std::map<int, PinnedStaging*> all;  // process lifetime (page-locked memory is reused)
    std::lock_guard<std::mutex> lk(mu);
    PinnedStaging*& st = all[device];
    if (!st) {
        auto* p = new PinnedStaging;
        bool ok = true;
        for (int i = 0; i < 2 && ok; ++i)
            ok = cudaHostAlloc(&p->slot[i], PinnedStaging::kSlot, cudaHostAllocDefault) == cudaSuccess &&
                 cudaEventCreateWithFlags(&p->done[i], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) {
            (void)cudaGetLastError();
            for (int i = 0; i < 2; ++i) {
                if (p->slot[i]) cudaFreeHost(p->slot[i]);
                if (p->done[i]) cudaEventDestroy(p->done[i]);
            }
            delete p;
            return nullptr;
        }
        st = p;
    }
    return st;
}

void parallel_memcpy(void* dst, const void* src, size_t n) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned T = std::min(8u, hw);
    if (n < (size_t(4) << 20) || T == 1) {
        memcpy(dst, src, n);
        return;
    }
    std::vector<std::thread> th;
    const size_t part = (n + T - 1) / T;
    for (unsigned t = 0; t < T; ++t) {
        const size_t a = t * part, b = std::min(n, a + part);
        if (a < b)
            th.emplace_back([=] { memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a); });
    }
    for (auto& x : th) x.join();
}

}  // namespace

void h2d_staged(Context& ctx, void* dst, const void* src_v, size_t len) {
    const char* src = static_cast<const char*>(src_v);
    cudaPointerAttributes attr{};
    const bool pinned = cudaPointerGetAttributes(&attr, src_v) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    (void)cudaGetLastError();
    // page-locked sources already copy at full link speed
    PinnedStaging* st = (!pinned && len >= (size_t(8) << 20)) ? staging_for(ctx.device()) : nullptr;
    if (!st) {
        h2d(ctx, dst, src, len);
        return;
    }
    std::lock_guard<std::mutex> lk(st->mu);
    size_t c = 0;
    for (size_t off = 0; off < len; off += PinnedStaging::kSlot, ++c) {
        const int i = static_cast<int>(c & 1);
        const size_t b = std::min(PinnedStaging::kSlot, len - off);
        cuda_check(cudaEventSynchronize(st->done[i]), "staging slot");  // its previous DMA has drained
        parallel_memcpy(st->slot[i], src + off, b);
        cuda_check(cudaMemcpyAsync(static_cast<char*>(dst) + off, st->slot[i], b, cudaMemcpyHostToDevice,
                                   ctx.stream()),
                   "host->device copy");
        cuda_check(cudaEventRecord(st->done[i], ctx.stream()), "staging event");
    }
    ctx.h2d_bytes += static_cast<long long>(len);
    // the slots are reused by the next upload only after these copies drain (event waits above)
}

// ---------------------------------------------------------------- caching pool
namespace {
struct PoolBlock {
    void* p;
    cudaStream_t stream;  // stream of the thread that freed it (nullptr: idle when freed)
    cudaEvent_t ready;    // recorded on `stream` at the free
};
std::mutex g_pool_mu;
std::multimap<std::pair<int, size_t>, PoolBlock> g_pool;  // (device, capacity) -> block
// recycled stream-order events per device (cudaEventCreate costs microseconds on every free of a
// latency-bound estimate; a recorded event is reusable once its block has been handed out again)
std::map<int, std::vector<cudaEvent_t>> g_free_events;

cudaEvent_t take_event(int device) {
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        auto& v = g_free_events[device];
        if (!v.empty()) {
            cudaEvent_t e = v.back();
            v.pop_back();
            return e;
        }
    }
    cudaEvent_t e = nullptr;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
        (void)cudaGetLastError();
        return nullptr;
    }
    return e;
}
thread_local cudaStream_t t_stream = nullptr;

size_t pool_round(size_t bytes) {
    const size_t g = bytes >= (size_t(1) << 21) ? (size_t(1) << 21) : 512;
    return (bytes + g - 1) / g * g;
}
}  // namespace

void set_current_stream(cudaStream_t s) { t_stream = s; }

void* pool_alloc(size_t bytes, size_t* capacity, int* device) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    const size_t want = pool_round(bytes);
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        const size_t cap_max = 2 * want + (size_t(1) << 21);
        auto first = g_pool.lower_bound({dev, want});
        auto pick = g_pool.end();
        // prefer a block this stream freed itself (stream order makes it reusable at once)
        for (auto it = first; it != g_pool.end() && it->first.first == dev && it->first.second <= cap_max; ++it) {
            if (pick == g_pool.end()) pick = it;
            if (it->second.stream == t_stream) {
                pick = it;
                break;
            }
        }
        if (pick != g_pool.end()) {
            PoolBlock b = pick->second;
            *capacity = pick->first.second;
            *device = dev;
            g_pool.erase(pick);
            if (b.ready) {
                if (b.stream != t_stream) {  // order this stream after the freeing stream's queued work
                    if (t_stream) cudaStreamWaitEvent(t_stream, b.ready, 0);
                    else cudaEventSynchronize(b.ready);
                }
                g_free_events[dev].push_back(b.ready);  // the wait above (if any) is already enqueued
            }
            return b.p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaErrorMemoryAllocation) {
        (void)cudaGetLastError();
        pool_release_all();
        e = cudaMalloc(&p, want);
    }
    cuda_check(e, "cudaMalloc");
    *capacity = want;
    *device = dev;
    return p;
}

void pool_free(void* p, size_t capacity, int device) {
    if (!p) return;
    PoolBlock b{p, t_stream, nullptr};
    if (t_stream) {
        int cur = 0;
        cudaGetDevice(&cur);
        if (cur != device) cudaSetDevice(device);
        b.ready = take_event(device);
        if (b.ready && cudaEventRecord(b.ready, t_stream) != cudaSuccess) {
            (void)cudaGetLastError();
            cudaEventDestroy(b.ready);
            b.ready = nullptr;
        }
        if (!b.ready) {  // could not tag the free: make the block idle before it can be reused
            cudaDeviceSynchronize();
            b.stream = nullptr;
        }
        if (cur != device) cudaSetDevice(cur);
    }
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_pool.insert({{device, capacity}, b});
}

void pool_release_all() {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : g_pool) {
        cudaSetDevice(kv.first.first);
        if (kv.second.ready) {
            cudaEventSynchronize(kv.second.ready);
            cudaEventDestroy(kv.second.ready);
        }
        cudaFree(kv.second.p);
    }
    g_pool.clear();
    for (auto& kv : g_free_events) {
        cudaSetDevice(kv.first);
        for (cudaEvent_t e : kv.second) cudaEventDestroy(e);
    }
    g_free_events.clear();
    cudaSetDevice(cur);
}

// ---------------------------------------------------------------- DevBuf
DevBuf::~DevBuf() { release(); }
DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
    if (this != &o) {
        release();
        p_ = o.p_, n_ = o.n_, cap_ = o.cap_, dev_ = o.dev_;
        o.p_ = nullptr, o.n_ = 0, o.cap_ = 0;
    }
    return *this;
}
void DevBuf::alloc(size_t bytes) {
    release();
    if (bytes == 0) return;
    p_ = pool_alloc(bytes, &cap_, &dev_);
    n_ = bytes;
}
void DevBuf::ensure(size_t bytes) {
    if (bytes > n_) alloc(bytes);
}
void DevBuf::release() {
    // blocks may still be read by queued work on the engine stream: every public entry
    // point synchronises before its buffers go out of scope, and reuse is stream-ordered
    if (p_) pool_free(p_, cap_, dev_);
    p_ = nullptr, n_ = 0, cap_ = 0;
}

// ---------------------------------------------------------------- Context
Context::Context(int device) : device_(device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        (void)cudaGetLastError();
        fail(kNoDevice, "no CUDA device is visible; the renyi_b200 path requires an sm_100a GPU");
    }
    if (device < 0 || device >= count) fail(kInvalidArgument, "device index out of range");
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10) fail(kNoDevice, std::string("renyi_b200 kernels target sm_100a; found ") + prop.name);
    sms_ = prop.multiProcessorCount;
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    probe_err.alloc(sizeof(int));
    cuda_check(cudaMemsetAsync(probe_err.as<int>(), 0, sizeof(int), stream_), "memset");
    gram_ticket.alloc(sizeof(unsigned));
    cuda_check(cudaMemsetAsync(gram_ticket.as<unsigned>(), 0, sizeof(unsigned), stream_), "memset");
    if (const char* e = std::getenv("RB_SYMV")) symv = std::string(e) != "0";
    if (const char* e = std::getenv("RB_SPECULATE")) speculate = std::string(e) != "0";
}

double* Context::pinned_dots(size_t count) {
    if (count > pin_cap_) {
        if (pin_dots_) {
            cuda_check(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");  // no copy still lands in it
            cudaFreeHost(pin_dots_);
            pin_dots_ = nullptr;
        }
        const size_t cap = std::max<size_t>(count, 4096);
        cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&pin_dots_), cap * sizeof(double), cudaHostAllocDefault),
                   "cudaHostAlloc");
        pin_cap_ = cap;
    }
    return pin_dots_;
}

cudaEvent_t Context::dots_event(int i) {
    if (!dots_ev_[i]) cuda_check(cudaEventCreateWithFlags(&dots_ev_[i], cudaEventDisableTiming), "cudaEventCreate");
    return dots_ev_[i];
}

cudaStream_t Context::comm_stream() {
    if (!comm_) {
        cuda_check(cudaStreamCreateWithFlags(&comm_, cudaStreamNonBlocking), "cudaStreamCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_main_, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&ev_comm_, cudaEventDisableTiming), "cudaEventCreate");
    }
    return comm_;
}

void Context::comm_after_main() {
    cudaStream_t c = comm_stream();
    cuda_check(cudaEventRecord(ev_main_, stream_), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(c, ev_main_, 0), "cudaStreamWaitEvent");
}

void Context::main_after_comm() {
    cuda_check(cudaEventRecord(ev_comm_, comm_stream()), "cudaEventRecord");
    cuda_check(cudaStreamWaitEvent(stream_, ev_comm_, 0), "cudaStreamWaitEvent");
}

Context::~Context() {
    cudaSetDevice(device_);
    // the members' scratch returns to the pool after this body: the stream is drained and no
    // longer tags those frees
    if (comm_) cudaStreamSynchronize(comm_);
    if (stream_) cudaStreamSynchronize(stream_);
    if (t_stream == stream_) t_stream = nullptr;
    if (t0_) cudaEventDestroy(t0_);
    if (t1_) cudaEventDestroy(t1_);
    for (auto& e : events_) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    if (pin_dots_) cudaFreeHost(pin_dots_);
    for (cudaEvent_t e : dots_ev_)
        if (e) cudaEventDestroy(e);
    if (ev_main_) cudaEventDestroy(ev_main_);
    if (ev_comm_) cudaEventDestroy(ev_comm_);
    if (comm_) cudaStreamDestroy(comm_);
    if (stream_) cudaStreamDestroy(stream_);
}

namespace {
std::string probe_key(int64_t n, int cols, uint64_t seed, const char* label, int kind) {
    return std::to_string(n) + "/" + std::to_string(cols) + "/" + std::to_string(seed) + "/" + label + "/" +
           std::to_string(kind);
}
}  // namespace

void Context::prefetch_probes(const std::vector<ProbeReq>& reqs) {
    if (probe_source != 1) return;
    if (probe_job_.valid()) probe_job_.wait();  // one batch at a time
    struct Job {
        std::vector<ProbeReq> reqs;
        std::vector<uint64_t> base;
        std::vector<Panel> panels;
        std::vector<std::promise<Panel>> done;
        std::unique_ptr<std::atomic<int>[]> left;
        std::vector<std::pair<int, int>> tasks;  // (panel, column), in request order
    };
    auto job = std::make_shared<Job>();
    for (const ProbeReq& r : reqs) {
        const std::string key = probe_key(r.n, r.cols, r.seed, r.label.c_str(), r.kind);
        if (r.kind != kProbeGaussian || r.cols <= 0 || probe_prefetch_.count(key)) continue;
        const int p = static_cast<int>(job->reqs.size());
        job->reqs.push_back(r);
        job->base.push_back(derive_key(r.seed, hash_name(r.label.c_str())));
        job->panels.push_back(std::make_shared<std::vector<double>>(static_cast<size_t>(r.n) * r.cols));
        job->done.emplace_back();
        probe_prefetch_.emplace(key, job->done.back().get_future().share());
        for (int j = 0; j < r.cols; ++j) job->tasks.emplace_back(p, j);
    }
    if (job->tasks.empty()) return;
    job->left.reset(new std::atomic<int>[job->reqs.size()]);
    for (size_t p = 0; p < job->reqs.size(); ++p) job->left[p] = job->reqs[p].cols;
    probe_job_ = std::async(std::launch::async, [job] {
        std::atomic<size_t> next{0};
        auto work = [&] {
            for (size_t t; (t = next.fetch_add(1)) < job->tasks.size();) {
                const auto [p, j] = job->tasks[t];
                const ProbeReq& r = job->reqs[p];
                probe_column(job->base[p], j, r.n, r.kind, job->panels[p]->data() + static_cast<int64_t>(j) * r.n);
                if (job->left[p].fetch_sub(1) == 1) job->done[p].set_value(job->panels[p]);
            }
        };
        // leave two hardware threads to the engine's own thread (kernel launches, synchronisations)
        const unsigned hw = std::thread::hardware_concurrency();
        const unsigned nt = hw > 3 ? hw - 2 : 1;
        std::vector<std::thread> pool;
        for (unsigned i = 1; i < nt; ++i) pool.emplace_back(work);
        work();
        for (auto& th : pool) th.join();
    });
}

Context::Panel Context::take_probes(int64_t n, int cols, uint64_t seed, const char* label, int kind) {
    auto it = probe_prefetch_.find(probe_key(n, cols, seed, label, kind));
    if (it != probe_prefetch_.end()) {
        Panel v = it->second.get();
        probe_prefetch_.erase(it);
        return v;
    }
    auto v = std::make_shared<std::vector<double>>(static_cast<size_t>(n) * cols);
    probe_panel_mt(n, cols, seed, label, kind, v->data());
    return v;
}

void Context::drop_prefetched_probes() {
    if (probe_job_.valid()) probe_job_.wait();
    probe_prefetch_.clear();
}

void Context::sync() {
    cuda_check(cudaStreamSynchronize(stream_), "stream synchronize");
    if (comm_) cuda_check(cudaStreamSynchronize(comm_), "comm stream synchronize");
}

void Context::prof_enable(bool on) {
    prof_ = on;
    prof_used_ = 0;
    prof_bytes_ = prof_flops_ = 0.0;
}
void Context::prof_account(double bytes, double flops) {
    if (!prof_) return;
    prof_bytes_ += bytes;
    prof_flops_ += flops;
}
void Context::timer_begin() {
    if (!t0_) {
        cuda_check(cudaEventCreate(&t0_), "cudaEventCreate");
        cuda_check(cudaEventCreate(&t1_), "cudaEventCreate");
    }
    cuda_check(cudaEventRecord(t0_, stream_), "cudaEventRecord");
}
double Context::timer_end_ms() {
    if (!t0_) fail(kInvalidArgument, "timer_end without timer_begin");
    cuda_check(cudaEventRecord(t1_, stream_), "cudaEventRecord");
    cuda_check(cudaEventSynchronize(t1_), "cudaEventSynchronize");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, t0_, t1_), "cudaEventElapsedTime");
    return ms;
}
void Context::prof_begin() {
    if (!prof_) return;
    if (prof_used_ == events_.size()) {
        cudaEvent_t a, b;
        cuda_check(cudaEventCreate(&a), "cudaEventCreate");
        cuda_check(cudaEventCreate(&b), "cudaEventCreate");
        events_.push_back({a, b});
    }
    cuda_check(cudaEventRecord(events_[prof_used_].first, stream_), "cudaEventRecord");
}
void Context::prof_end() {
    if (!prof_) return;
    cuda_check(cudaEventRecord(events_[prof_used_].second, stream_), "cudaEventRecord");
    ++prof_used_;
}
void Context::prof_read(int* n, double* ms, double* bytes, double* flops) {
    sync();
    *bytes = prof_bytes_;
    *flops = prof_flops_;
    prof_bytes_ = prof_flops_ = 0.0;
    double total = 0.0;
    for (size_t i = 0; i < prof_used_; ++i) {
        float t = 0.f;
        cuda_check(cudaEventElapsedTime(&t, events_[i].first, events_[i].second), "cudaEventElapsedTime");
        total += t;
    }
    *n = static_cast<int>(prof_used_);
    *ms = total;
    prof_used_ = 0;
}

namespace {

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

inline void launched(Context& ctx, cudaError_t e, const char* what) {
    cuda_check(e, what);
    ++ctx.launches;
}

void assign_shard(Context& ctx, KernelMatrix& k) {
    k.world = ctx.world();
    k.rank = ctx.rank();
    shard_rows(k.n, k.world, k.rank, &k.row0, &k.rows, &k.rpr);
}

}  // namespace

void shard_rows(int64_t n, int world, int rank, int64_t* row0, int64_t* rows, int64_t* rpr) {
    if (world < 1 || rank < 0 || rank >= world) fail(kInvalidArgument, "bad rank/world");
    // equal chunks (a multiple of 256 rows = one block-product row block; the last chunk shorter)
    // so the per-pass all-gather of the operand planes is uniform
    const int64_t per = round_up((n + world - 1) / world, 256);
    *rpr = per;
    *row0 = std::min<int64_t>(n, per * rank);
    *rows = std::min<int64_t>(n, per * (rank + 1)) - *row0;
}

// ---------------------------------------------------------------- kernel matrices
KernelPtr build_gaussian(Context& ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double sigma, int prec,
                         const double* y, int64_t dy, int64_t ldy, double sigma_y) {
    NvtxRange nvtx("kernel build (Gram)");
    // upload column-major as given; validate_samples (proj/src/kernel.cpp:25-29) runs on the device copy
    if (n < 2) fail(kInvalidArgument, "need at least 2 samples, got " + std::to_string(n));
    if (d < 1) fail(kInvalidArgument, "samples need at least one feature");
    if (ldx < n || (y && ldy < n)) fail(kInvalidArgument, "leading dimension smaller than the sample count");
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    DevBuf xs;
    const int64_t dt = d + (y ? dy : 0);
    xs.alloc(static_cast<size_t>(n) * dt * sizeof(double));
    // contiguous panels (ld == n) take the page-locked staged path when large
    if (ldx == n) h2d_staged(ctx, xs.as<double>(), x, static_cast<size_t>(n) * d * sizeof(double));
    else h2d_2d(ctx, xs.as<double>(), n * sizeof(double), x, ldx * sizeof(double), n * sizeof(double), d);
    if (y && ldy == n) h2d_staged(ctx, xs.as<double>() + n * d, y, static_cast<size_t>(n) * dy * sizeof(double));
    else if (y) h2d_2d(ctx, xs.as<double>() + n * d, n * sizeof(double), y, ldy * sizeof(double), n * sizeof(double), dy);
    KernelPtr k = build_gaussian_dev(ctx, xs.as<double>(), n, d, n, sigma, prec, y ? xs.as<double>() + n * d : nullptr,
                                     dy, n, sigma_y);
    ctx.sync();  // xs goes out of scope
    return k;
}

KernelPtr build_gaussian_dev(Context& ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double sigma, int prec,
                             const double* y, int64_t dy, int64_t ldy, double sigma_y) {
    NvtxRange nvtx("kernel build (Gram)");
    // build_kernel(X, GaussianKernel{sigma}) (proj/src/kernel.cpp:35-72), samples resident on the device
    if (n < 2) fail(kInvalidArgument, "need at least 2 samples, got " + std::to_string(n));
    if (d < 1) fail(kInvalidArgument, "samples need at least one feature");
    if (!(sigma > 0.0)) fail(kInvalidArgument, "gaussian kernel needs sigma > 0");
    if (y) {
        if (dy < 1) fail(kInvalidArgument, "second variable needs at least one feature");
        if (!(sigma_y > 0.0)) fail(kInvalidArgument, "gaussian kernel needs sigma > 0");
    }
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    // finiteness (kernel.cpp:27) and, for fp32, representability of the squared norms
    ctx.small.ensure(4 * sizeof(unsigned));
    unsigned* flags = ctx.small.as<unsigned>();
    cuda_check(cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned), ctx.stream()), "memset");
    launched(ctx, launch_check_samples(x, n, static_cast<int>(d), 1, ldx, flags, ctx.stream()), "check_samples");
    if (y) launched(ctx, launch_check_samples(y, n, static_cast<int>(dy), 1, ldy, flags, ctx.stream()), "check_samples");
    unsigned hf[2];
    d2h(ctx, hf, flags, sizeof(hf));
    ctx.sync();
    if (hf[0]) fail(kNonFinite, "sample matrix contains non-finite values");
    float mx;
    std::memcpy(&mx, &hf[1], sizeof(float));
    if (prec != kF64 && mx > 1e18f) fail(kNonFinite, "sample values exceed the fp32 range of the fp32 configuration");

    auto k = std::make_unique<KernelMatrix>();
    k->n = n;
    k->prec = prec;
    assign_shard(ctx, *k);
    if (prec == kF64 && k->world > 1) fail(kInvalidArgument, "the fp64 configuration is single-rank");
    k->ld = matrix_pitch(n);
    const double inv_n = 1.0 / static_cast<double>(n);
    k->normalized = true;
    k->a_norm = 1.0;
    if (prec == kMF) {
        // matrix-free: keep bf16 samples and the per-sample bias; kernel entries are recomputed per pass.
        // One variable: exp(-|x_i-x_j|^2/(2σ^2)) from bf16(x). Joint (x, y): the normalised Hadamard
        // product is the Gaussian of the concatenated features [x/σx, y/σy] with σ = 1.
        const int64_t dt = d + (y ? dy : 0);
        if (dt > 128) fail(kInvalidArgument, "the matrix-free path supports up to 128 features");
        k->dp = dt <= 64 ? 64 : 128;
        k->dfeat = static_cast<int>(dt);
        const double l2e = 1.4426950408889634;
        const int64_t npad = round_up(n, 128);
        k->xb.alloc(static_cast<size_t>(npad) * k->dp * sizeof(__nv_bfloat16));
        k->xa.alloc(static_cast<size_t>(2) * npad * mf_aug_cols() * sizeof(__nv_bfloat16));
        cuda_check(cudaMemsetAsync(k->xb.as<void>(), 0, k->xb.bytes(), ctx.stream()), "memset");
        cuda_check(cudaMemsetAsync(k->xa.as<void>(), 0, k->xa.bytes(), ctx.stream()), "memset");
        if (!y) {
            k->c2 = l2e / (sigma * sigma);
            launched(ctx,
                     launch_mf_prepare(x, n, static_cast<int>(d), 1, ldx, k->dp, npad, k->xb.as<__nv_bfloat16>(),
                                       k->xa.as<__nv_bfloat16>(), ctx.stream()),
                     "mf_prepare");
        } else {
            DevBuf cat;
            cat.alloc(static_cast<size_t>(n) * dt * sizeof(double));
            launched(ctx, launch_scale_columns(x, n, static_cast<int>(d), 1, ldx, 1.0 / sigma, cat.as<double>(),
                                               ctx.stream()),
                     "scale_columns");
            launched(ctx, launch_scale_columns(y, n, static_cast<int>(dy), 1, ldy, 1.0 / sigma_y,
                                               cat.as<double>() + n * d, ctx.stream()),
                     "scale_columns");
            k->c2 = l2e;
            launched(ctx,
                     launch_mf_prepare(cat.as<double>(), n, static_cast<int>(dt), 1, n, k->dp, npad,
                                       k->xb.as<__nv_bfloat16>(), k->xa.as<__nv_bfloat16>(), ctx.stream()),
                     "mf_prepare");
            ctx.sync();
        }
        k->unscale = inv_n;
        return k;
    }
    GramArgs g;
    g.x = x;
    g.dx = static_cast<int>(d);
    g.x_rs = 1, g.x_cs = ldx;
    g.inv_two_sigma2_x = 1.0 / (2.0 * sigma * sigma);
    g.y = y;
    g.dy = static_cast<int>(dy);
    g.y_rs = 1, g.y_cs = ldy;
    g.inv_two_sigma2_y = y ? 1.0 / (2.0 * sigma_y * sigma_y) : 0.0;
    g.n = n;
    g.row0 = k->row0;
    g.rows = k->rows;
    g.ld = k->ld;
    g.inv_n = inv_n;
    g.f32_compute = prec == kF32 ? 1 : 0;
    const size_t elems = static_cast<size_t>(k->rows) * k->ld;
    if (prec == kF32) {
        k->hi.alloc(elems * sizeof(__half));
        k->lo.alloc(elems * sizeof(__half));
        k->unscale = inv_n / kSplitScale;
        DevBuf scratch;
        scratch.alloc(gram_split_scratch_bytes(g));
        launched(ctx, launch_gram_split(g, k->hi.as<__half>(), k->lo.as<__half>(), scratch.as<void>(), ctx.stream()),
                 "gram_split");  // scratch goes back to the pool: reuse is stream-ordered
    } else {
        k->a64.alloc(elems * sizeof(double));
        k->unscale = 1.0;
        launched(ctx, launch_gram_f64(g, k->a64.as<double>(), ctx.stream()), "gram_f64");
    }
    return k;
}

KernelPtr build_polynomial(Context& ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int degree, double offset,
                           int prec) {
    if (n < 2) fail(kInvalidArgument, "need at least 2 samples, got " + std::to_string(n));
    if (d < 1) fail(kInvalidArgument, "samples need at least one feature");
    if (ldx < n) fail(kInvalidArgument, "leading dimension smaller than the sample count");
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    DevBuf xs;
    xs.alloc(static_cast<size_t>(n) * d * sizeof(double));
    if (ldx == n) h2d_staged(ctx, xs.as<double>(), x, static_cast<size_t>(n) * d * sizeof(double));
    else h2d_2d(ctx, xs.as<double>(), n * sizeof(double), x, ldx * sizeof(double), n * sizeof(double), d);
    KernelPtr k = build_polynomial_dev(ctx, xs.as<double>(), n, d, n, degree, offset, prec);
    ctx.sync();  // xs goes out of scope
    return k;
}

KernelPtr build_polynomial_dev(Context& ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int degree,
                               double offset, int prec) {
    NvtxRange nvtx("kernel build (polynomial Gram)");
    // validate_samples (kernel.cpp:25-29), then the spec (kernel.cpp:44-45)
    if (n < 2) fail(kInvalidArgument, "need at least 2 samples, got " + std::to_string(n));
    if (d < 1) fail(kInvalidArgument, "samples need at least one feature");
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    ctx.small.ensure(4 * sizeof(unsigned));
    unsigned* flags = ctx.small.as<unsigned>();
    cuda_check(cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned), ctx.stream()), "memset");
    launched(ctx, launch_check_samples(x, n, static_cast<int>(d), 1, ldx, flags, ctx.stream()), "check_samples");
    unsigned hf[2];
    d2h(ctx, hf, flags, sizeof(hf));
    ctx.sync();
    if (hf[0]) fail(kNonFinite, "sample matrix contains non-finite values");
    if (degree < 1) fail(kInvalidArgument, "polynomial kernel needs degree >= 1");
    if (!(offset >= 0.0)) fail(kInvalidArgument, "polynomial kernel needs offset >= 0");
    if (prec == kMF) fail(kInvalidArgument, "the matrix-free path recomputes Gaussian kernel entries only");

    auto k = std::make_unique<KernelMatrix>();
    k->n = n;
    k->prec = prec;
    assign_shard(ctx, *k);
    if (prec == kF64 && k->world > 1) fail(kInvalidArgument, "the fp64 configuration is single-rank");
    k->ld = matrix_pitch(n);
    const double inv_n = 1.0 / static_cast<double>(n);
    k->normalized = true;
    k->a_norm = 1.0;  // |A_ij| <= 1/n (Cauchy-Schwarz on the PSD kernel): row sums <= 1
    GramArgs g{};
    g.x = x;
    g.dx = static_cast<int>(d);
    g.x_rs = 1, g.x_cs = ldx;
    g.n = n;
    g.row0 = k->row0;
    g.rows = k->rows;
    g.ld = k->ld;
    g.inv_n = inv_n;
    const size_t elems = static_cast<size_t>(k->rows) * k->ld;
    DevBuf isd;
    isd.alloc(static_cast<size_t>(n) * sizeof(double));
    cuda_check(cudaMemsetAsync(flags, 0, sizeof(unsigned), ctx.stream()), "memset");
    cuda_check(cudaMemsetAsync(flags + 1, 0xFF, sizeof(unsigned), ctx.stream()), "memset");
    if (prec == kF32) {
        k->hi.alloc(elems * sizeof(__half));
        k->lo.alloc(elems * sizeof(__half));
        k->unscale = inv_n / kSplitScale;
        launched(ctx, launch_poly_gram(g, degree, offset, isd.as<double>(), k->hi.as<__half>(), k->lo.as<__half>(),
                                       nullptr, flags, ctx.stream()),
                 "poly_gram");
    } else {
        k->a64.alloc(elems * sizeof(double));
        k->unscale = 1.0;
        launched(ctx, launch_poly_gram(g, degree, offset, isd.as<double>(), nullptr, nullptr, k->a64.as<double>(),
                                       flags, ctx.stream()),
                 "poly_gram");
    }
    // a non-finite entry in any rank's rows fails every rank (the diagonal is computed on all of them)
    if (ctx.exchange) ctx.exchange->allreduce_max_u32(flags, 1, ctx.stream());
    d2h(ctx, hf, flags, sizeof(hf));
    ctx.sync();  // isd goes out of scope
    if (hf[0]) fail(kNonFinite, "kernel evaluation produced non-finite values");
    if (hf[1] != 0xFFFFFFFFu)
        fail(kZeroDiagonal, "kernel diagonal entry " + std::to_string(hf[1]) + " is not positive");
    return k;
}

namespace {
// n x n fp64 Gram of host samples into a host column-major matrix (the Gram is exactly symmetric, so
// the device's row-major rows are the host's columns)
template <typename Launch>
void raw_gram(Context& ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double* k, Launch&& launch) {
    if (n < 1 || d < 1) fail(kInvalidArgument, "samples must be non-empty");
    if (ldx < n) fail(kInvalidArgument, "leading dimension smaller than the sample count");
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    DevBuf xs, out;
    xs.alloc(static_cast<size_t>(n) * d * sizeof(double));
    h2d_2d(ctx, xs.as<double>(), n * sizeof(double), x, ldx * sizeof(double), n * sizeof(double), d);
    const int64_t ld = matrix_pitch(n);
    out.alloc(static_cast<size_t>(n) * ld * sizeof(double));
    GramArgs g{};
    g.x = xs.as<double>();
    g.dx = static_cast<int>(d);
    g.x_rs = 1, g.x_cs = n;
    g.n = n, g.row0 = 0, g.rows = n, g.ld = ld;
    g.inv_n = 1.0;  // fl(1·K) = K: the unnormalised Gram
    launched(ctx, launch(g, out.as<double>()), "gram");
    d2h_2d(ctx, k, n * sizeof(double), out.as<double>(), ld * sizeof(double), n * sizeof(double), n);
    ctx.sync();
}
}  // namespace

void ops_gaussian_gram(Context& ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double sigma, double* k) {
    NvtxRange nvtx("ops::gaussian_gram");
    raw_gram(ctx, x, n, d, ldx, k, [&](GramArgs& g, double* out) {
        g.inv_two_sigma2_x = 1.0 / (2.0 * sigma * sigma);  // ops.cpp:42
        return launch_gram_f64(g, out, ctx.stream());
    });
}

void ops_polynomial_gram(Context& ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int degree, double offset,
                         double* k) {
    NvtxRange nvtx("ops::polynomial_gram");
    ctx.small.ensure(4 * sizeof(unsigned));  // the raw op checks nothing (ops.cpp:58-64); flags unused
    raw_gram(ctx, x, n, d, ldx, k, [&](GramArgs& g, double* out) {
        return launch_poly_gram(g, degree, offset, nullptr, nullptr, nullptr, out, ctx.small.as<unsigned>(),
                                ctx.stream());
    });
}

void ops_hadamard_scaled(Context& ctx, const double* a, const double* b, int64_t rows, int64_t cols, double scale,
                         double* c) {
    NvtxRange nvtx("ops::hadamard_scaled");
    if (rows < 0 || cols < 0) fail(kInvalidArgument, "matrix sizes must be non-negative");
    const int64_t count = rows * cols;
    if (count == 0) return;
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    DevBuf da, db;
    da.alloc(static_cast<size_t>(count) * sizeof(double));
    db.alloc(static_cast<size_t>(count) * sizeof(double));
    h2d(ctx, da.as<double>(), a, static_cast<size_t>(count) * sizeof(double));
    h2d(ctx, db.as<double>(), b, static_cast<size_t>(count) * sizeof(double));
    launched(ctx, launch_scaled_product(da.as<double>(), db.as<double>(), count, scale, da.as<double>(), ctx.stream()),
             "scaled_product");
    d2h(ctx, c, da.as<double>(), static_cast<size_t>(count) * sizeof(double));
    ctx.sync();
}

KernelPtr from_matrix(Context& ctx, const double* a, int64_t n, int prec) {
    if (n < 1) fail(kInvalidArgument, "matrix must be non-empty");
    if (prec == kMF) fail(kInvalidArgument, "the matrix-free precision builds from samples only");
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    auto k = std::make_unique<KernelMatrix>();
    k->n = n;
    k->prec = prec;
    assign_shard(ctx, *k);
    if (prec == kF64 && k->world > 1) fail(kInvalidArgument, "the fp64 configuration is single-rank");
    k->ld = matrix_pitch(n);
    k->normalized = false;
    std::vector<double> rm(static_cast<size_t>(k->rows) * k->ld, 0.0);
    double mx = 0.0, norm = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double rs = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            const double v = a[i + j * n];
            if (!std::isfinite(v)) fail(kNonFinite, "matrix contains non-finite values");
            rs += std::abs(v);
            mx = std::max(mx, std::abs(v));
        }
        norm = std::max(norm, rs);
    }
    for (int64_t i = 0; i < k->rows; ++i)
        for (int64_t j = 0; j < n; ++j) rm[i * k->ld + j] = a[(k->row0 + i) + j * n];
    k->a_norm = norm;
    DevBuf up;
    up.alloc(rm.size() * sizeof(double));
    h2d(ctx, up.as<double>(), rm.data(), rm.size() * sizeof(double));
    if (prec == kF32) {
        int e = 0;
        if (mx > 0.0) {
            int E;
            std::frexp(mx, &E);  // mx < 2^E
            e = kSplitScaleLog2 - E;
        }
        const double scale = std::ldexp(1.0, e);
        k->unscale = std::ldexp(1.0, -e);
        const size_t elems = static_cast<size_t>(k->rows) * k->ld;
        k->hi.alloc(elems * sizeof(__half));
        k->lo.alloc(elems * sizeof(__half));
        cuda_check(cudaMemsetAsync(k->hi.as<__half>(), 0, elems * sizeof(__half), ctx.stream()), "memset");
        cuda_check(cudaMemsetAsync(k->lo.as<__half>(), 0, elems * sizeof(__half), ctx.stream()), "memset");
        launched(ctx,
                 launch_matrix_to_split(up.as<double>(), k->rows, n, k->ld, scale, k->hi.as<__half>(),
                                        k->lo.as<__half>(), k->ld, ctx.stream()),
                 "matrix_to_split");
        ctx.sync();
    } else {
        k->unscale = 1.0;
        ctx.sync();
        k->a64 = std::move(up);
    }
    return k;
}

KernelPtr hadamard_joint(Context& ctx, const KernelMatrix& a, const KernelMatrix& b) {
    // proj/src/kernel.cpp:74-101 with L = 2 (the product is commutative, so the
    // canonical content order only matters for L >= 3 rounding)
    if (a.n != b.n)
        fail(kSizeMismatch,
             "hadamard_joint kernel sizes differ: " + std::to_string(a.n) + " vs " + std::to_string(b.n));
    if (a.prec != b.prec) fail(kInvalidArgument, "hadamard_joint needs kernels of the same precision");
    if (a.prec == kMF)
        fail(kInvalidArgument, "matrix-free joints are built from samples (renyi_kernel_build_gaussian_joint)");
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    auto c = std::make_unique<KernelMatrix>();
    c->n = a.n, c->row0 = a.row0, c->rows = a.rows, c->ld = a.ld, c->prec = a.prec;
    c->rpr = a.rpr, c->world = a.world, c->rank = a.rank;
    const double nd = static_cast<double>(a.n);
    const double inv_n = 1.0 / nd;
    // |n A_ij B_ij| row sums: <= n * max|B| * ||A||_inf (<= 1 for normalised factors)
    c->a_norm = (a.normalized && b.normalized) ? 1.0 : std::max(1.0, a.a_norm * b.a_norm * nd);
    c->normalized = a.normalized && b.normalized;
    const size_t elems = static_cast<size_t>(c->rows) * c->ld;
    if (a.prec == kF32) {
        c->unscale = inv_n / kSplitScale;
        const double factor = nd * a.unscale * b.unscale / c->unscale;
        const double diag = inv_n / c->unscale;
        c->hi.alloc(elems * sizeof(__half));
        c->lo.alloc(elems * sizeof(__half));
        launched(ctx,
                 launch_hadamard_split(a.hi.as<__half>(), a.lo.as<__half>(), b.hi.as<__half>(), b.lo.as<__half>(),
                                       c->rows, c->n, c->ld, c->row0, factor, diag, c->hi.as<__half>(),
                                       c->lo.as<__half>(), ctx.stream()),
                 "hadamard_split");
    } else {
        c->unscale = 1.0;
        c->a64.alloc(elems * sizeof(double));
        launched(ctx,
                 launch_hadamard_f64(a.a64.as<double>(), b.a64.as<double>(), c->rows, c->n, c->ld, c->row0, nd,
                                     c->a64.as<double>(), ctx.stream()),
                 "hadamard_f64");
    }
    ctx.sync();
    return c;
}

// canonical ordering key of a stored kernel: the row hashes folded in row order (equal content, equal
// key; the reference orders by an FNV-1a of the fp64 bytes, kernel.cpp:13-23,83-88 -- any content key
// gives the same permutation invariance)
uint64_t content_key(Context& ctx, const KernelMatrix& k) {
    DevBuf rh;
    rh.alloc(static_cast<size_t>(std::max<int64_t>(k.rows, 1)) * sizeof(uint64_t));
    launched(ctx,
             launch_row_hash(k.prec == kF64 ? k.a64.as<double>() : nullptr, k.prec == kF64 ? nullptr : k.hi.as<__half>(),
                             k.prec == kF64 ? nullptr : k.lo.as<__half>(), k.rows, k.n, k.ld, rh.as<uint64_t>(),
                             ctx.stream()),
             "row_hash");
    std::vector<uint64_t> h(static_cast<size_t>(k.rows));
    d2h(ctx, h.data(), rh.as<uint64_t>(), h.size() * sizeof(uint64_t));
    ctx.sync();
    uint64_t key = 0xcbf29ce484222325ULL;
    for (uint64_t v : h) key = mix64(key ^ v);
    return key;
}

KernelPtr hadamard_joint_n(Context& ctx, const std::vector<const KernelMatrix*>& ks) {
    // proj/src/kernel.cpp:74-101 for any L: factors in a canonical content order (bitwise permutation
    // invariant), p = M_0 ∘ ... with the single n^(L-1) scale on the last product, diag 1/n
    if (ks.size() < 2) fail(kInvalidArgument, "hadamard_joint needs at least 2 kernels");
    const KernelMatrix& k0 = *ks.front();
    for (const KernelMatrix* k : ks)
        if (k->n != k0.n)
            fail(kSizeMismatch,
                 "hadamard_joint kernel sizes differ: " + std::to_string(k0.n) + " vs " + std::to_string(k->n));
    if (ks.size() == 2) return hadamard_joint(ctx, *ks[0], *ks[1]);  // commutative: order-free
    if (static_cast<int>(ks.size()) > kMaxJoint)
        fail(kInvalidArgument, "hadamard_joint supports up to " + std::to_string(kMaxJoint) + " kernels");
    for (const KernelMatrix* k : ks) {
        if (k->prec != k0.prec) fail(kInvalidArgument, "hadamard_joint needs kernels of the same precision");
        if (k->prec == kMF)
            fail(kInvalidArgument, "matrix-free joints are built from samples (renyi_kernel_build_gaussian_joint)");
        if (k->world != 1) fail(kInvalidArgument, "hadamard_joint of three or more kernels is single-rank");
        if (k->groups > 1) fail(kInvalidArgument, "hadamard_joint needs single kernels, not grouped stacks");
    }
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    std::vector<std::pair<uint64_t, const KernelMatrix*>> order;
    for (const KernelMatrix* k : ks) order.push_back({content_key(ctx, *k), k});
    std::stable_sort(order.begin(), order.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    const double nd = static_cast<double>(k0.n), inv_n = 1.0 / nd;
    double scale = 1.0;
    for (size_t l = 1; l < order.size(); ++l) scale *= nd;  // kernel.cpp:91-92
    HadamardFactors hf{};
    hf.count = static_cast<int>(order.size());
    bool normalized = true;
    for (int l = 0; l < hf.count; ++l) {
        const KernelMatrix& k = *order[l].second;
        hf.a64[l] = k.prec == kF64 ? k.a64.as<double>() : nullptr;
        hf.hi[l] = k.prec == kF64 ? nullptr : k.hi.as<__half>();
        hf.lo[l] = k.prec == kF64 ? nullptr : k.lo.as<__half>();
        hf.unscale[l] = k.unscale;
        normalized = normalized && k.normalized;
    }
    auto c = std::make_unique<KernelMatrix>();
    c->n = k0.n, c->row0 = k0.row0, c->rows = k0.rows, c->ld = k0.ld, c->prec = k0.prec;
    c->rpr = k0.rpr, c->world = k0.world, c->rank = k0.rank;
    c->normalized = normalized;
    c->a_norm = normalized ? 1.0 : [&] {
        double b = 1.0;
        for (const KernelMatrix* k : ks) b *= std::max(1.0, k->a_norm);
        return std::max(1.0, b * scale);
    }();
    const size_t elems = static_cast<size_t>(c->rows) * c->ld;
    if (c->prec == kF32) {
        c->unscale = inv_n / kSplitScale;
        c->hi.alloc(elems * sizeof(__half));
        c->lo.alloc(elems * sizeof(__half));
        launched(ctx, launch_hadamard_n(hf, c->rows, c->n, c->ld, c->row0, scale, inv_n, c->unscale, nullptr,
                                        c->hi.as<__half>(), c->lo.as<__half>(), ctx.stream()),
                 "hadamard_n");
    } else {
        c->unscale = 1.0;
        c->a64.alloc(elems * sizeof(double));
        launched(ctx, launch_hadamard_n(hf, c->rows, c->n, c->ld, c->row0, scale, inv_n, 1.0, c->a64.as<double>(),
                                        nullptr, nullptr, ctx.stream()),
                 "hadamard_n");
    }
    ctx.sync();
    return c;
}

void download(Context& ctx, const KernelMatrix& k, double* out) {
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    if (k.prec == kMF) fail(kInvalidArgument, "matrix-free kernels are never materialised");
    std::vector<double> rm(static_cast<size_t>(k.rows) * k.n);
    if (k.prec == kF32) {
        DevBuf tmp;
        tmp.alloc(rm.size() * sizeof(double));
        launched(ctx,
                 launch_split_to_f64(k.hi.as<__half>(), k.lo.as<__half>(), k.rows, k.n, k.ld, k.unscale,
                                     tmp.as<double>(), k.n, ctx.stream()),
                 "split_to_f64");
        d2h(ctx, rm.data(), tmp.as<double>(), rm.size() * sizeof(double));
        ctx.sync();
    } else {
        d2h_2d(ctx, rm.data(), k.n * sizeof(double), k.a64.as<double>(), k.ld * sizeof(double), k.n * sizeof(double),
               k.rows);
        ctx.sync();
    }
    for (int64_t i = 0; i < k.rows; ++i)
        for (int64_t j = 0; j < k.n; ++j) out[(k.row0 + i) + j * k.n] = rm[i * k.n + j];
}

// ---------------------------------------------------------------- panel sessions
namespace {

bool split_operand(const Context& ctx, bool vectors_out) {
    return ctx.operand_mode == 0 || (ctx.operand_mode == 2 && vectors_out);
}

// a seeded Gaussian probe panel drawn on the device hit the reference's redraw branch (u1 <= 0,
// p = 2^-53 per pair, rng.cpp:47): the device draws cannot follow it, so the estimate is refused
void check_probe_err(Context& ctx, int err) {
    if (!err) return;
    cudaMemsetAsync(ctx.probe_err.as<int>(), 0, sizeof(int), ctx.stream());
    ctx.sync();
    fail(kInternal, "probe stream hit the 2^-53 Box-Muller redraw; pass the probes explicitly");
}

class PanelSession {
public:
    // ws: the session's buffers (default ctx.ws); tri: the panel is one operand of a fused
    // mutual-information pass (128-row stream-K plan of launch_block_av_tri)
    PanelSession(Context& ctx, const KernelMatrix& k, const double* x, int64_t ldx, int s, int max_passes,
                 double* acc_out, double acc_coef0, bool vectors_out, PanelWorkspace* ws = nullptr, bool tri = false)
        : ctx_(ctx), w_(ws ? *ws : ctx.ws), k_(k), s_(s), max_passes_(max_passes), acc_(acc_out) {
        if (s < 1 || s > kMaxPanelCols) fail(kInternal, "panel width must be in [1,128]");
        if (k.world != ctx.world() || k.rank != ctx.rank())
            fail(kInvalidArgument, "kernel matrix was built for a different rank layout");
        rows_ = k.rows;
        ld_ = k.rpr;  // state [s][rpr] (local rows); operand planes [world][s][rpr]
        mf_ = k.prec == kMF;
        // row-sharded: each pass's product runs as two K windows, the rank's own operand chunk (ready
        // after its own epilogue, overlapping the all-gather of the others on the comm stream) and the
        // rest; both windows' partials meet in the epilogue (SURVEY §8(e) "overlap")
        split_ = ctx.exchange && ctx.world() > 1 && k.prec != kF64;
        if (split_) ctx.main_after_comm();  // a previous session's last gather may still be in flight
        const KWindow own{k.row0, rows_}, rest{k.row0 + rows_, k.n - rows_};
        // s = 1 on one whole symmetric fp32 matrix: the upper-triangle product (half the bytes of A)
        symv_ = k.prec == kF32 && s == 1 && !tri && !split_ && k.world == 1 && k.groups <= 1 && k.normalized &&
                ctx.symv && k.rows == k.n && split_operand(ctx, vectors_out);
        if (symv_) {
            nb_ = symv_blocks(k.n);
            plan_ = StreamKPlan{};
            plan_.row_blocks = static_cast<int>(nb_);
            plan_.rows_per_block = 128;
            plan_.cluster = 1;
            plan_.slots = static_cast<int>(nb_ * nb_);
            plan_.grid = ctx.sms();  // persistent: one CTA per SM (a 3-stage 65 KB TMA ring each)
            npad_ = 1;
        } else if (k.prec == kF32) {
            const int grid = k.group_grid > 0 ? k.group_grid : ctx.grid > 0 ? ctx.grid : ctx.sms();
            auto mk = [&](KWindow w) {
                return tri ? make_tri_plan(rows_, k.n, grid, ctx.kc, w) : make_streamk_plan(rows_, k.n, grid, ctx.kc, w);
            };
            plan_ = mk(split_ ? own : KWindow{});
            if (split_) plan2_ = mk(rest);
            npad_ = tc_npad(s);
        } else if (mf_) {
            const int grid = ctx.grid > 0 ? ctx.grid : ctx.sms();
            plan_ = make_mf_plan(rows_, k.n, grid, std::max(1, ctx.mf_kc), split_ ? own : KWindow{});
            if (split_) plan2_ = make_mf_plan(rows_, k.n, grid, std::max(1, ctx.mf_kc), rest);
            npad_ = tc_npad(s);
        } else {
            plan_ = make_f64_plan(rows_, k.n, 2 * ctx.sms());
            npad_ = f64_npad(s);
        }
        const int rpb = plan_.rows_per_block;
        R_ = static_cast<int>((rows_ + rpb - 1) / rpb);
        const bool f32 = k.prec != kF64;  // fp32 state for the split and matrix-free paths
        const size_t st = f32 ? sizeof(float) : sizeof(double);
        for (auto& b : w_.state) b.ensure(static_cast<size_t>(s) * ld_ * st);
        if (f32) {
            // rank chunks of the operand planes: s columns of rpr rows, plus (row-sharded) a 512-byte tail
            // carrying the rank's column maxima of the pass through the same all-gather (gather_planes)
            slice_elems_ = static_cast<int64_t>(s) * ld_ + (ctx.exchange ? kTailElems : 0);
            const size_t plane = static_cast<size_t>(k.world) * slice_elems_ * sizeof(__half);
            w_.vhi.ensure(plane);
            // rows past n in the last chunk are never written: keep them zero (A's columns there are
            // TMA-zero, but 0 x garbage could be NaN)
            cuda_check(cudaMemsetAsync(w_.vhi.as<__half>(), 0, plane, ctx.stream()), "memset");
            if (split_operand(ctx, vectors_out) && !mf_) {
                w_.vlo.ensure(plane);
                cuda_check(cudaMemsetAsync(w_.vlo.as<__half>(), 0, plane, ctx.stream()), "memset");
            }
            slice_ = static_cast<size_t>(k.rank) * slice_elems_;
        }
        // the matrix-free P·V product takes one fp16 operand plane (P itself is fp16)
        vlo_ = (k.prec == kF32 && split_operand(ctx, vectors_out)) ? w_.vlo.as<__half>() : nullptr;
        const size_t P1 = static_cast<size_t>(max_passes) + 1;
        w_.stats.ensure(P1 * 3 * std::max(R_, 1) * s * sizeof(double));
        w_.red.ensure(P1 * 3 * s * sizeof(double));
        w_.cmax.ensure(P1 * s * sizeof(unsigned));
        w_.eexp.ensure(P1 * s * sizeof(int));
        cuda_check(cudaMemsetAsync(w_.cmax.as<unsigned>(), 0, P1 * s * sizeof(unsigned), ctx.stream()), "memset");
        if (f32) {
            w_.partial.ensure(static_cast<size_t>(plan_.slots) * npad_ * rpb * sizeof(float));
            if (split_) w_.partial2.ensure(static_cast<size_t>(plan2_.slots) * npad_ * rpb * sizeof(float));
            PrepArgs<float> p{};
            p.x = x, p.ldx = ldx, p.rows = rows_, p.rows_per_block = rpb, p.s = s, p.ld = ld_;
            p.t0 = buf<float>(0);
            p.cmax0 = w_.cmax.as<unsigned>();
            p.stats = w_.stats.as<double>();
            p.e0 = w_.eexp.as<int>();
            p.vop = w_.vhi.as<__half>() + slice_;
            p.vop_lo = vlo_ ? vlo_ + slice_ : nullptr;
            p.acc = acc_out, p.acc_coef = acc_coef0;
            if (rows_ > 0) launched(ctx, launch_prepare_split_stats(p, ctx.stream()), "prepare");
            if (ctx.exchange) ctx.exchange->allreduce_max_u32(w_.cmax.as<unsigned>(), s, ctx.stream());
            launched(ctx, launch_prepare_split_planes(p, ctx.stream()), "prepare");  // also writes e0
            gather_planes(-1);
        } else {
            w_.partial.ensure(static_cast<size_t>(plan_.slots) * npad_ * rpb * sizeof(double));
            PrepArgs<double> p{};
            p.x = x, p.ldx = ldx, p.rows = rows_, p.rows_per_block = rpb, p.s = s, p.ld = ld_;
            p.t0 = buf<double>(0);
            p.cmax0 = w_.cmax.as<unsigned>();
            p.stats = w_.stats.as<double>();
            p.acc = acc_out, p.acc_coef = acc_coef0;
            launched(ctx, launch_prepare_f64(p, ctx.stream()), "prepare");
        }
    }

    // all ranks' operand slices -> full planes (in place), on the comm stream after the epilogue that
    // wrote this rank's slice. The column maxima of pass `cmax_pass` (>= 0; the next epilogue's plane
    // scale) ride in the tail of every rank's chunk and are merged after the gather -- no separate
    // all-reduce. The next product's own-chunk window runs meanwhile; its other window waits for these
    // (product()).
    void gather_planes(int cmax_pass) {
        NvtxRange nvtx("all-gather operand planes");
        if (!ctx_.exchange || k_.prec == kF64) return;
        unsigned* cm = cmax_pass >= 0 ? w_.cmax.as<unsigned>() + static_cast<size_t>(cmax_pass) * s_ : nullptr;
        __half* tail = w_.vhi.as<__half>() + slice_ + static_cast<int64_t>(s_) * ld_;
        if (cm)
            cuda_check(cudaMemcpyAsync(tail, cm, static_cast<size_t>(s_) * sizeof(unsigned), cudaMemcpyDeviceToDevice,
                                       ctx_.stream()),
                       "column maxima -> chunk tail");
        ctx_.comm_after_main();
        cudaStream_t cs = ctx_.comm_stream();
        const size_t chunk = static_cast<size_t>(slice_elems_) * sizeof(__half);
        ctx_.exchange->allgather_inplace(w_.vhi.as<__half>(), chunk, cs);
        if (vlo_) ctx_.exchange->allgather_inplace(vlo_, chunk, cs);
        if (cm)
            launched(ctx_,
                     launch_merge_tails(w_.vhi.as<__half>(), slice_elems_, static_cast<int64_t>(s_) * ld_, k_.world, s_,
                                        cm, cs),
                     "merge_tails");
    }

    void step(double a1, double a2, double a3, double acc_coef) {
        if (k_.prec != kF64) {
            product();
            finish(a1, a2, a3, acc_coef);
        } else {
            step_f64(a1, a2, a3, acc_coef);
        }
    }

    // the operand planes of the next pass, the partial buffers and the plans (fused MI pass); split():
    // two K windows (plan: own operand chunk, plan2: the rest after the all-gather)
    SplitPanelView operand() const {
        return SplitPanelView{w_.vhi.as<__half>(), vlo_, k_.n, s_, ld_, k_.world, k_.group_rows, slice_elems_};
    }
    float* partial() const { return w_.partial.as<float>(); }
    float* partial2() const { return w_.partial2.as<float>(); }
    const StreamKPlan& plan() const { return plan_; }
    const StreamKPlan& plan2() const { return plan2_; }
    bool split() const { return split_; }
    int64_t rows() const { return rows_; }

    // block product of the current pass into the partials (split / matrix-free paths)
    void product() {
        NvtxRange nvtx("block product");
        if (k_done_ >= max_passes_) fail(kInternal, "panel session pass budget exceeded");
        const SplitPanelView v = operand();
        for (int w = 0; w < (split_ ? 2 : 1); ++w) {
            const StreamKPlan& pl = w == 0 ? plan_ : plan2_;
            float* part = w == 0 ? w_.partial.as<float>() : w_.partial2.as<float>();
            if (w == 1) ctx_.main_after_comm();  // the other ranks' operand chunks have landed
            // fraction of the pass's columns in this window (algorithmic accounting)
            const double frac = split_ ? static_cast<double>(w == 0 ? rows_ : k_.n - rows_) / k_.n : 1.0;
            ctx_.prof_begin();
            if (mf_) {
                MfMatrixView a{k_.xb.as<__nv_bfloat16>(), k_.xa.as<__nv_bfloat16>(), k_.n, round_up(k_.n, 128), k_.dp,
                               k_.row0, k_.c2};
                if (rows_ > 0 && pl.k_tiles > 0)
                    launched(ctx_, launch_block_av_mf(a, v, pl, part, ctx_.stream()), "block_av_mf");
                ctx_.prof_end();
                // algorithmic flops (SURVEY §8d matrix-free): 2·n_local·n·(d + s); bytes: X, V, Y
                ctx_.prof_account(frac * (2.0 * k_.n * k_.dfeat + 2.0 * k_.n * s_) + 4.0 * rows_ * s_,
                                  frac * 2.0 * rows_ * k_.n * (k_.dfeat + s_));
            } else if (symv_) {
                SplitMatrixView a{k_.hi.as<__half>(), k_.lo.as<__half>(), rows_, k_.n, k_.ld};
                launched(ctx_, launch_symv_split(a, v.v, v.vlo, part, pl.grid, ctx_.stream()), "symv");
                ctx_.prof_end();
                // algorithmic bytes of the symmetric product: the upper triangle of A (4 B/entry) + x + y
                const double nn = static_cast<double>(k_.n);
                ctx_.prof_account(4.0 * nn * (nn + 1.0) / 2.0 + (vlo_ ? 4.0 : 2.0) * nn + 4.0 * nn, 2.0 * nn * nn);
                continue;
            } else {
                SplitMatrixView a{k_.hi.as<__half>(), k_.lo.as<__half>(), rows_, k_.n, k_.ld};
                if (rows_ > 0 && pl.k_tiles > 0)
                    launched(ctx_, launch_block_av_tc(a, v, pl, part, ctx_.stream()), "block_av_tc");
                ctx_.prof_end();
                // algorithmic bytes: A (4 B/entry) + V planes (4 B) + Y (4 B)
                ctx_.prof_account(frac * (4.0 * rows_ * k_.n + (vlo_ ? 4.0 : 2.0) * k_.n * s_) + 4.0 * rows_ * s_,
                                  frac * 2.0 * rows_ * k_.n * s_);
            }
        }
    }

    // pass epilogue over the partials the product left: T_new = a1·(A T) + a2·T + a3·T_prev, next planes
    void finish(double a1, double a2, double a3, double acc_coef) {
        NvtxRange nvtx("pass epilogue");
        if (k_done_ >= max_passes_) fail(kInternal, "panel session pass budget exceeded");
        const int k = k_done_;
        const size_t s = static_cast<size_t>(s_);
        {
            EpiArgs<float, float> e{};
            e.partial = w_.partial.as<float>();
            e.npad = npad_;
            e.total_iters = plan_.total_iters, e.k_tiles = plan_.k_tiles, e.grid = plan_.grid;
            e.cluster = plan_.cluster;
            e.dp_blocks = plan_.dp_blocks;
            e.symv_nb = symv_ ? nb_ : 0;
            e.rows = rows_, e.rows_per_block = plan_.rows_per_block, e.s = s_, e.ld = ld_;
            e.e_cur = w_.eexp.as<int>() + k * s;
            e.e_next = w_.eexp.as<int>() + (k + 1) * s;
            e.unscale = k_.unscale;
            e.cmax_cur = w_.cmax.as<unsigned>() + k * s;
            e.cmax_prev = k > 0 ? w_.cmax.as<unsigned>() + (k - 1) * s : nullptr;
            e.cmax_new = w_.cmax.as<unsigned>() + (k + 1) * s;
            e.a1 = a1, e.a2 = a2, e.a3 = a3, e.a_norm = k_.a_norm, e.gscale = gscale_;
            e.t_cur = buf<float>(k);
            e.t_prev = k > 0 ? buf<float>(k - 1) : nullptr;
            e.t_new = buf<float>(k + 1);
            e.x0 = buf<float>(0);
            e.vop = w_.vhi.as<__half>() + slice_;
            e.vop_lo = vlo_ ? vlo_ + slice_ : nullptr;
            e.stats = w_.stats.as<double>() + static_cast<size_t>(k + 1) * 3 * R_ * s;
            e.acc = acc_, e.acc_coef = acc_coef;
            if (split_) {
                e.partial2 = w_.partial2.as<float>();
                e.total_iters2 = plan2_.total_iters, e.k_tiles2 = plan2_.k_tiles, e.grid2 = plan2_.grid;
                e.dp_blocks2 = plan2_.dp_blocks;
            }
            if (rows_ > 0) launched(ctx_, launch_epilogue_split(e, ctx_.stream()), "epilogue");
            // the last pass of the budget has no successor: no all-gather (its maxima are not read)
            if (ctx_.exchange && k + 1 < max_passes_) gather_planes(k + 1);
        }
        ++k_done_;
    }

    void step_f64(double a1, double a2, double a3, double acc_coef) {
        if (k_done_ >= max_passes_) fail(kInternal, "panel session pass budget exceeded");
        const int k = k_done_;
        const size_t s = static_cast<size_t>(s_);
        {
            ctx_.prof_begin();
            launched(ctx_,
                     launch_block_av_f64(k_.a64.as<double>(), rows_, k_.n, k_.ld, buf<double>(k), s_, ld_, plan_,
                                         w_.partial.as<double>(), ctx_.stream()),
                     "block_av_f64");
            ctx_.prof_end();
            ctx_.prof_account(8.0 * rows_ * k_.n + 8.0 * k_.n * s_ + 8.0 * rows_ * s_, 2.0 * rows_ * k_.n * s_);
            EpiArgs<double, double> e{};
            e.partial = w_.partial.as<double>();
            e.npad = npad_;
            e.total_iters = plan_.total_iters, e.k_tiles = plan_.k_tiles, e.grid = plan_.grid;
            e.cluster = plan_.cluster;
            e.dp_blocks = plan_.dp_blocks;
            e.rows = rows_, e.rows_per_block = plan_.rows_per_block, e.s = s_, e.ld = ld_;
            e.unscale = 1.0;
            e.cmax_cur = w_.cmax.as<unsigned>() + k * s;
            e.cmax_prev = k > 0 ? w_.cmax.as<unsigned>() + (k - 1) * s : nullptr;
            e.cmax_new = w_.cmax.as<unsigned>() + (k + 1) * s;
            e.a1 = a1, e.a2 = a2, e.a3 = a3, e.a_norm = k_.a_norm, e.gscale = gscale_;
            e.t_cur = buf<double>(k);
            e.t_prev = k > 0 ? buf<double>(k - 1) : nullptr;
            e.t_new = buf<double>(k + 1);
            e.x0 = buf<double>(0);
            e.stats = w_.stats.as<double>() + static_cast<size_t>(k + 1) * 3 * R_ * s;
            e.acc = acc_, e.acc_coef = acc_coef;
            launched(ctx_, launch_epilogue_f64(e, ctx_.stream()), "epilogue");
        }
        ++k_done_;
    }

    // dots for passes [p0, p1] (inclusive), [p][3][s]; synchronizes
    std::vector<double> dots(int p0, int p1) {
        NvtxRange nvtx("trace partials (reduce, all-reduce, read back)");
        const int np = p1 - p0 + 1;
        const size_t s = static_cast<size_t>(s_);
        if (R_ > 0) {
            launched(ctx_,
                     launch_reduce_stats(w_.stats.as<double>() + static_cast<size_t>(p0) * 3 * R_ * s, np, R_, s_,
                                         w_.red.as<double>(), ctx_.stream()),
                     "reduce_stats");
        } else {
            cuda_check(cudaMemsetAsync(w_.red.as<double>(), 0, np * 3 * s * sizeof(double), ctx_.stream()),
                       "memset");
        }
        // row-separable trace partials: one sum over ranks
        if (ctx_.exchange) ctx_.exchange->allreduce_sum_f64(w_.red.as<double>(), np * 3 * s, ctx_.stream());
        std::vector<double> out(static_cast<size_t>(np) * 3 * s);
        d2h(ctx_, out.data(), w_.red.as<double>(), out.size() * sizeof(double));
        int err = 0;
        d2h(ctx_, &err, ctx_.probe_err.as<int>(), sizeof(int));
        ctx_.sync();
        check_probe_err(ctx_, err);
        return out;
    }

    // dots of groups g = 0..groups-1 of a grouped stack (rg row blocks each; single rank), one device
    // round trip: [g][p][3][s]
    std::vector<double> dots_groups(int p0, int p1, int groups, int rg) {
        const int np = p1 - p0 + 1;
        const size_t s = static_cast<size_t>(s_), per = static_cast<size_t>(np) * 3 * s;
        w_.red.ensure(groups * per * sizeof(double));
        for (int g = 0; g < groups; ++g)
            launched(ctx_,
                     launch_reduce_stats(w_.stats.as<double>() + static_cast<size_t>(p0) * 3 * R_ * s, np, R_, s_,
                                         w_.red.as<double>() + g * per, ctx_.stream(), g * rg, rg),
                     "reduce_stats");
        std::vector<double> out(groups * per);
        d2h(ctx_, out.data(), w_.red.as<double>(), out.size() * sizeof(double));
        int err = 0;
        d2h(ctx_, &err, ctx_.probe_err.as<int>(), sizeof(int));
        ctx_.sync();
        check_probe_err(ctx_, err);
        return out;
    }
    int rows_per_block() const { return plan_.rows_per_block; }

    // the epilogue's a1, a2, a3 are multiplied by *g (device) from here on
    void set_gscale(const double* g) { gscale_ = g; }

    // the dots of pass p (single rank) into dst (device, [3][s]); no synchronize
    void reduce_pass(int p, double* dst) {
        if (R_ > 0)
            launched(ctx_,
                     launch_reduce_stats(w_.stats.as<double>() + static_cast<size_t>(p) * 3 * R_ * s_, 1, R_, s_, dst,
                                         ctx_.stream()),
                     "reduce_stats");
        else
            cuda_check(cudaMemsetAsync(dst, 0, 3 * static_cast<size_t>(s_) * sizeof(double), ctx_.stream()), "memset");
    }

    void state_f64(int k, double* out, int64_t ldo) {
        const bool f32 = k_.prec != kF64;
        launched(ctx_,
                 launch_state_to_f64(f32 ? static_cast<const void*>(buf<float>(k))
                                         : static_cast<const void*>(buf<double>(k)),
                                     f32, rows_, s_, ld_, out, ldo, ctx_.stream()),
                 "state_to_f64");
    }

    int passes() const { return k_done_; }
    int64_t ld() const { return ld_; }

private:
    template <typename T>
    T* buf(int k) const {
        if (k == 0) return w_.state[0].as<T>();
        return w_.state[1 + (k - 1) % 3].as<T>();
    }

    Context& ctx_;
    PanelWorkspace& w_;
    const KernelMatrix& k_;
    int s_;
    int max_passes_;
    double* acc_;
    int64_t rows_ = 0, ld_ = 0;
    int R_ = 0;
    int npad_ = 0;
    int k_done_ = 0;
    bool mf_ = false;
    __half* vlo_ = nullptr;
    size_t slice_ = 0;  // this rank's chunk offset in the operand planes
    int64_t slice_elems_ = 0;  // elements per rank chunk (s·rpr + the column-maxima tail when sharded)
    static constexpr int64_t kTailElems = 256;  // 512 bytes: up to 128 uint32 column maxima
    StreamKPlan plan_, plan2_;
    bool split_ = false;
    bool symv_ = false;  // s = 1 through the upper-triangle product (symv.cu)
    const double* gscale_ = nullptr;
    int64_t nb_ = 0;     // its 128-row blocks
};

}  // namespace

PanelResult run_panel(Context& ctx, const KernelMatrix& k, const double* x, int64_t ldx, int s,
                      const std::vector<std::array<double, 3>>& coeffs, const std::vector<double>* acc_coef,
                      double* acc_out, double* last_out, int64_t ldo) {
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    const int P = static_cast<int>(coeffs.size());
    PanelSession ps(ctx, k, x, ldx, s, std::max(P, 1), acc_out, acc_coef ? (*acc_coef)[0] : 0.0,
                    acc_out != nullptr || last_out != nullptr);
    for (int p = 0; p < P; ++p)
        ps.step(coeffs[p][0], coeffs[p][1], coeffs[p][2], acc_coef ? (*acc_coef)[p + 1] : 0.0);
    if (last_out) ps.state_f64(P, last_out, ldo);
    PanelResult r;
    r.passes = P;
    r.s = s;
    r.dots = ps.dots(0, P);
    return r;
}

namespace {

std::vector<std::array<double, 3>> schedule(const MatFun& f) {
    std::vector<std::array<double, 3>> c(f.degree);
    for (int k = 0; k < f.degree; ++k) f.pass_coeffs(k, &c[k][0], &c[k][1], &c[k][2]);
    return c;
}

// upload a host column-major panel (n x s) into a device fp64 buffer [s][ld]
void upload_panel(Context& ctx, DevBuf& dst, const double* host, int64_t n, int s, int64_t ld) {
    dst.ensure(static_cast<size_t>(s) * ld * sizeof(double));
    h2d_2d(ctx, dst.as<double>(), ld * sizeof(double), host, n * sizeof(double), n * sizeof(double), s);
}

void download_panel(Context& ctx, const double* dev, int64_t ld, int64_t n, int s, double* host) {
    d2h_2d(ctx, host, n * sizeof(double), dev, ld * sizeof(double), n * sizeof(double), s);
    ctx.sync();
}

void require_single_rank(Context& ctx, const char* what) {
    if (ctx.exchange && ctx.exchange->world() > 1)
        fail(kInvalidArgument, std::string(what) + " is a single-rank parity seam");
}

}  // namespace

void block_product(Context& ctx, const KernelMatrix& k, const double* v, int s, double* y) {
    require_single_rank(ctx, "matmul_panel");
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    const int64_t n = k.n, ld = round_up(n, 8);
    for (int j0 = 0; j0 < s; j0 += kMaxPanelCols) {
        const int w = std::min(kMaxPanelCols, s - j0);
        upload_panel(ctx, ctx.x0, v + j0 * n, n, w, ld);
        ctx.work.ensure(static_cast<size_t>(w) * ld * sizeof(double));
        run_panel(ctx, k, ctx.x0.as<double>(), ld, w, {{1.0, 0.0, 0.0}}, nullptr, nullptr, ctx.work.as<double>(),
                  ld);
        download_panel(ctx, ctx.work.as<double>(), ld, n, w, y + j0 * n);
    }
}

void apply_panel(Context& ctx, const KernelMatrix& k, const MatFun& f, const double* v, int s, double* y) {
    require_single_rank(ctx, "apply_panel");
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    const int64_t n = k.n, ld = round_up(n, 8);
    std::vector<double> coef(f.degree + 1, 0.0);
    double post = 1.0;
    if (f.kind == kTaylor) {
        for (int i = 0; i <= f.degree; ++i) coef[i] = f.coeffs[i];
        post = std::pow(f.v, f.alpha);
    } else if (f.kind == kChebyshev) {
        coef[0] = 0.5 * f.coeffs[0];
        for (int i = 1; i <= f.degree; ++i) coef[i] = f.coeffs[i];
    }
    for (int j0 = 0; j0 < s; j0 += kMaxPanelCols) {
        const int w = std::min(kMaxPanelCols, s - j0);
        upload_panel(ctx, ctx.x0, v + j0 * n, n, w, ld);
        // the vector accumulator shares the state layout [s][rpr]
        ctx.acc.ensure(static_cast<size_t>(w) * k.rpr * sizeof(double));
        if (f.kind == kIntPower) {
            run_panel(ctx, k, ctx.x0.as<double>(), ld, w, schedule(f), nullptr, nullptr, ctx.acc.as<double>(),
                      k.rpr);
        } else {
            run_panel(ctx, k, ctx.x0.as<double>(), ld, w, schedule(f), &coef, ctx.acc.as<double>(), nullptr, 0);
        }
        download_panel(ctx, ctx.acc.as<double>(), k.rpr, n, w, y + j0 * n);
        if (post != 1.0)
            for (int64_t i = 0; i < n * w; ++i) y[j0 * n + i] *= post;
    }
}

namespace {

// Moments mu_p = x^T P_p(A) x, p = 0..degree, of column j from ceil(degree/2) passes (moment doubling).
// A is symmetric, so with t_k = P_k(A) x:
//   power / Taylor (P_k = M^k, M = A or A/v - I):  mu_2k = t_k.t_k,   mu_2k+1 = t_k.t_k+1
//   Chebyshev (T_m T_n = (T_m+n + T_|m-n|)/2):     mu_2k = 2 t_k.t_k - mu_0,   mu_2k+1 = 2 t_k.t_k+1 - mu_1
// The pass epilogue already reduces x0.t_k+1, t_k.t_k+1 and t_k+1.t_k+1 in fp64 (dots q = 0, 1, 2).
void doubled_moments(const MatFun& f, const PanelResult& r, int j, double* mu) {
    const int m = f.degree;
    const double mu0 = r.dot(0, 0, j);
    mu[0] = mu0;
    if (f.kind == kChebyshev) {
        const double mu1 = m >= 1 ? r.dot(1, 0, j) : 0.0;
        if (m >= 1) mu[1] = mu1;
        for (int p = 2; p <= m; ++p) {
            const int k = p / 2;
            mu[p] = (p % 2 == 0) ? 2.0 * r.dot(k, 2, j) - mu0 : 2.0 * r.dot(k + 1, 1, j) - mu1;
        }
    } else {
        for (int p = 1; p <= m; ++p) {
            const int k = p / 2;
            mu[p] = (p % 2 == 0) ? r.dot(k, 2, j) : r.dot(k + 1, 1, j);
        }
    }
}

// per-column traces x_j^T f(A) x_j for a device panel [s][ldx], in groups of <= 128 columns. The
// reference applies f(A) with `degree` sequential products (proj/src/poly.cpp:97-134) and then takes
// x.f(A)x (hutchpp.cpp:33-51); the same quadratic forms come from half the passes over A by moment
// doubling (doubled_moments), which is where the trace-only estimators spend their time.
std::vector<double> panel_traces(Context& ctx, const KernelMatrix& k, const MatFun& f, const double* x, int64_t ldx,
                                 int s) {
    std::vector<double> tr(s, 0.0);
    const auto full = schedule(f);
    const int passes = (f.degree + 1) / 2;
    const std::vector<std::array<double, 3>> sched(full.begin(), full.begin() + passes);
    for (int j0 = 0; j0 < s; j0 += kMaxPanelCols) {
        const int w = std::min(kMaxPanelCols, s - j0);
        PanelResult r = run_panel(ctx, k, x + static_cast<int64_t>(j0) * ldx, ldx, w, sched);
        std::vector<double> mu(f.degree + 1);
        for (int j = 0; j < w; ++j) {
            doubled_moments(f, r, j, mu.data());
            tr[j0 + j] = f.combine(mu.data(), 1);
        }
    }
    return tr;
}

}  // namespace

void matfun_traces(Context& ctx, const KernelMatrix& k, const MatFun& f, const double* x, int s, double* out) {
    require_single_rank(ctx, "matfun_traces");
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    const int64_t n = k.n, ld = k.rpr;
    DevBuf xs;
    upload_panel(ctx, xs, x, n, s, ld);
    std::vector<double> tr = panel_traces(ctx, k, f, xs.as<double>(), ld, s);
    std::copy(tr.begin(), tr.end(), out);
}

// ---------------------------------------------------------------- spectrum
PowerRes power_method(Context& ctx, const KernelMatrix& k, const PowerOpts& o, double shift) {
    NvtxRange nvtx("power iteration");
    // proj/src/spectrum.cpp:13-49; shift > 0 runs on (shift·I − A) without forming it
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    const int64_t ld = k.rpr;  // local rows of the start vector (row-sharded: counters from row0)
    ctx.x0.ensure(static_cast<size_t>(ld) * sizeof(double));
    const uint64_t key = derive_key(o.seed, hash_name("power-start"));
    if (ctx.probe_source == 1) {  // seeded_start (spectrum.cpp:13-21) with the reference's own draws
        std::vector<double> v(static_cast<size_t>(k.n));
        RandomStream rs(key);
        for (double& e : v) e = rs.next_gaussian();
        h2d(ctx, ctx.x0.as<double>(), v.data() + k.row0, static_cast<size_t>(k.rows) * sizeof(double));
        ctx.sync();  // v is pageable host memory owned by this frame
    } else {
        launched(ctx,
                 launch_rng_panel(key, false, kProbeGaussian, k.row0, k.rows, 1, 0, ctx.x0.as<double>(), ld,
                                  ctx.probe_err.as<int>(), ctx.stream()),
                 "rng_panel");
    }
    PowerRes res;
    const int iters = std::max(o.max_iters, 0);
    PanelSession ps(ctx, k, ctx.x0.as<double>(), ld, 1, std::max(iters, 1), nullptr, 0.0, false);
    std::vector<double> d0 = ps.dots(0, 0);
    double norm = std::sqrt(d0[2]);
    if (norm == 0.0) fail(kInternal, "power-start vector is zero");
    double g = 1.0 / norm;  // x = T/||T||
    double prev = 0.0;
    if (ctx.speculate && ctx.world() == 1 && iters > 0) {
        // Pass it+1 is queued before the host reads pass it's dots: its normalisation g = 1/||T_it|| is
        // computed on the device (launch_power_norm, the same IEEE sqrt and division as the host's) and
        // scales the epilogue's coefficients, so every pass is bitwise the one the synchronous loop
        // below runs; the host's readback and convergence test overlap the next product, and the pass
        // queued past convergence is discarded.
        DevBuf dd;
        dd.alloc(sizeof(double) * (3 * static_cast<size_t>(iters + 1) + 1));
        double* red = dd.as<double>();
        double* gdev = red + 3 * static_cast<size_t>(iters + 1);
        double* pin = ctx.pinned_dots(3 * static_cast<size_t>(iters + 1));
        ps.reduce_pass(0, red);
        launched(ctx, launch_power_norm(red, gdev, ctx.stream()), "power_norm");
        ps.set_gscale(gdev);
        auto enqueue = [&](int p) {
            if (shift != 0.0)
                ps.step(-1.0, shift, 0.0, 0.0);  // (-1)·g = -g, shift·g: the coefficients below
            else
                ps.step(1.0, 0.0, 0.0, 0.0);
            double* rp = red + 3 * static_cast<size_t>(p);
            ps.reduce_pass(p, rp);
            launched(ctx, launch_power_norm(rp, gdev, ctx.stream()), "power_norm");
            cuda_check(cudaMemcpyAsync(pin + 3 * static_cast<size_t>(p), rp, 3 * sizeof(double),
                                       cudaMemcpyDeviceToHost, ctx.stream()),
                       "device->host copy");
            ctx.d2h_bytes += 3 * sizeof(double);
            cuda_check(cudaEventRecord(ctx.dots_event(p & 1), ctx.stream()), "cudaEventRecord");
        };
        enqueue(1);
        for (int it = 1; it <= iters; ++it) {
            if (it < iters) enqueue(it + 1);
            cuda_check(cudaEventSynchronize(ctx.dots_event(it & 1)), "power iteration dots");
            const double* d = pin + 3 * static_cast<size_t>(it);
            const double quotient = g * d[1];
            res.rayleigh = quotient;
            res.iterations = it;
            if (it > 1 && std::abs(quotient - prev) <= o.tol * std::abs(quotient)) {
                res.converged = true;
                break;
            }
            prev = quotient;
            const double ny = std::sqrt(d[2]);
            if (ny == 0.0) {
                res.converged = true;
                break;
            }
            g = 1.0 / ny;
        }
        return res;
    }
    for (int it = 1; it <= iters; ++it) {
        if (shift != 0.0)
            ps.step(-g, shift * g, 0.0, 0.0);
        else
            ps.step(g, 0.0, 0.0, 0.0);
        std::vector<double> d = ps.dots(it, it);
        const double quotient = g * d[1];
        res.rayleigh = quotient;
        res.iterations = it;
        if (it > 1 && std::abs(quotient - prev) <= o.tol * std::abs(quotient)) {
            res.converged = true;
            break;
        }
        prev = quotient;
        const double ny = std::sqrt(d[2]);
        if (ny == 0.0) {
            res.converged = true;
            break;
        }
        g = 1.0 / ny;
    }
    return res;
}

SpectrumBoundsH estimate_bounds(Context& ctx, const KernelMatrix& k, const PowerOpts& o) {
    // proj/src/spectrum.cpp:80-103
    SpectrumBoundsH b;
    const PowerRes rv = power_method(ctx, k, o, 0.0);
    const double inv_n = 1.0 / static_cast<double>(k.n);
    b.v = std::clamp(rv.rayleigh * (1.0 + o.tol), inv_n, 1.0);
    b.v_converged = rv.converged;
    PowerOpts so = o;
    so.seed = derive_key(o.seed, hash_name("shifted"));
    const PowerRes ru = power_method(ctx, k, so, b.v);
    b.u_converged = ru.converged;
    double u = (b.v - ru.rayleigh) * (1.0 - o.tol);
    const double floor = std::max(o.rank_floor, b.v * o.tol * 100.0);
    if (u < floor) {
        u = 0.0;
        b.rank_deficient = true;
    }
    b.u = std::min(u, inv_n);
    b.kappa = b.u > 0.0 ? b.v / b.u : std::numeric_limits<double>::infinity();
    b.iterations_used = rv.iterations + ru.iterations;
    return b;
}

// ---------------------------------------------------------------- Hutch++
namespace {

// fp64 probe panel on the device [cols][ld]: injected host panel or the reference stream
void make_probes(Context& ctx, const KernelMatrix& k, DevBuf& dst, int cols, int64_t ld, const double* host,
                 uint64_t seed, const char* label, int kind) {
    // this rank's rows [row0, row0 + rows) of the n x cols probe panel
    dst.ensure(static_cast<size_t>(cols) * ld * sizeof(double));
    if (host) {
        h2d_2d(ctx, dst.as<double>(), ld * sizeof(double), host + k.row0, k.n * sizeof(double),
               k.rows * sizeof(double), cols);
        return;
    }
    if (ctx.probe_source == 1 && kind == kProbeGaussian) {  // the reference's draws, bitwise (host threads)
        const auto v = ctx.take_probes(k.n, cols, seed, label, kind);
        h2d_2d(ctx, dst.as<double>(), ld * sizeof(double), v->data() + k.row0, k.n * sizeof(double),
               k.rows * sizeof(double), cols);
        ctx.sync();  // v is pageable host memory owned by this frame
        return;
    }
    // no round trip here: a (p = 2^-53) Box-Muller redraw raises ctx.probe_err, which every pass
    // session reads back with its trace partials (check_probe_err) before any result leaves
    launched(ctx,
             launch_rng_panel(derive_key(seed, hash_name(label)), true, kind, k.row0, k.rows, cols, 0,
                              dst.as<double>(), ld, ctx.probe_err.as<int>(), ctx.stream()),
             "rng_panel");
}

std::vector<double> gram_host(Context& ctx, const double* x, int p, int64_t ldx, const double* z, int q,
                              int64_t ldz, int64_t rows) {
    std::vector<double> out(static_cast<size_t>(p) * q);
    if (p > 128) {  // wide sketches (s/4 > 128 columns): row blocks of X^T Z, assembled on the host
        for (int p0 = 0; p0 < p; p0 += 128) {
            const int pb = std::min(128, p - p0);
            const std::vector<double> sub = gram_host(ctx, x + static_cast<int64_t>(p0) * ldx, pb, ldx, z, q, ldz, rows);
            for (int c = 0; c < q; ++c)
                for (int r = 0; r < pb; ++r) out[(p0 + r) + static_cast<size_t>(c) * p] = sub[r + static_cast<size_t>(c) * pb];
        }
        return out;
    }
    const int grid = std::min<int64_t>(ctx.sms(), std::max<int64_t>(1, (rows + 31) / 32));
    // column blocks of z so p * qb <= 2048 and the kernel's 32-row staging of p + qb columns (plus its
    // static shared flag) fits the 48 KB default
    const int qb_max = std::max(1, std::min(2048 / std::max(p, 1), 190 - p));
    ctx.small.ensure(static_cast<size_t>(p) * q * sizeof(double));
    for (int b0 = 0; b0 < q; b0 += qb_max) {
        const int qb = std::min(qb_max, q - b0);
        ctx.gram_partial.ensure(static_cast<size_t>(grid) * p * qb * sizeof(double));
        launched(ctx,
                 launch_panel_gram(x, p, ldx, z + static_cast<int64_t>(b0) * ldz, qb, ldz, rows,
                                   ctx.gram_partial.as<double>(), grid, ctx.small.as<double>() + static_cast<size_t>(b0) * p,
                                   ctx.stream(), ctx.gram_ticket.as<unsigned>()),
                 "panel_gram");
    }
    // Grams over row-sharded panels: one sum over ranks (CholeskyQR2 / projection)
    if (ctx.exchange) ctx.exchange->allreduce_sum_f64(ctx.small.as<double>(), out.size(), ctx.stream());
    d2h(ctx, out.data(), ctx.small.as<double>(), out.size() * sizeof(double));
    ctx.sync();
    return out;
}

// W = beta*G + X*C on the device; C is a host p x q column-major matrix
void update(Context& ctx, double beta, const double* g, int64_t ldg, const double* x, int p, int64_t ldx,
            const std::vector<double>& c, int q, int64_t rows, double* w, int64_t ldw) {
    DevBuf cd;
    cd.alloc(c.size() * sizeof(double));
    h2d(ctx, cd.as<double>(), c.data(), c.size() * sizeof(double));
    // smem limit: split q
    const int qb_max = std::max(1, (48 * 1024 / 8) / std::max(p, 1));
    for (int b0 = 0; b0 < q; b0 += qb_max) {
        const int qb = std::min(qb_max, q - b0);
        launched(ctx,
                 launch_panel_update(beta, g ? g + static_cast<int64_t>(b0) * ldg : nullptr, ldg, x, p, ldx,
                                     cd.as<double>() + static_cast<size_t>(b0) * p, qb, rows,
                                     w + static_cast<int64_t>(b0) * ldw, ldw, ctx.stream()),
                 "panel_update");
    }
    ctx.sync();
}

// Orthonormal basis of range(Y) (Y device [p][ld], n rows) by CholeskyQR2 with an eigen-based,
// rank-revealing first step, plus one residual pass; returns the rank and writes Q [rank][ld].
// Replaces Eigen::ColPivHouseholderQR + setThreshold(1e-12) (proj/src/hutchpp.cpp:91-108):
// tr(Q^T f Q) and I - QQ^T are basis-invariant, so only the kept subspace matters. The Gram's
// eigenvalues resolve singular values only down to ~1e-7 of the largest, so the directions
// between 1e-12 and 1e-7 (fast-decaying spectra, e.g. 1-D feature kernels) are recovered from
// the residual Y - Q Q^T Y, whose own Gram resolves them; the kept set is then
// { sigma_i > 1e-12 sigma_0 }, the reference's rank rule stated on singular values.
int orthonormal_range(Context& ctx, const double* y, int p, int64_t ld, int64_t n, DevBuf& q_out) {
    std::vector<double> g = gram_host(ctx, y, p, ld, y, p, ld, n);
    std::vector<double> w, v;
    sym_eig_desc(p, g, w, v);
    if (!(w.size() > 0 && w[0] > 0.0)) return 0;
    const double w0 = w[0];
    int k = 0;
    while (k < p && w[k] > 1e-13 * w0) ++k;
    if (k == 0) return 0;
    // orthonormalise X·M with CholeskyQR (eigen fallback), X [cols][ld]
    auto chol_qr = [&](const double* x, int cols, double* out) {
        std::vector<double> g2 = gram_host(ctx, x, cols, ld, x, cols, ld, n);
        std::vector<double> r2;
        if (cholesky_upper(cols, g2, r2)) {
            update(ctx, 0.0, nullptr, ld, x, cols, ld, upper_inverse(cols, r2), cols, n, out, ld);
        } else {
            std::vector<double> w2, v2;
            sym_eig_desc(cols, g2, w2, v2);
            std::vector<double> m2(static_cast<size_t>(cols) * cols);
            for (int c = 0; c < cols; ++c)
                for (int r = 0; r < cols; ++r)
                    m2[r + static_cast<size_t>(c) * cols] = v2[r + static_cast<size_t>(c) * cols] / std::sqrt(w2[c]);
            update(ctx, 0.0, nullptr, ld, x, cols, ld, m2, cols, n, out, ld);
        }
    };
    auto scaled_vectors = [&](const std::vector<double>& ww, const std::vector<double>& vv, int cols) {
        std::vector<double> m(static_cast<size_t>(p) * cols);
        for (int c = 0; c < cols; ++c) {
            const double sc = 1.0 / std::sqrt(ww[c]);
            for (int r = 0; r < p; ++r) m[r + static_cast<size_t>(c) * p] = vv[r + static_cast<size_t>(c) * p] * sc;
        }
        return m;
    };
    DevBuf q1, qa;
    q1.alloc(static_cast<size_t>(p) * ld * sizeof(double));
    qa.alloc(static_cast<size_t>(p) * ld * sizeof(double));
    update(ctx, 0.0, nullptr, ld, y, p, ld, scaled_vectors(w, v, k), k, n, q1.as<double>(), ld);
    chol_qr(q1.as<double>(), k, qa.as<double>());  // second pass: orthogonal to working precision
    int rank = k;
    if (k < p) {
        // residual pass: Y2 = Y - Q (Q^T Y); keep sigma(Y2) > 1e-12 sigma_0(Y)
        std::vector<double> c = gram_host(ctx, qa.as<double>(), k, ld, y, p, ld, n);
        for (double& x : c) x = -x;
        DevBuf y2;
        y2.alloc(static_cast<size_t>(p) * ld * sizeof(double));
        update(ctx, 1.0, y, ld, qa.as<double>(), k, ld, c, p, n, y2.as<double>(), ld);
        std::vector<double> g2 = gram_host(ctx, y2.as<double>(), p, ld, y2.as<double>(), p, ld, n);
        std::vector<double> w2, v2;
        sym_eig_desc(p, g2, w2, v2);
        int k2 = 0;
        while (k2 < p - k && w2[k2] > 1e-24 * w0) ++k2;
        if (k2 > 0) {
            double* dst = qa.as<double>() + static_cast<int64_t>(k) * ld;
            update(ctx, 0.0, nullptr, ld, y2.as<double>(), p, ld, scaled_vectors(w2, v2, k2), k2, n, q1.as<double>(),
                   ld);
            // re-orthogonalise against the first block, then CholeskyQR
            std::vector<double> c2 = gram_host(ctx, qa.as<double>(), k, ld, q1.as<double>(), k2, ld, n);
            for (double& x : c2) x = -x;
            update(ctx, 1.0, q1.as<double>(), ld, qa.as<double>(), k, ld, c2, k2, n, y2.as<double>(), ld);
            chol_qr(y2.as<double>(), k2, dst);
            rank += k2;
        }
    }
    q_out.ensure(static_cast<size_t>(rank) * ld * sizeof(double));
    cuda_check(cudaMemcpyAsync(q_out.as<double>(), qa.as<double>(), static_cast<size_t>(rank) * ld * sizeof(double),
                               cudaMemcpyDeviceToDevice, ctx.stream()),
               "copy Q");
    return rank;
}

double exact_trace(Context& ctx, const KernelMatrix& k, const MatFun& f) {
    // proj/src/hutchpp.cpp:53-65: identity panels (single rank)
    const int64_t n = k.n, ld = k.rpr;
    double sum = 0.0;
    DevBuf eye;
    for (int64_t j0 = 0; j0 < n; j0 += kMaxPanelCols) {
        const int w = static_cast<int>(std::min<int64_t>(kMaxPanelCols, n - j0));
        std::vector<double> h(static_cast<size_t>(n) * w, 0.0);
        for (int j = 0; j < w; ++j) h[(j0 + j) + static_cast<size_t>(j) * n] = 1.0;
        upload_panel(ctx, eye, h.data(), n, w, ld);
        std::vector<double> tr = panel_traces(ctx, k, f, eye.as<double>(), ld, w);
        for (double t : tr) sum += t;
    }
    return sum;
}

}  // namespace

TraceEst hutchpp(Context& ctx, const KernelMatrix& k, const MatFun& f, const SketchCfg& cfg) {
    NvtxRange nvtx("hutchpp");
    // proj/src/hutchpp.cpp:69-115, with probe injection / explicit split / Q-empty Hutchinson.
    // Row-sharded: every panel below holds this rank's rows; Grams are summed over ranks.
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    const int64_t n = k.n, ld = k.rpr, rows = k.rows;
    const bool single = ctx.world() == 1;
    const int s_q = cfg.s_q, s_g = cfg.s_g;
    const int cost = f.query_cost();
    if (s_q < 0 || s_g < 0 || s_q + s_g < 1) fail(kInvalidArgument, "hutchpp needs a positive query budget");
    TraceEst est;
    if (s_q >= n) {
        if (!single) fail(kInvalidArgument, "the exact-degeneration branch (s/4 >= n) is single-rank");
        est.value = est.low_rank_part = exact_trace(ctx, k, f);
        est.residual_part = 0.0;
        est.sketch_rank = static_cast<int>(n);
        est.queries_used = static_cast<int>(n) * cost;
        est.exact = true;
        return est;
    }
    DevBuf qbuf;
    int rank = 0;
    if (s_q > 0) {
        DevBuf sk;
        make_probes(ctx, k, sk, s_q, ld, cfg.sketch, cfg.seed, "hutchpp-sketch", cfg.probe_kind);
        DevBuf y;
        y.alloc(static_cast<size_t>(s_q) * ld * sizeof(double));
        for (int j0 = 0; j0 < s_q; j0 += kMaxPanelCols) {
            const int w = std::min(kMaxPanelCols, s_q - j0);
            run_panel(ctx, k, sk.as<double>() + j0 * ld, ld, w, {{1.0, 0.0, 0.0}}, nullptr, nullptr,
                      y.as<double>() + j0 * ld, ld);
        }
        rank = orthonormal_range(ctx, y.as<double>(), s_q, ld, rows, qbuf);
        if (rank == 0) fail(kRankCollapse, "hutchpp sketch A*S is numerically zero");
        est.sketch_rank = rank;
        est.queries_used = s_q + rank * cost;
    }
    const int64_t codim = n - rank;
    if (s_q > 0 && s_g >= codim) {
        // trace the complement exactly (proj/src/hutchpp.cpp:100-106)
        if (!single) fail(kInvalidArgument, "the exact-complement branch (s_g >= n - rank) is single-rank");
        std::vector<double> qh(static_cast<size_t>(n) * rank);
        download_panel(ctx, qbuf.as<double>(), ld, n, rank, qh.data());
        std::vector<double> full = complete_basis(n, rank, qh);
        DevBuf fb;
        upload_panel(ctx, fb, full.data(), n, static_cast<int>(n), ld);
        std::vector<double> tr = panel_traces(ctx, k, f, fb.as<double>(), ld, static_cast<int>(n));
        double low = 0.0, res = 0.0;
        for (int j = 0; j < rank; ++j) low += tr[j];
        for (int64_t j = rank; j < n; ++j) res += tr[j];
        est.low_rank_part = low;
        est.residual_part = res;
        est.queries_used += static_cast<int>(codim) * cost;
        est.exact = true;
    } else {
        // X0 = [Q | W],  W = G - Q (Q^T G)
        const int cols = rank + s_g;
        DevBuf x0;
        x0.alloc(static_cast<size_t>(cols) * ld * sizeof(double));
        if (rank > 0)
            cuda_check(cudaMemcpyAsync(x0.as<double>(), qbuf.as<double>(), static_cast<size_t>(rank) * ld * sizeof(double),
                                       cudaMemcpyDeviceToDevice, ctx.stream()),
                       "copy Q");
        if (s_g > 0) {
            double* wdst = x0.as<double>() + static_cast<int64_t>(rank) * ld;
            DevBuf gp;
            make_probes(ctx, k, gp, s_g, ld, cfg.probes, cfg.seed, "hutchpp-probe", cfg.probe_kind);
            if (rank > 0) {
                std::vector<double> c = gram_host(ctx, qbuf.as<double>(), rank, ld, gp.as<double>(), s_g, ld, rows);
                for (double& v : c) v = -v;
                update(ctx, 1.0, gp.as<double>(), ld, qbuf.as<double>(), rank, ld, c, s_g, rows, wdst, ld);
            } else {
                cuda_check(cudaMemcpyAsync(wdst, gp.as<double>(), static_cast<size_t>(s_g) * ld * sizeof(double),
                                           cudaMemcpyDeviceToDevice, ctx.stream()),
                           "copy probes");
            }
        }
        std::vector<double> tr = panel_traces(ctx, k, f, x0.as<double>(), ld, cols);
        double low = 0.0, res = 0.0;
        for (int j = 0; j < rank; ++j) low += tr[j];
        for (int j = rank; j < cols; ++j) res += tr[j];
        est.low_rank_part = low;
        est.residual_part = s_g > 0 ? res / s_g : 0.0;
        est.queries_used += s_g * cost;
    }
    est.value = est.low_rank_part + est.residual_part;
    return est;
}

// ---------------------------------------------------------------- estimators
namespace {

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

SketchCfg sketch_cfg(const EstParams& p, int s) {
    SketchCfg cfg;
    if (p.s_q >= 0 || p.s_g >= 0) {
        cfg.s_q = std::max(p.s_q, 0);
        cfg.s_g = std::max(p.s_g, 0);
    } else {
        if (s < 8) fail(kInvalidArgument, "hutchpp needs a query budget s >= 8");
        cfg.s_q = s / 4;
        cfg.s_g = s - 2 * (s / 4);
    }
    cfg.seed = p.seed;
    cfg.probe_kind = p.probe_kind;
    return cfg;
}

EntropyEst entropy_of(const TraceEst& tr, double alpha, int method, int s, int m_used) {
    EntropyEst est;
    est.trace = tr;
    est.trace_estimate = tr.value;
    est.entropy = entropy_from_trace(tr.value, alpha);
    est.method_used = method;
    est.s_used = s;
    est.m_used = m_used;
    est.deterministic = tr.exact;
    return est;
}

// Everything estimate() decides before the trace estimator runs (proj/src/entropy.cpp:201-275):
// routing, bounds, (s, m) selection and the matrix function. Seed-independent except for the
// bounds' power iteration, which uses derive_key(p.seed, "bounds").
struct Resolved {
    int method = kMethodInt;
    MatFun f;
    double alpha = 2.0;
    int s = 0, m_used = 0;
    bool has_bounds = false;
    SpectrumBoundsH bounds;
};

Resolved resolve(Context& ctx, const KernelMatrix& k, const EstParams& p) {
    validate_alpha(p.alpha);
    const int64_t n = k.n;
    int alpha_int = 0;
    const bool is_int = integer_alpha(p.alpha, &alpha_int);
    Resolved r;
    r.has_bounds = p.has_bounds;
    r.bounds = p.bounds;
    auto ensure_bounds = [&]() -> const SpectrumBoundsH& {
        if (!r.has_bounds) {
            PowerOpts o = p.power;
            o.seed = derive_key(p.seed, hash_name("bounds"));
            r.bounds = estimate_bounds(ctx, k, o);
            r.has_bounds = true;
        }
        return r.bounds;
    };
    int method = p.method;
    if (method == kMethodAuto) {
        if (is_int) {
            method = kMethodInt;
        } else {
            const SpectrumBoundsH& b = ensure_bounds();
            const bool flat_full_rank = b.u > 0.0 && b.kappa <= 50.0;
            const bool flat_deficient = b.u == 0.0 && b.v * static_cast<double>(n) <= 50.0;
            method = (flat_full_rank || flat_deficient) ? kMethodTaylor : kMethodChebyshev;
        }
    }
    r.method = method;
    switch (method) {
        case kMethodExact:
            fail(kInvalidArgument,
                 "method=exact is the O(n^3) eigendecomposition check oracle; it is not a device path");
        case kMethodInt: {
            if (!is_int) fail(kInvalidArgument, "method=int needs an integer alpha >= 2");
            r.s = p.s > 0 ? p.s : select_params(p.alpha, p.epsilon, p.delta, SpectrumBoundsH{}, n, kMethodInt).s;
            if (alpha_int < 2) fail(kInvalidArgument, "entropy_int needs integer alpha >= 2");
            r.f = MatFun::int_power(alpha_int);
            r.alpha = alpha_int;
            r.m_used = 0;
            break;
        }
        case kMethodTaylor:
        case kMethodChebyshev: {
            const SpectrumBoundsH& b = ensure_bounds();
            SelectedParams sel;
            if (p.s > 0 && p.m > 0) {
                sel = {p.s, p.m};
            } else {
                sel = select_params(p.alpha, p.epsilon, p.delta, b, n, method);
                if (p.s > 0) sel.s = p.s;
                if (p.m > 0) sel.m = p.m;
            }
            r.s = sel.s;
            r.alpha = p.alpha;
            if (method == kMethodTaylor) {
                require_non_integer(p.alpha, "entropy_taylor");
                const int m = std::max(sel.m, static_cast<int>(std::ceil(p.alpha)) + 1);
                r.f = MatFun::taylor(p.alpha, m, b.v);
                r.m_used = m;
            } else {
                require_non_integer(p.alpha, "entropy_chebyshev");
                r.f = MatFun::chebyshev(p.alpha, sel.m, b.u, b.v);
                r.m_used = sel.m;
            }
            break;
        }
        default:
            fail(kInvalidArgument, "unresolved auto method");
    }
    return r;
}

}  // namespace

EntropyEst estimate(Context& ctx, const KernelMatrix& k, const EstParams& p) {
    NvtxRange nvtx("estimate");
    // proj/src/entropy.cpp:201-275
    const auto t0 = std::chrono::steady_clock::now();
    const Resolved r = resolve(ctx, k, p);
    EntropyEst est = entropy_of(hutchpp(ctx, k, r.f, sketch_cfg(p, r.s)), r.alpha, r.method, r.s, r.m_used);
    est.has_bounds = r.has_bounds;
    est.bounds_used = r.bounds;
    est.elapsed = seconds_since(t0);
    return est;
}

// ---------------------------------------------------------------- batched trials
namespace {

// Hutch++ for several probe seeds at once: the sketch products and the
// f(A)·[Q_t | W_t] recurrences of all trials share the same passes over A as extra panel columns
// (up to 128 per pass), so K trials cost ~ceil(K·cols/128) passes instead of K. Each column's
// arithmetic is the same as in a single-trial run.
std::vector<TraceEst> hutchpp_batch(Context& ctx, const KernelMatrix& k, const MatFun& f, const SketchCfg& base,
                                    const std::vector<uint64_t>& seeds) {
    const int K = static_cast<int>(seeds.size());
    const int64_t n = k.n, ld = k.rpr, rows = k.rows;
    const int s_q = base.s_q, s_g = base.s_g, cost = f.query_cost();
    std::vector<TraceEst> out(K);
    if (s_q < 0 || s_g < 0 || s_q + s_g < 1) fail(kInvalidArgument, "hutchpp needs a positive query budget");
    if (s_q >= n || base.sketch || base.probes) {  // exact branch or injected probes: one trial at a time
        for (int t = 0; t < K; ++t) {
            SketchCfg c = base;
            c.seed = seeds[t];
            out[t] = hutchpp(ctx, k, f, c);
        }
        return out;
    }
    // sketch products of every trial: Y = A·[S_0 | S_1 | ...]
    std::vector<DevBuf> q(K);
    std::vector<int> rank(K, 0);
    if (s_q > 0) {
        const int cols = K * s_q;
        DevBuf sk, y;
        sk.alloc(static_cast<size_t>(cols) * ld * sizeof(double));
        y.alloc(static_cast<size_t>(cols) * ld * sizeof(double));
        for (int t = 0; t < K; ++t) {
            DevBuf one;
            make_probes(ctx, k, one, s_q, ld, nullptr, seeds[t], "hutchpp-sketch", base.probe_kind);
            cuda_check(cudaMemcpyAsync(sk.as<double>() + static_cast<int64_t>(t) * s_q * ld, one.as<double>(),
                                       static_cast<size_t>(s_q) * ld * sizeof(double), cudaMemcpyDeviceToDevice,
                                       ctx.stream()),
                       "copy sketch");
        }
        for (int j0 = 0; j0 < cols; j0 += kMaxPanelCols) {
            const int w = std::min(kMaxPanelCols, cols - j0);
            run_panel(ctx, k, sk.as<double>() + static_cast<int64_t>(j0) * ld, ld, w, {{1.0, 0.0, 0.0}}, nullptr,
                      nullptr, y.as<double>() + static_cast<int64_t>(j0) * ld, ld);
        }
        for (int t = 0; t < K; ++t) {
            rank[t] = orthonormal_range(ctx, y.as<double>() + static_cast<int64_t>(t) * s_q * ld, s_q, ld, rows, q[t]);
            if (rank[t] == 0) fail(kRankCollapse, "trial " + std::to_string(t) + ": hutchpp sketch A*S is numerically zero");
            if (s_g >= n - rank[t]) {  // exact-complement branch for this trial: run it on its own
                SketchCfg c = base;
                c.seed = seeds[t];
                out[t] = hutchpp(ctx, k, f, c);
                rank[t] = -1;
            }
        }
    }
    // X0 = [Q_0 | W_0 | Q_1 | W_1 | ...],  W_t = G_t - Q_t (Q_tᵀ G_t)
    std::vector<int64_t> off(K, 0);
    int64_t total = 0;
    for (int t = 0; t < K; ++t) {
        off[t] = total;
        if (rank[t] >= 0) total += rank[t] + s_g;
    }
    if (total == 0) return out;
    DevBuf x0;
    x0.alloc(static_cast<size_t>(total) * ld * sizeof(double));
    for (int t = 0; t < K; ++t) {
        if (rank[t] < 0) continue;
        double* dst = x0.as<double>() + off[t] * ld;
        if (rank[t] > 0)
            cuda_check(cudaMemcpyAsync(dst, q[t].as<double>(), static_cast<size_t>(rank[t]) * ld * sizeof(double),
                                       cudaMemcpyDeviceToDevice, ctx.stream()),
                       "copy Q");
        if (s_g > 0) {
            double* wdst = dst + static_cast<int64_t>(rank[t]) * ld;
            DevBuf gp;
            make_probes(ctx, k, gp, s_g, ld, nullptr, seeds[t], "hutchpp-probe", base.probe_kind);
            if (rank[t] > 0) {
                std::vector<double> c = gram_host(ctx, q[t].as<double>(), rank[t], ld, gp.as<double>(), s_g, ld, rows);
                for (double& v : c) v = -v;
                update(ctx, 1.0, gp.as<double>(), ld, q[t].as<double>(), rank[t], ld, c, s_g, rows, wdst, ld);
            } else {
                cuda_check(cudaMemcpyAsync(wdst, gp.as<double>(), static_cast<size_t>(s_g) * ld * sizeof(double),
                                           cudaMemcpyDeviceToDevice, ctx.stream()),
                           "copy probes");
                ctx.sync();
            }
        }
    }
    const std::vector<double> tr = panel_traces(ctx, k, f, x0.as<double>(), ld, static_cast<int>(total));
    for (int t = 0; t < K; ++t) {
        if (rank[t] < 0) continue;
        TraceEst& e = out[t];
        double low = 0.0, res = 0.0;
        for (int j = 0; j < rank[t]; ++j) low += tr[off[t] + j];
        for (int j = 0; j < s_g; ++j) res += tr[off[t] + rank[t] + j];
        e.sketch_rank = rank[t];
        e.low_rank_part = low;
        e.residual_part = s_g > 0 ? res / s_g : 0.0;
        e.queries_used = (s_q > 0 ? s_q + rank[t] * cost : 0) + s_g * cost;
        e.value = e.low_rank_part + e.residual_part;
    }
    return out;
}

}  // namespace

std::vector<EntropyEst> estimate_trials(Context& ctx, const KernelMatrix& k, const EstParams& p, int trials) {
    // K trials of estimate() with seeds derive_key(p.seed, t) and the bounds resolved once, as
    // measure_cell does them (proj/src/simulate.cpp:19-51), batched over shared passes.
    if (trials < 1) fail(kInvalidArgument, "need at least one trial");
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    const auto t0 = std::chrono::steady_clock::now();
    const Resolved r = resolve(ctx, k, p);
    std::vector<uint64_t> seeds(trials);
    for (int t = 0; t < trials; ++t) seeds[t] = derive_key(p.seed, static_cast<uint64_t>(t));
    const SketchCfg base = sketch_cfg(p, r.s);
    const std::vector<TraceEst> tr = hutchpp_batch(ctx, k, r.f, base, seeds);
    const double per = seconds_since(t0) / trials;
    std::vector<EntropyEst> out(trials);
    for (int t = 0; t < trials; ++t) {
        try {
            out[t] = entropy_of(tr[t], r.alpha, r.method, r.s, r.m_used);
        } catch (const Error& e) {
            fail(e.code(), "trial " + std::to_string(t) + ": " + e.what());
        }
        out[t].has_bounds = r.has_bounds;
        out[t].bounds_used = r.bounds;
        out[t].elapsed = per;
    }
    return out;
}

MreCell measure_cell(Context& ctx, const KernelMatrix& k, double exact_entropy, const EstParams& p, int trials) {
    // proj/src/simulate.cpp:19-72
    if (trials < 1) fail(kInvalidArgument, "need at least one trial");
    const std::vector<EntropyEst> est = estimate_trials(ctx, k, p, trials);
    MreCell cell;
    cell.alpha = p.alpha;
    cell.s = p.s;
    cell.m = p.m;
    cell.method = p.method;
    cell.trials = trials;
    double sum = 0.0, tsum = 0.0;
    std::vector<double> rel(trials);
    for (int t = 0; t < trials; ++t) {
        rel[t] = std::abs(est[t].entropy - exact_entropy) / std::abs(exact_entropy);
        sum += rel[t];
        tsum += est[t].elapsed;
    }
    cell.mre = sum / trials;
    double var = 0.0;
    for (double x : rel) var += (x - cell.mre) * (x - cell.mre);
    cell.sd = trials > 1 ? std::sqrt(var / (trials - 1)) : 0.0;
    cell.mean_elapsed = tsum / trials;
    return cell;
}

EstParams with_seed(const EstParams& p, const char* term) {
    EstParams q = p;
    q.seed = derive_key(p.seed, hash_name(term));
    return q;
}

// ---------------------------------------------------------------- fused mutual information
// The three terms of I(X;Y) = S(A) + S(B) - S(n·A∘B) (proj/src/measures.cpp:36-46) run their Hutch++
// estimates in lockstep: every pass is one launch_block_av_tri over A and B that also forms the joint
// kernel J = n·(A∘B) (proj/src/kernel.cpp:74-108) tile by tile, so J is never stored and each pass reads
// 8 B per entry instead of 12 B. Per-term arithmetic (probes, recurrences, QR, traces) is unchanged.
namespace {

struct JointMeta {
    KernelMatrix k;  // metadata only (no storage): what the sessions and resolve() read
    double factor = 0.0, diag = 0.0;
};

JointMeta joint_meta(const KernelMatrix& a, const KernelMatrix& b) {
    // the same stored representation hadamard_joint() materialises (split planes of J·n·2^14)
    JointMeta m;
    KernelMatrix& c = m.k;
    c.n = a.n, c.row0 = a.row0, c.rows = a.rows, c.ld = a.ld, c.prec = a.prec;
    c.rpr = a.rpr, c.world = a.world, c.rank = a.rank;
    const double nd = static_cast<double>(a.n);
    const double inv_n = 1.0 / nd;
    c.a_norm = (a.normalized && b.normalized) ? 1.0 : std::max(1.0, a.a_norm * b.a_norm * nd);
    c.normalized = a.normalized && b.normalized;
    c.unscale = inv_n / kSplitScale;
    m.factor = nd * a.unscale * b.unscale / c.unscale;
    m.diag = inv_n / c.unscale;
    // the fused kernel prescales A and B by exact powers of two: factor = 2^e up to rounding of n·fl(1/n)
    int e = 0;
    const double fr = std::frexp(m.factor, &e);
    m.factor = std::abs(fr - 0.5) <= 1e-12 ? std::ldexp(1.0, e - 1) : 0.0;  // 0: not fusable
    return m;
}

struct Tri {
    const KernelMatrix* a;
    const KernelMatrix* b;
    JointMeta j;
    const KernelMatrix* op(int i) const { return i == 0 ? a : (i == 1 ? b : &j.k); }
};

// P lockstep passes over three panels x_i of width s (<= tri_max_cols): sched[i][p] are operand i's
// recurrence coefficients; last_out[i] (optional) receives T_P
std::array<PanelResult, 3> run_panel3(Context& ctx, const Tri& t, const double* const* x, int64_t ldx, int s,
                                      const std::array<std::vector<std::array<double, 3>>, 3>& sched,
                                      double* const* last_out, int64_t ldo) {
    const int P = static_cast<int>(sched[0].size());
    PanelWorkspace* ws[3] = {&ctx.ws, &ctx.ws_aux[0], &ctx.ws_aux[1]};
    std::array<std::unique_ptr<PanelSession>, 3> ps;
    for (int i = 0; i < 3; ++i)
        ps[i] = std::make_unique<PanelSession>(ctx, *t.op(i), x[i], ldx, s, std::max(P, 1), nullptr, 0.0,
                                               last_out != nullptr, ws[i], true);
    const KernelMatrix& a = *t.a;
    const KernelMatrix& b = *t.b;
    const SplitMatrixView av{a.hi.as<__half>(), a.lo.as<__half>(), a.rows, a.n, a.ld};
    const SplitMatrixView bv{b.hi.as<__half>(), b.lo.as<__half>(), b.rows, b.n, b.ld};
    for (int p = 0; p < P; ++p) {
        const SplitPanelView v[3] = {ps[0]->operand(), ps[1]->operand(), ps[2]->operand()};
        float* const part[3] = {ps[0]->partial(), ps[1]->partial(), ps[2]->partial()};
        float* const part2[3] = {ps[0]->partial2(), ps[1]->partial2(), ps[2]->partial2()};
        NvtxRange nvtx("fused MI pass");
        // row-sharded: the rank's own operand chunk first, the other chunks after the sessions' all-gathers
        for (int w = 0; w < (ps[0]->split() ? 2 : 1); ++w) {
            const StreamKPlan& pl = w == 0 ? ps[0]->plan() : ps[0]->plan2();
            if (w == 1) ctx.main_after_comm();
            const double frac = ps[0]->split() ? static_cast<double>(w == 0 ? a.rows : a.n - a.rows) / a.n : 1.0;
            ctx.prof_begin();
            if (a.rows > 0 && pl.k_tiles > 0)
                launched(ctx,
                         launch_block_av_tri(av, bv, v, pl, w == 0 ? part : part2, a.row0, t.j.factor, t.j.diag,
                                             ctx.stream()),
                         "block_av_tri");
            ctx.prof_end();
            // algorithmic bytes: A and B (4 B/entry each) + three operand panels + three results
            ctx.prof_account(frac * (8.0 * a.rows * a.n + 3.0 * (v[0].vlo ? 4.0 : 2.0) * a.n * s) +
                                 3.0 * 4.0 * a.rows * s,
                             frac * 3.0 * 2.0 * a.rows * a.n * s);
        }
        for (int i = 0; i < 3; ++i) ps[i]->finish(sched[i][p][0], sched[i][p][1], sched[i][p][2], 0.0);
    }
    std::array<PanelResult, 3> r;
    for (int i = 0; i < 3; ++i) {
        if (last_out) ps[i]->state_f64(P, last_out[i], ldo);
        r[i].passes = P;
        r[i].s = s;
        r[i].dots = ps[i]->dots(0, P);
    }
    return r;
}

// per-column traces x_j^T f_i(M_i) x_j of three device panels [cols][ldx] (moment doubling, as panel_traces)
std::array<std::vector<double>, 3> panel_traces3(Context& ctx, const Tri& t, const std::array<MatFun, 3>& f,
                                                 const double* const* x, int64_t ldx, int cols) {
    std::array<std::vector<double>, 3> tr;
    std::array<std::vector<std::array<double, 3>>, 3> sched;
    const int passes = (f[0].degree + 1) / 2;
    for (int i = 0; i < 3; ++i) {
        tr[i].assign(cols, 0.0);
        const auto full = schedule(f[i]);
        sched[i].assign(full.begin(), full.begin() + passes);
    }
    const int W = tri_max_cols();
    for (int j0 = 0; j0 < cols; j0 += W) {
        const int w = std::min(W, cols - j0);
        const double* xs[3] = {x[0] + static_cast<int64_t>(j0) * ldx, x[1] + static_cast<int64_t>(j0) * ldx,
                               x[2] + static_cast<int64_t>(j0) * ldx};
        const auto r = run_panel3(ctx, t, xs, ldx, w, sched, nullptr, 0);
        for (int i = 0; i < 3; ++i) {
            std::vector<double> mu(f[i].degree + 1);
            for (int j = 0; j < w; ++j) {
                doubled_moments(f[i], r[i], j, mu.data());
                tr[i][j0 + j] = f[i].combine(mu.data(), 1);
            }
        }
    }
    return tr;
}

// hutchpp() for the three terms in lockstep (main branch; the caller guarantees s_q + s_g < n)
std::array<TraceEst, 3> hutchpp3(Context& ctx, const Tri& t, const std::array<MatFun, 3>& f,
                                 const std::array<SketchCfg, 3>& cfg) {
    const KernelMatrix& k0 = *t.a;
    const int64_t ld = k0.rpr, rows = k0.rows;
    const int s_q = cfg[0].s_q, s_g = cfg[0].s_g;
    std::array<TraceEst, 3> est;
    std::array<DevBuf, 3> qbuf;
    std::array<int, 3> rank{0, 0, 0};
    if (s_q > 0) {
        std::array<DevBuf, 3> sk, y;
        for (int i = 0; i < 3; ++i) {
            make_probes(ctx, *t.op(i), sk[i], s_q, ld, cfg[i].sketch, cfg[i].seed, "hutchpp-sketch",
                        cfg[i].probe_kind);
            y[i].alloc(static_cast<size_t>(s_q) * ld * sizeof(double));
        }
        const std::array<std::vector<std::array<double, 3>>, 3> one{{{{1.0, 0.0, 0.0}}, {{1.0, 0.0, 0.0}},
                                                                      {{1.0, 0.0, 0.0}}}};
        const int W = tri_max_cols();
        for (int j0 = 0; j0 < s_q; j0 += W) {
            const int w = std::min(W, s_q - j0);
            const double* xs[3];
            double* ys[3];
            for (int i = 0; i < 3; ++i) {
                xs[i] = sk[i].as<double>() + j0 * ld;
                ys[i] = y[i].as<double>() + j0 * ld;
            }
            run_panel3(ctx, t, xs, ld, w, one, ys, ld);
        }
        for (int i = 0; i < 3; ++i) {
            rank[i] = orthonormal_range(ctx, y[i].as<double>(), s_q, ld, rows, qbuf[i]);
            if (rank[i] == 0) fail(kRankCollapse, "hutchpp sketch A*S is numerically zero");
            est[i].sketch_rank = rank[i];
            est[i].queries_used = s_q + rank[i] * f[i].query_cost();
        }
    }
    // X0_i = [Q_i | W_i | 0]: one width for the lockstep panels (zero columns trace to zero)
    const int cols = *std::max_element(rank.begin(), rank.end()) + s_g;
    std::array<DevBuf, 3> x0;
    for (int i = 0; i < 3; ++i) {
        x0[i].alloc(static_cast<size_t>(cols) * ld * sizeof(double));
        cuda_check(cudaMemsetAsync(x0[i].as<double>(), 0, static_cast<size_t>(cols) * ld * sizeof(double),
                                   ctx.stream()),
                   "memset");
        if (rank[i] > 0)
            cuda_check(cudaMemcpyAsync(x0[i].as<double>(), qbuf[i].as<double>(),
                                       static_cast<size_t>(rank[i]) * ld * sizeof(double), cudaMemcpyDeviceToDevice,
                                       ctx.stream()),
                       "copy Q");
        if (s_g > 0) {
            double* wdst = x0[i].as<double>() + static_cast<int64_t>(rank[i]) * ld;
            DevBuf gp;
            make_probes(ctx, *t.op(i), gp, s_g, ld, cfg[i].probes, cfg[i].seed, "hutchpp-probe", cfg[i].probe_kind);
            if (rank[i] > 0) {
                std::vector<double> c =
                    gram_host(ctx, qbuf[i].as<double>(), rank[i], ld, gp.as<double>(), s_g, ld, rows);
                for (double& v : c) v = -v;
                update(ctx, 1.0, gp.as<double>(), ld, qbuf[i].as<double>(), rank[i], ld, c, s_g, rows, wdst, ld);
            } else {
                cuda_check(cudaMemcpyAsync(wdst, gp.as<double>(), static_cast<size_t>(s_g) * ld * sizeof(double),
                                           cudaMemcpyDeviceToDevice, ctx.stream()),
                           "copy probes");
            }
            ctx.sync();  // gp is released at scope end
        }
    }
    const double* xs[3] = {x0[0].as<double>(), x0[1].as<double>(), x0[2].as<double>()};
    const auto tr = panel_traces3(ctx, t, f, xs, ld, cols);
    for (int i = 0; i < 3; ++i) {
        double low = 0.0, res = 0.0;
        for (int j = 0; j < rank[i]; ++j) low += tr[i][j];
        for (int j = rank[i]; j < rank[i] + s_g; ++j) res += tr[i][j];
        est[i].low_rank_part = low;
        est[i].residual_part = s_g > 0 ? res / s_g : 0.0;
        est[i].queries_used += s_g * f[i].query_cost();
        est[i].value = est[i].low_rank_part + est[i].residual_part;
    }
    return est;
}

// the fused pass needs no spectrum bounds of J (J is never formed as a matrix)
bool fused_mi_params(const EstParams& p) {
    int ai = 0;
    const bool is_int = integer_alpha(p.alpha, &ai);
    if (p.method == kMethodExact) return false;
    return p.has_bounds || (is_int && (p.method == kMethodAuto || p.method == kMethodInt));
}

bool mutual_information_fused(Context& ctx, const KernelMatrix& a, const KernelMatrix& b, const EstParams& p,
                              MutualInfo* out) {
    if (!ctx.fused_mi || !fused_mi_params(p)) return false;
    if (a.prec != kF32 || b.prec != kF32 || a.n != b.n || a.rows != b.rows || a.row0 != b.row0 || a.ld != b.ld ||
        a.rpr != b.rpr || a.world != b.world || a.rank != b.rank)
        return false;
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    Tri t{&a, &b, joint_meta(a, b)};
    if (t.j.factor == 0.0) return false;
    const EstParams q[3] = {with_seed(p, "term:vars"), with_seed(p, "term:target"), with_seed(p, "term:joint")};
    std::array<Resolved, 3> r;
    std::array<MatFun, 3> f;
    std::array<SketchCfg, 3> cfg;
    for (int i = 0; i < 3; ++i) {
        r[i] = resolve(ctx, *t.op(i), q[i]);
        f[i] = r[i].f;
        cfg[i] = sketch_cfg(q[i], r[i].s);
    }
    for (int i = 1; i < 3; ++i)
        if (f[i].degree != f[0].degree || cfg[i].s_q != cfg[0].s_q || cfg[i].s_g != cfg[0].s_g) return false;
    const int s_q = cfg[0].s_q, s_g = cfg[0].s_g;
    if (s_q < 0 || s_g < 0 || s_q + s_g < 1) fail(kInvalidArgument, "hutchpp needs a positive query budget");
    if (static_cast<int64_t>(s_q) + s_g >= a.n) return false;  // exact branches: the sequential path
    const auto tr = hutchpp3(ctx, t, f, cfg);
    double h[3];
    for (int i = 0; i < 3; ++i) h[i] = entropy_of(tr[i], r[i].alpha, r[i].method, r[i].s, r[i].m_used).entropy;
    out->vars_entropy = h[0];
    out->target_entropy = h[1];
    out->joint_entropy = h[2];
    out->value = h[0] + h[1] - h[2];
    return true;
}

}  // namespace

MutualInfo mutual_information(Context& ctx, const KernelMatrix& a, const KernelMatrix& b, const EstParams& p) {
    NvtxRange nvtx("mutual_information");
    // proj/src/measures.cpp:36-46 (single-variable set: vars_joint = a)
    MutualInfo fused;
    if (mutual_information_fused(ctx, a, b, p, &fused)) return fused;
    KernelPtr joint = hadamard_joint(ctx, a, b);
    MutualInfo mi;
    mi.vars_entropy = estimate(ctx, a, with_seed(p, "term:vars")).entropy;
    mi.target_entropy = estimate(ctx, b, with_seed(p, "term:target")).entropy;
    mi.joint_entropy = estimate(ctx, *joint, with_seed(p, "term:joint")).entropy;
    mi.value = mi.vars_entropy + mi.target_entropy - mi.joint_entropy;
    return mi;
}

MutualInfo mutual_information_samples(Context& ctx, const double* x, int64_t n, int64_t dx, int64_t ldx,
                                      double sigma_x, const double* y, int64_t dy, int64_t ldy, double sigma_y,
                                      const EstParams& p, int prec) {
    // host buffers: upload X and Y once (column-major as given), then the device path (which validates)
    if (n < 2) fail(kInvalidArgument, "need at least 2 samples, got " + std::to_string(n));
    if (dx < 1 || dy < 1) fail(kInvalidArgument, "samples need at least one feature");
    if (ldx < n || ldy < n) fail(kInvalidArgument, "leading dimension smaller than the sample count");
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    DevBuf xs;
    xs.alloc(static_cast<size_t>(n) * (dx + dy) * sizeof(double));
    if (ldx == n) h2d_staged(ctx, xs.as<double>(), x, static_cast<size_t>(n) * dx * sizeof(double));
    else h2d_2d(ctx, xs.as<double>(), n * sizeof(double), x, ldx * sizeof(double), n * sizeof(double), dx);
    if (ldy == n) h2d_staged(ctx, xs.as<double>() + n * dx, y, static_cast<size_t>(n) * dy * sizeof(double));
    else h2d_2d(ctx, xs.as<double>() + n * dx, n * sizeof(double), y, ldy * sizeof(double), n * sizeof(double), dy);
    MutualInfo mi = mutual_information_samples_dev(ctx, xs.as<double>(), n, dx, n, sigma_x, xs.as<double>() + n * dx,
                                                   dy, n, sigma_y, p, prec);
    ctx.sync();
    return mi;
}

MutualInfo mutual_information_samples_dev(Context& ctx, const double* x, int64_t n, int64_t dx, int64_t ldx,
                                          double sigma_x, const double* y, int64_t dy, int64_t ldy, double sigma_y,
                                          const EstParams& p, int prec) {
    MutualInfo mi;
    if (prec == kF32 && ctx.fused_mi && fused_mi_params(p)) {
        // host-drawn probes: all six panels (sketch and residual probes of the three terms,
        // hutchpp3's seeds and labels) are generated on the host while the device builds A and B
        if (ctx.probe_source == 1 && p.s > 0) {  // sketch panels first: they are needed first
            std::vector<Context::ProbeReq> reqs;
            for (const char* label : {"hutchpp-sketch", "hutchpp-probe"})
                for (const char* term : {"term:vars", "term:target", "term:joint"}) {
                    const SketchCfg c = sketch_cfg(with_seed(p, term), p.s);
                    reqs.push_back({n, label[8] == 's' ? c.s_q : c.s_g, c.seed, label, c.probe_kind});
                }
            ctx.prefetch_probes(reqs);
        }
        // A and B resident together; the joint term is formed inside the fused passes
        KernelPtr a = build_gaussian_dev(ctx, x, n, dx, ldx, sigma_x, prec);
        KernelPtr b = build_gaussian_dev(ctx, y, n, dy, ldy, sigma_y, prec);
        const bool done = mutual_information_fused(ctx, *a, *b, p, &mi);
        ctx.drop_prefetched_probes();
        if (done) return mi;
    }
    {
        KernelPtr a = build_gaussian_dev(ctx, x, n, dx, ldx, sigma_x, prec);
        mi.vars_entropy = estimate(ctx, *a, with_seed(p, "term:vars")).entropy;
    }
    {
        KernelPtr b = build_gaussian_dev(ctx, y, n, dy, ldy, sigma_y, prec);
        mi.target_entropy = estimate(ctx, *b, with_seed(p, "term:target")).entropy;
    }
    {
        KernelPtr j = build_gaussian_dev(ctx, x, n, dx, ldx, sigma_x, prec, y, dy, ldy, sigma_y);
        mi.joint_entropy = estimate(ctx, *j, with_seed(p, "term:joint")).entropy;
    }
    mi.value = mi.vars_entropy + mi.target_entropy - mi.joint_entropy;
    return mi;
}

// ---------------------------------------------------------------- feature tools
// proj/src/features.cpp: every score is S(F) + S(Y) - S(F∘Y) with the mutual_information seed
// schedule; kernels stay resident on the device (select keeps all d feature kernels).
std::string FeatureData::name(int j) const {
    return j < static_cast<int>(names.size()) ? names[j] : "feature_" + std::to_string(j);
}

// ---------------------------------------------------------------- grouped estimates (feature tools)
// Scoring feature candidates (proj/src/features.cpp:44-162) is many estimates with identical
// parameters over different n x n kernels of the same n; at the reference's n <= 14k each estimate
// alone is latency-bound (a few hundred KB-MB per pass, host round trips for Hutch++'s QR). Here G
// candidates' kernels sit in ONE stacked allocation (KernelMatrix::groups) and every pass is one
// block product over all of them (the operand chunk of each group read through the stacked operand
// planes), one epilogue, one trace reduction per group; only the small per-candidate QR stays
// per group. Every row block is computed whole by one CTA pair (the stack is padded to whole
// pair-block waves), so a candidate's numbers do not depend on its position in the stack: identical
// features score bitwise identically, as in the reference's sequential loop.
namespace {

constexpr int kGroupMax = 64;                  // candidates per stack
constexpr double kGroupBytes = 12e9;           // per stacked matrix

int64_t group_rows_of(int64_t n) { return round_up(n, 512); }

int group_capacity(int64_t n) {
    const double per = static_cast<double>(group_rows_of(n)) * matrix_pitch(n) * 4.0;
    return static_cast<int>(std::max(1.0, std::min<double>(kGroupMax, std::floor(kGroupBytes / per))));
}

KernelPtr alloc_group(Context& ctx, int64_t n, int groups) {
    auto k = std::make_unique<KernelMatrix>();
    k->n = n, k->prec = kF32, k->world = 1, k->rank = 0, k->row0 = 0;
    k->ld = matrix_pitch(n);
    k->groups = groups;
    k->group_rows = group_rows_of(n);
    const int64_t pb = static_cast<int64_t>(groups) * k->group_rows / 512;  // CTA-pair row blocks
    const int64_t pairs = std::max<int64_t>(1, std::min<int64_t>(ctx.sms() / 2, pb));
    const int64_t waves = (pb + pairs - 1) / pairs;
    k->rows = pairs * waves * 512;  // zero pair blocks pad the last wave
    k->rpr = k->rows;
    k->group_grid = static_cast<int>(2 * pairs);
    k->unscale = (1.0 / static_cast<double>(n)) / kSplitScale;
    k->a_norm = 1.0;
    k->normalized = true;
    const size_t elems = static_cast<size_t>(k->rows) * k->ld;
    k->hi.alloc(elems * sizeof(__half));
    k->lo.alloc(elems * sizeof(__half));
    cuda_check(cudaMemsetAsync(k->hi.as<void>(), 0, elems * sizeof(__half), ctx.stream()), "memset");
    cuda_check(cudaMemsetAsync(k->lo.as<void>(), 0, elems * sizeof(__half), ctx.stream()), "memset");
    return k;
}

__half* group_hi(const KernelMatrix& k, int g) { return k.hi.as<__half>() + static_cast<size_t>(g) * k.group_rows * k.ld; }
__half* group_lo(const KernelMatrix& k, int g) { return k.lo.as<__half>() + static_cast<size_t>(g) * k.group_rows * k.ld; }

// build_kernel(X[:, col], GaussianKernel{sigma}) into group g: the fp32 build_gaussian_dev's Gram, same
// arguments, so the planes are bitwise those of a singly built feature kernel
void group_gram(Context& ctx, const KernelMatrix& k, int g, const double* d_col, double sigma) {
    GramArgs ga{};
    ga.x = d_col, ga.dx = 1, ga.x_rs = 1, ga.x_cs = k.n;
    ga.inv_two_sigma2_x = 1.0 / (2.0 * sigma * sigma);
    ga.y = nullptr, ga.dy = 0, ga.y_rs = 1, ga.y_cs = 0, ga.inv_two_sigma2_y = 0.0;
    ga.n = k.n, ga.row0 = 0, ga.rows = k.n, ga.ld = k.ld;
    ga.inv_n = 1.0 / static_cast<double>(k.n);
    ga.f32_compute = 1;
    DevBuf scratch;
    scratch.alloc(gram_split_scratch_bytes(ga));
    launched(ctx, launch_gram_split(ga, group_hi(k, g), group_lo(k, g), scratch.as<void>(), ctx.stream()), "gram_split");
}

// group g <- hadamard_joint(a, b) (proj/src/kernel.cpp:74-101, L = 2), a / b single fp32 kernels or groups
void group_hadamard(Context& ctx, const KernelMatrix& out, int g, const __half* ahi, const __half* alo,
                    const __half* bhi, const __half* blo) {
    const double inv_n = 1.0 / static_cast<double>(out.n);
    const double factor = static_cast<double>(out.n) * out.unscale * out.unscale / out.unscale;
    const double diag = inv_n / out.unscale;
    launched(ctx,
             launch_hadamard_split(ahi, alo, bhi, blo, out.n, out.n, out.ld, 0, factor, diag, group_hi(out, g),
                                   group_lo(out, g), ctx.stream()),
             "hadamard_split");
}

// ---- batched small panel algebra for the groups: every step below issues the device work of all
// groups and synchronises once, instead of once per group (orthonormal_range runs ~12 round trips)
struct GramJob {
    const double* x;
    int p;
    const double* z;
    int q;
};
// X_iᵀ Z_i (n rows, leading dimension ld) for every job, one device round trip
std::vector<std::vector<double>> grams_batch(Context& ctx, const std::vector<GramJob>& jobs, int64_t ld, int64_t n) {
    size_t total = 0;
    for (const auto& j : jobs) total += static_cast<size_t>(j.p) * j.q;
    std::vector<std::vector<double>> out(jobs.size());
    if (total == 0) return out;
    for (const auto& j : jobs)
        if (j.p > 128) {  // wide sketches: one row-blocked Gram per job (gram_host)
            for (size_t i = 0; i < jobs.size(); ++i) out[i] = gram_host(ctx, jobs[i].x, jobs[i].p, ld, jobs[i].z, jobs[i].q, ld, n);
            return out;
        }
    const int grid = std::min<int64_t>(ctx.sms(), std::max<int64_t>(1, (n + 31) / 32));
    ctx.small.ensure(total * sizeof(double));
    size_t off = 0;
    for (const auto& j : jobs) {
        const int qb_max = std::max(1, std::min(2048 / std::max(j.p, 1), 190 - j.p));
        for (int b0 = 0; b0 < j.q; b0 += qb_max) {
            const int qb = std::min(qb_max, j.q - b0);
            ctx.gram_partial.ensure(static_cast<size_t>(grid) * j.p * qb * sizeof(double));
            launched(ctx,
                     launch_panel_gram(j.x, j.p, ld, j.z + static_cast<int64_t>(b0) * ld, qb, ld, n,
                                       ctx.gram_partial.as<double>(), grid,
                                       ctx.small.as<double>() + off + static_cast<size_t>(b0) * j.p, ctx.stream(),
                                       ctx.gram_ticket.as<unsigned>()),
                     "panel_gram");
        }
        off += static_cast<size_t>(j.p) * j.q;
    }
    std::vector<double> all(total);
    d2h(ctx, all.data(), ctx.small.as<double>(), total * sizeof(double));
    ctx.sync();
    off = 0;
    for (size_t i = 0; i < jobs.size(); ++i) {
        const size_t sz = static_cast<size_t>(jobs[i].p) * jobs[i].q;
        out[i].assign(all.begin() + off, all.begin() + off + sz);
        off += sz;
    }
    return out;
}

struct UpdateJob {
    double beta;
    const double* g;  // may be null (beta = 0)
    const double* x;
    int p;
    std::vector<double> c;  // p x q column-major
    int q;
    double* w;
};
// W = beta G + X C for every job (leading dimension ld, n rows): one upload of all C, no round trip
void updates_batch(Context& ctx, const std::vector<UpdateJob>& jobs, int64_t ld, int64_t n) {
    size_t total = 0;
    for (const auto& j : jobs) total += j.c.size();
    if (total == 0) return;
    std::vector<double> all;
    all.reserve(total);
    for (const auto& j : jobs) all.insert(all.end(), j.c.begin(), j.c.end());
    DevBuf cd;
    cd.alloc(total * sizeof(double));
    h2d(ctx, cd.as<double>(), all.data(), total * sizeof(double));
    size_t off = 0;
    for (const auto& j : jobs) {
        const int qb_max = std::max(1, (48 * 1024 / 8) / std::max(j.p, 1));
        for (int b0 = 0; b0 < j.q; b0 += qb_max) {
            const int qb = std::min(qb_max, j.q - b0);
            launched(ctx,
                     launch_panel_update(j.beta, j.g ? j.g + static_cast<int64_t>(b0) * ld : nullptr, ld, j.x, j.p, ld,
                                         cd.as<double>() + off + static_cast<size_t>(b0) * j.p, qb, n,
                                         j.w + static_cast<int64_t>(b0) * ld, ld, ctx.stream()),
                     "panel_update");
        }
        off += j.c.size();
    }
    ctx.sync();  // `all` (host) and cd outlive the copies
}

// orthonormal_range (above) for a batch of sketches Y_i [p][ld] (n rows each): the same steps and
// rank rules per sketch, each step issued for every sketch before one synchronisation
std::vector<int> orthonormal_range_batch(Context& ctx, const std::vector<const double*>& ys, int p, int64_t ld,
                                         int64_t n, std::vector<DevBuf>& q_out) {
    const size_t G = ys.size();
    std::vector<int> rank(G, 0), k(G, 0);
    std::vector<double> w0(G, 0.0);
    std::vector<DevBuf> q1(G), qa(G), y2(G);
    auto scaled_vectors = [&](const std::vector<double>& ww, const std::vector<double>& vv, int cols) {
        std::vector<double> m(static_cast<size_t>(p) * cols);
        for (int c = 0; c < cols; ++c) {
            const double sc = 1.0 / std::sqrt(ww[c]);
            for (int r = 0; r < p; ++r) m[r + static_cast<size_t>(c) * p] = vv[r + static_cast<size_t>(c) * p] * sc;
        }
        return m;
    };
    // CholeskyQR (eigen fallback) of X_i (cols_i columns) into out_i, batched
    auto chol_qr = [&](const std::vector<size_t>& ids, const std::vector<const double*>& xs, const std::vector<int>& cols,
                       const std::vector<double*>& outs) {
        std::vector<GramJob> gj;
        for (size_t t = 0; t < ids.size(); ++t) gj.push_back({xs[t], cols[t], xs[t], cols[t]});
        std::vector<std::vector<double>> gs = grams_batch(ctx, gj, ld, n);
        std::vector<UpdateJob> uj;
        for (size_t t = 0; t < ids.size(); ++t) {
            std::vector<double> r2;
            const int c = cols[t];
            if (cholesky_upper(c, gs[t], r2)) {
                uj.push_back({0.0, nullptr, xs[t], c, upper_inverse(c, r2), c, outs[t]});
            } else {
                std::vector<double> w2, v2;
                sym_eig_desc(c, gs[t], w2, v2);
                std::vector<double> m2(static_cast<size_t>(c) * c);
                for (int cc = 0; cc < c; ++cc)
                    for (int r = 0; r < c; ++r)
                        m2[r + static_cast<size_t>(cc) * c] = v2[r + static_cast<size_t>(cc) * c] / std::sqrt(w2[cc]);
                uj.push_back({0.0, nullptr, xs[t], c, std::move(m2), c, outs[t]});
            }
        }
        updates_batch(ctx, uj, ld, n);
    };
    std::vector<GramJob> gj;
    for (size_t g = 0; g < G; ++g) gj.push_back({ys[g], p, ys[g], p});
    std::vector<std::vector<double>> gs = grams_batch(ctx, gj, ld, n);
    std::vector<UpdateJob> uj;
    std::vector<size_t> live;
    for (size_t g = 0; g < G; ++g) {
        std::vector<double> w, v;
        sym_eig_desc(p, gs[g], w, v);
        if (!(w.size() > 0 && w[0] > 0.0)) continue;
        w0[g] = w[0];
        while (k[g] < p && w[k[g]] > 1e-13 * w0[g]) ++k[g];
        if (k[g] == 0) continue;
        q1[g].alloc(static_cast<size_t>(p) * ld * sizeof(double));
        qa[g].alloc(static_cast<size_t>(p) * ld * sizeof(double));
        uj.push_back({0.0, nullptr, ys[g], p, scaled_vectors(w, v, k[g]), k[g], q1[g].as<double>()});
        live.push_back(g);
    }
    updates_batch(ctx, uj, ld, n);
    {
        std::vector<const double*> xs;
        std::vector<int> cols;
        std::vector<double*> outs;
        for (size_t g : live) xs.push_back(q1[g].as<double>()), cols.push_back(k[g]), outs.push_back(qa[g].as<double>());
        chol_qr(live, xs, cols, outs);  // second pass: orthogonal to working precision
    }
    for (size_t g : live) rank[g] = k[g];
    // residual pass for sketches that dropped columns: Y2 = Y - Q (Q^T Y); keep sigma(Y2) > 1e-12 sigma_0
    std::vector<size_t> res;
    for (size_t g : live)
        if (k[g] < p) res.push_back(g);
    if (!res.empty()) {
        gj.clear();
        for (size_t g : res) gj.push_back({qa[g].as<double>(), k[g], ys[g], p});
        gs = grams_batch(ctx, gj, ld, n);
        uj.clear();
        for (size_t t = 0; t < res.size(); ++t) {
            const size_t g = res[t];
            for (double& x : gs[t]) x = -x;
            y2[g].alloc(static_cast<size_t>(p) * ld * sizeof(double));
            uj.push_back({1.0, ys[g], qa[g].as<double>(), k[g], gs[t], p, y2[g].as<double>()});
        }
        updates_batch(ctx, uj, ld, n);
        gj.clear();
        for (size_t g : res) gj.push_back({y2[g].as<double>(), p, y2[g].as<double>(), p});
        gs = grams_batch(ctx, gj, ld, n);
        std::vector<size_t> more;
        std::vector<int> k2(G, 0);
        uj.clear();
        for (size_t t = 0; t < res.size(); ++t) {
            const size_t g = res[t];
            std::vector<double> w2, v2;
            sym_eig_desc(p, gs[t], w2, v2);
            while (k2[g] < p - k[g] && w2[k2[g]] > 1e-24 * w0[g]) ++k2[g];
            if (k2[g] == 0) continue;
            uj.push_back({0.0, nullptr, y2[g].as<double>(), p, scaled_vectors(w2, v2, k2[g]), k2[g], q1[g].as<double>()});
            more.push_back(g);
        }
        updates_batch(ctx, uj, ld, n);
        if (!more.empty()) {  // re-orthogonalise against the first block, then CholeskyQR
            gj.clear();
            for (size_t g : more) gj.push_back({qa[g].as<double>(), k[g], q1[g].as<double>(), k2[g]});
            gs = grams_batch(ctx, gj, ld, n);
            uj.clear();
            for (size_t t = 0; t < more.size(); ++t) {
                const size_t g = more[t];
                for (double& x : gs[t]) x = -x;
                uj.push_back({1.0, q1[g].as<double>(), qa[g].as<double>(), k[g], gs[t], k2[g], y2[g].as<double>()});
            }
            updates_batch(ctx, uj, ld, n);
            std::vector<const double*> xs;
            std::vector<int> cols;
            std::vector<double*> outs;
            for (size_t g : more) {
                xs.push_back(y2[g].as<double>()), cols.push_back(k2[g]);
                outs.push_back(qa[g].as<double>() + static_cast<int64_t>(k[g]) * ld);
            }
            chol_qr(more, xs, cols, outs);
            for (size_t g : more) rank[g] += k2[g];
        }
    }
    q_out.resize(G);
    for (size_t g : live) q_out[g] = std::move(qa[g]);  // [rank][ld] (the buffer holds p columns)
    return rank;
}

// Hutch++ (proj/src/hutchpp.cpp:69-115) for groups [0, count) of a stack, seeded probes shared by all
// (every candidate of a feature-scoring step uses the same term seed). Callers guarantee the
// non-degenerate branch: 0 < s_q < n and s_g < n - s_q. errors[g] receives a candidate's failure.
std::vector<TraceEst> hutchpp_group(Context& ctx, const KernelMatrix& k, int count, const MatFun& f,
                                    const SketchCfg& cfg, std::vector<std::string>& errors, std::vector<int>& codes) {
    const int64_t n = k.n, gr = k.group_rows, ld = k.rpr;
    const int s_q = cfg.s_q, s_g = cfg.s_g, cost = f.query_cost();
    std::vector<TraceEst> est(count);
    auto replicate = [&](DevBuf& dst, int cols, const char* label) {
        DevBuf one;
        one.alloc(static_cast<size_t>(cols) * n * sizeof(double));
        if (ctx.probe_source == 1 && cfg.probe_kind == kProbeGaussian) {  // the reference's draws (host)
            const auto v = ctx.take_probes(n, cols, cfg.seed, label, cfg.probe_kind);
            h2d(ctx, one.as<double>(), v->data(), v->size() * sizeof(double));
            ctx.sync();
        } else {
            launched(ctx,
                     launch_rng_panel(derive_key(cfg.seed, hash_name(label)), true, cfg.probe_kind, 0, n, cols, 0,
                                      one.as<double>(), n, ctx.probe_err.as<int>(), ctx.stream()),
                     "rng_panel");
        }
        dst.alloc(static_cast<size_t>(cols) * ld * sizeof(double));
        cuda_check(cudaMemsetAsync(dst.as<void>(), 0, static_cast<size_t>(cols) * ld * sizeof(double), ctx.stream()),
                   "memset");
        for (int g = 0; g < count; ++g)
            cuda_check(cudaMemcpy2DAsync(dst.as<double>() + g * gr, ld * sizeof(double), one.as<double>(),
                                         n * sizeof(double), n * sizeof(double), cols, cudaMemcpyDeviceToDevice,
                                         ctx.stream()),
                       "replicate probes");
        ctx.sync();  // `one` is released at scope end; probe_err is read with the trace partials
    };
    // sketch products of every group in one pass: Y = A·S
    DevBuf sk, y;
    replicate(sk, s_q, "hutchpp-sketch");
    y.alloc(static_cast<size_t>(s_q) * ld * sizeof(double));
    for (int j0 = 0; j0 < s_q; j0 += kMaxPanelCols) {
        const int w = std::min(kMaxPanelCols, s_q - j0);
        run_panel(ctx, k, sk.as<double>() + static_cast<int64_t>(j0) * ld, ld, w, {{1.0, 0.0, 0.0}}, nullptr, nullptr,
                  y.as<double>() + static_cast<int64_t>(j0) * ld, ld);
    }
    std::vector<DevBuf> q;
    std::vector<const double*> ys(count);
    for (int g = 0; g < count; ++g) ys[g] = y.as<double>() + g * gr;
    const std::vector<int> rank = orthonormal_range_batch(ctx, ys, s_q, ld, n, q);  // per-candidate QR, batched
    int rmax = 0;
    for (int g = 0; g < count; ++g) {
        if (rank[g] == 0 && errors[g].empty()) {
            errors[g] = "hutchpp sketch A*S is numerically zero";
            codes[g] = kRankCollapse;
        }
        rmax = std::max(rmax, rank[g]);
    }
    // X0 = [Q_g (zero-padded to rmax columns) | W_g],  W_g = G - Q_g (Q_gᵀ G)
    const int cols = rmax + s_g;
    DevBuf gp, x0;
    replicate(gp, s_g, "hutchpp-probe");
    x0.alloc(static_cast<size_t>(cols) * ld * sizeof(double));
    cuda_check(cudaMemsetAsync(x0.as<void>(), 0, static_cast<size_t>(cols) * ld * sizeof(double), ctx.stream()),
               "memset");
    std::vector<GramJob> gj;
    std::vector<int> with_q;
    for (int g = 0; g < count; ++g) {
        double* xg = x0.as<double>() + g * gr;
        double* wg = xg + static_cast<int64_t>(rmax) * ld;
        const double* gg = gp.as<double>() + g * gr;
        if (rank[g] > 0) {
            cuda_check(cudaMemcpy2DAsync(xg, ld * sizeof(double), q[g].as<double>(), ld * sizeof(double),
                                         n * sizeof(double), rank[g], cudaMemcpyDeviceToDevice, ctx.stream()),
                       "copy Q");
            if (s_g > 0) {
                gj.push_back({q[g].as<double>(), rank[g], gg, s_g});
                with_q.push_back(g);
            }
        } else if (s_g > 0) {
            cuda_check(cudaMemcpy2DAsync(wg, ld * sizeof(double), gg, ld * sizeof(double), n * sizeof(double), s_g,
                                         cudaMemcpyDeviceToDevice, ctx.stream()),
                       "copy probes");
        }
    }
    {  // W_g = G - Q_g (Q_gᵀ G), batched
        std::vector<std::vector<double>> cs = grams_batch(ctx, gj, ld, n);
        std::vector<UpdateJob> uj;
        for (size_t t = 0; t < with_q.size(); ++t) {
            const int g = with_q[t];
            for (double& v : cs[t]) v = -v;
            uj.push_back({1.0, gp.as<double>() + g * gr, q[g].as<double>(), rank[g], std::move(cs[t]), s_g,
                          x0.as<double>() + g * gr + static_cast<int64_t>(rmax) * ld});
        }
        updates_batch(ctx, uj, ld, n);
    }
    // quadratic forms of every group by moment doubling (panel_traces), dots reduced per group
    const auto full = schedule(f);
    const int passes = (f.degree + 1) / 2;
    const std::vector<std::array<double, 3>> sched(full.begin(), full.begin() + passes);
    std::vector<std::vector<double>> tr(count, std::vector<double>(cols, 0.0));
    for (int j0 = 0; j0 < cols; j0 += kMaxPanelCols) {
        const int w = std::min(kMaxPanelCols, cols - j0);
        PanelSession ps(ctx, k, x0.as<double>() + static_cast<int64_t>(j0) * ld, ld, w, std::max(passes, 1), nullptr,
                        0.0, false);
        for (int p = 0; p < passes; ++p) ps.step(sched[p][0], sched[p][1], sched[p][2], 0.0);
        const int rg = static_cast<int>(gr / ps.rows_per_block());
        std::vector<double> mu(f.degree + 1);
        const std::vector<double> all = ps.dots_groups(0, passes, count, rg);
        const size_t per = static_cast<size_t>(passes + 1) * 3 * w;
        for (int g = 0; g < count; ++g) {
            PanelResult r;
            r.passes = passes;
            r.s = w;
            r.dots.assign(all.begin() + g * per, all.begin() + (g + 1) * per);
            for (int j = 0; j < w; ++j) {
                doubled_moments(f, r, j, mu.data());
                tr[g][j0 + j] = f.combine(mu.data(), 1);
            }
        }
    }
    for (int g = 0; g < count; ++g) {
        TraceEst& e = est[g];
        e.sketch_rank = rank[g];
        e.queries_used = s_q + rank[g] * cost + s_g * cost;
        double low = 0.0, res = 0.0;
        for (int j = 0; j < rank[g]; ++j) low += tr[g][j];
        for (int j = rmax; j < cols; ++j) res += tr[g][j];
        e.low_rank_part = low;
        e.residual_part = s_g > 0 ? res / s_g : 0.0;
        e.value = e.low_rank_part + e.residual_part;
    }
    return est;
}

// whether estimate() with these parameters runs as a grouped Hutch++ (no per-kernel power iteration,
// no exact branches, seeded probes)
bool group_eligible(Context& ctx, const KernelMatrix& k, const EstParams& p) {
    if (!ctx.feature_groups || k.prec != kF32 || ctx.world() != 1 || p.method == kMethodExact) return false;
    int ai = 0;
    if (!integer_alpha(p.alpha, &ai) && !p.has_bounds) return false;
    try {
        const Resolved r = resolve(ctx, k, p);
        const SketchCfg c = sketch_cfg(p, r.s);
        return c.s_q > 0 && c.s_q < k.n && c.s_g < k.n - c.s_q;
    } catch (const Error&) {
        return false;  // the sequential path raises the reference's error
    }
}

// estimate() (proj/src/entropy.cpp:201-275) for groups [0, count) of a stack
std::vector<EntropyEst> estimate_group(Context& ctx, const KernelMatrix& k, int count, const EstParams& p,
                                       std::vector<std::string>& errors, std::vector<int>& codes) {
    const Resolved r = resolve(ctx, k, p);
    const std::vector<TraceEst> tr = hutchpp_group(ctx, k, count, r.f, sketch_cfg(p, r.s), errors, codes);
    std::vector<EntropyEst> out(count);
    for (int g = 0; g < count; ++g) {
        if (!errors[g].empty()) continue;
        try {
            out[g] = entropy_of(tr[g], r.alpha, r.method, r.s, r.m_used);
            out[g].has_bounds = r.has_bounds;
            out[g].bounds_used = r.bounds;
        } catch (const Error& e) {
            errors[g] = e.what();
            codes[g] = e.code();
        }
    }
    return out;
}

bool features_finite(Context& ctx, const double* d_x, int64_t n, int64_t d) {
    ctx.small.ensure(4 * sizeof(unsigned));
    unsigned* flags = ctx.small.as<unsigned>();
    cuda_check(cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned), ctx.stream()), "memset");
    launched(ctx, launch_check_samples(d_x, n, static_cast<int>(d), 1, n, flags, ctx.stream()), "check_samples");
    unsigned hf[2];
    d2h(ctx, hf, flags, sizeof(hf));
    ctx.sync();
    float mx;
    std::memcpy(&mx, &hf[1], sizeof(float));
    return hf[0] == 0 && !(mx > 1e18f);
}

}  // namespace

namespace {

void validate_features(const FeatureData& data, int k) {  // features.cpp:18-26
    if (data.labels.empty()) fail(kInvalidArgument, "dataset has no label column");
    if (static_cast<int64_t>(data.labels.size()) != data.n) fail(kSizeMismatch, "label count does not match sample count");
    if (k < 1 || k > data.d)
        fail(kInvalidArgument, "k must be in [1, d]; got k=" + std::to_string(k) + " with d=" + std::to_string(data.d));
    if (data.ldx < data.n) fail(kInvalidArgument, "leading dimension smaller than the sample count");
}

// one_hot_labels (features.cpp:83-93): distinct labels in sorted order, column-major n x C
std::vector<double> one_hot(const std::vector<std::string>& labels, int* classes_out) {
    std::map<std::string, int> classes;
    for (const auto& l : labels) classes.emplace(l, 0);
    int idx = 0;
    for (auto& kv : classes) kv.second = idx++;
    const size_t n = labels.size();
    std::vector<double> e(n * classes.size(), 0.0);
    for (size_t i = 0; i < n; ++i) e[i + static_cast<size_t>(classes[labels[i]]) * n] = 1.0;
    *classes_out = idx;
    return e;
}

KernelPtr label_kernel(Context& ctx, const FeatureData& data, double sigma, int prec) {
    int c = 0;
    const std::vector<double> e = one_hot(data.labels, &c);
    return build_gaussian(ctx, e.data(), data.n, c, data.n, sigma, prec);
}

KernelPtr feature_kernel(Context& ctx, const FeatureData& data, const double* d_x, double sigma, int prec, int j) {
    try {  // features.cpp:33-39
        return build_gaussian_dev(ctx, d_x + static_cast<int64_t>(j) * data.n, data.n, 1, data.n, sigma, prec);
    } catch (const Error& e) {
        fail(e.code(), "feature '" + data.name(j) + "': " + e.what());
    }
}

struct StepScorer {  // features.cpp:44-75
    Context& ctx;
    const KernelMatrix& label;
    EstParams step;
    double label_entropy = 0.0;
    StepScorer(Context& c, const KernelMatrix& l, const EstParams& p, uint64_t step_seed) : ctx(c), label(l), step(p) {
        step.seed = step_seed;
        EstParams q = step;
        q.seed = derive_key(step_seed, hash_name("term:target"));
        label_entropy = estimate(ctx, label, q).entropy;
    }
    double score(const KernelMatrix& feats, const std::string& name) const {
        try {
            EstParams pv = step;
            pv.seed = derive_key(step.seed, hash_name("term:vars"));
            const double s_f = estimate(ctx, feats, pv).entropy;
            EstParams pj = step;
            pj.seed = derive_key(step.seed, hash_name("term:joint"));
            KernelPtr joint = hadamard_joint(ctx, feats, label);
            const double s_fy = estimate(ctx, *joint, pj).entropy;
            return s_f + label_entropy - s_fy;
        } catch (const Error& e) {
            fail(e.code(), "feature '" + name + "': " + e.what());
        }
    }
};

DevBuf upload_features(Context& ctx, const FeatureData& data) {
    DevBuf xs;
    xs.alloc(static_cast<size_t>(data.n) * data.d * sizeof(double));
    h2d_2d(ctx, xs.as<double>(), data.n * sizeof(double), data.x, data.ldx * sizeof(double), data.n * sizeof(double),
           data.d);
    return xs;
}

// Scores S(F) + S(Y) - S(F∘Y) (StepScorer::score) of candidates `cand` in stacks of up to
// group_capacity(n): build(stack, g, j) fills group g with candidate j's kernel F; the joints F∘Y are
// stacked beside them and each term is one grouped estimate. Errors surface for the first failing
// candidate in order, with the reference's "feature '<name>': " prefix.
template <typename Build>
void score_grouped(Context& ctx, const FeatureData& data, const KernelMatrix& label, const StepScorer& scorer,
                   const std::vector<int>& cand, Build&& build, std::vector<double>& sc, std::vector<double>* elapsed) {
    const int64_t n = data.n;
    const int cap = group_capacity(n);
    EstParams pv = scorer.step, pj = scorer.step;
    pv.seed = derive_key(scorer.step.seed, hash_name("term:vars"));
    pj.seed = derive_key(scorer.step.seed, hash_name("term:joint"));
    for (size_t c0 = 0; c0 < cand.size(); c0 += cap) {
        const auto t0 = std::chrono::steady_clock::now();
        const int cnt = static_cast<int>(std::min<size_t>(cap, cand.size() - c0));
        KernelPtr f = alloc_group(ctx, n, cnt), jk = alloc_group(ctx, n, cnt);
        for (int g = 0; g < cnt; ++g) {
            build(*f, g, cand[c0 + g]);
            group_hadamard(ctx, *jk, g, group_hi(*f, g), group_lo(*f, g), label.hi.as<__half>(), label.lo.as<__half>());
        }
        std::vector<std::string> ef(cnt), ej(cnt);
        std::vector<int> cf(cnt, 0), cj(cnt, 0);
        const std::vector<EntropyEst> sv = estimate_group(ctx, *f, cnt, pv, ef, cf);
        const std::vector<EntropyEst> sj = estimate_group(ctx, *jk, cnt, pj, ej, cj);
        for (int g = 0; g < cnt; ++g) {
            const int j = cand[c0 + g];
            if (!ef[g].empty()) fail(cf[g], "feature '" + data.name(j) + "': " + ef[g]);
            if (!ej[g].empty()) fail(cj[g], "feature '" + data.name(j) + "': " + ej[g]);
            sc[j] = sv[g].entropy + scorer.label_entropy - sj[g].entropy;
        }
        const double per = seconds_since(t0) / cnt;
        if (elapsed)
            for (int g = 0; g < cnt; ++g) (*elapsed)[cand[c0 + g]] = per;
    }
}

}  // namespace

FeatureRanking rank_features(Context& ctx, const FeatureData& data, double sigma, const EstParams& p, int prec, int k) {
    // features.cpp:95-123
    validate_features(data, k);
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    const int d = static_cast<int>(data.d);
    KernelPtr label = label_kernel(ctx, data, sigma, prec);
    DevBuf xs = upload_features(ctx, data);
    const StepScorer scorer(ctx, *label, p, derive_key(p.seed, 0));
    std::vector<double> scores(d), elapsed(d);
    if (group_eligible(ctx, *label, scorer.step) && features_finite(ctx, xs.as<double>(), data.n, d)) {
        std::vector<int> cand(d);
        for (int j = 0; j < d; ++j) cand[j] = j;
        const double* dx = xs.as<double>();
        score_grouped(ctx, data, *label, scorer, cand,
                      [&](const KernelMatrix& st, int g, int j) { group_gram(ctx, st, g, dx + j * data.n, sigma); },
                      scores, &elapsed);
    } else {
        for (int j = 0; j < d; ++j) {
            const auto t0 = std::chrono::steady_clock::now();
            KernelPtr f = feature_kernel(ctx, data, xs.as<double>(), sigma, prec, j);
            scores[j] = scorer.score(*f, data.name(j));
            elapsed[j] = seconds_since(t0);
        }
    }
    std::vector<int> order(d);
    for (int j = 0; j < d; ++j) order[j] = j;
    std::sort(order.begin(), order.end(), [&](int a, int b) {
        if (scores[a] != scores[b]) return scores[a] > scores[b];
        return a < b;
    });
    FeatureRanking res;
    res.elapsed = std::move(elapsed);
    for (int r = 0; r < k; ++r) {
        res.columns.push_back(order[r]);
        res.scores.push_back(scores[order[r]]);
    }
    return res;
}

FeatureSelection select_features(Context& ctx, const FeatureData& data, double sigma, const EstParams& p, int prec,
                                 int k) {
    // features.cpp:125-162
    validate_features(data, k);
    cuda_check(cudaSetDevice(ctx.device()), "cudaSetDevice");
    const int d = static_cast<int>(data.d);
    KernelPtr label = label_kernel(ctx, data, sigma, prec);
    std::vector<KernelPtr> kernels;
    {
        DevBuf xs = upload_features(ctx, data);
        for (int j = 0; j < d; ++j) kernels.push_back(feature_kernel(ctx, data, xs.as<double>(), sigma, prec, j));
        ctx.sync();
    }
    FeatureSelection res;
    std::vector<bool> taken(d, false);
    KernelPtr selected;  // running Hadamard product of the picks
    const bool grouped = group_eligible(ctx, *label, p);  // every step's estimates as grouped stacks
    for (int step = 0; step < k; ++step) {
        const auto t0 = std::chrono::steady_clock::now();
        const StepScorer scorer(ctx, *label, p, derive_key(p.seed, static_cast<uint64_t>(step)));
        int best = -1;
        double best_score = 0.0;
        KernelPtr best_joint;
        if (grouped) {  // candidates' kernels (step 0) or joints with the picks so far, stacked
            std::vector<int> cand;
            for (int j = 0; j < d; ++j)
                if (!taken[j]) cand.push_back(j);
            std::vector<double> sc(d, 0.0);
            score_grouped(ctx, data, *label, scorer, cand,
                          [&](const KernelMatrix& st, int g, int j) {
                              if (step == 0) {
                                  const size_t bytes = static_cast<size_t>(data.n) * st.ld * sizeof(__half);
                                  cuda_check(cudaMemcpyAsync(group_hi(st, g), kernels[j]->hi.as<__half>(), bytes,
                                                             cudaMemcpyDeviceToDevice, ctx.stream()), "copy kernel");
                                  cuda_check(cudaMemcpyAsync(group_lo(st, g), kernels[j]->lo.as<__half>(), bytes,
                                                             cudaMemcpyDeviceToDevice, ctx.stream()), "copy kernel");
                              } else {
                                  group_hadamard(ctx, st, g, selected->hi.as<__half>(), selected->lo.as<__half>(),
                                                 kernels[j]->hi.as<__half>(), kernels[j]->lo.as<__half>());
                              }
                          },
                          sc, nullptr);
            for (int j : cand) {  // first maximum in column order (features.cpp:140-152)
                if (best < 0 || sc[j] > best_score) {
                    best = j;
                    best_score = sc[j];
                }
            }
            if (step > 0) best_joint = hadamard_joint(ctx, *selected, *kernels[best]);
        } else {
            for (int j = 0; j < d; ++j) {
                if (taken[j]) continue;
                KernelPtr cand = step == 0 ? nullptr : hadamard_joint(ctx, *selected, *kernels[j]);
                const KernelMatrix& cm = step == 0 ? *kernels[j] : *cand;
                const double sc = scorer.score(cm, data.name(j));
                if (best < 0 || sc > best_score) {
                    best = j;
                    best_score = sc;
                    best_joint = std::move(cand);
                }
            }
        }
        taken[best] = true;
        if (step == 0)
            selected = std::move(kernels[best]);  // the first pick's own kernel (no longer a candidate)
        else
            selected = std::move(best_joint);
        res.columns.push_back(best);
        res.objective.push_back(best_score);
        res.elapsed.push_back(seconds_since(t0));
    }
    return res;
}

}  // namespace rb
