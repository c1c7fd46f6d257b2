// Multi-rank exchange backends for the row-sharded path.
//
//   * NcclExchange — one process per GPU, NCCL over NVLink/NVSwitch: an in-place
//     all-gather of the next fp16 operand planes per pass, a max all-reduce of the
//     per-column maxima (so every rank picks the same plane scale), and a sum
//     all-reduce of the fp64 trace partials / CholeskyQR2 Grams. libnccl is opened
//     at run time (no link-time dependency for single-GPU users).
//   * LocalGroupExchange — ranks as host threads of one process (one Context each,
//     any devices, including several ranks on one GPU for validation). Collectives
//     are host-driven: every rank synchronises its stream, the threads meet at a
//     barrier and copy with blocking cudaMemcpy, so no kernel ever waits on another.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "engine.h"

namespace rb {

// ---------------------------------------------------------------- local group
struct LocalGroup {
    explicit LocalGroup(int w) : world(w), ptrs(w, nullptr) {}
    int world;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long generation = 0;
    std::vector<void*> ptrs;

    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

namespace {

class LocalGroupExchange : public Exchange {
public:
    LocalGroupExchange(std::shared_ptr<LocalGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}
    int rank() const override { return rank_; }
    int world() const override { return g_->world; }

    void allgather_inplace(void* buf, size_t chunk, cudaStream_t s) override {
        NvtxRange nvtx("local group all-gather");
        cuda_check(cudaStreamSynchronize(s), "local group: stream sync");
        g_->ptrs[rank_] = buf;
        g_->barrier();
        for (int q = 0; q < g_->world; ++q) {
            if (q == rank_) continue;
            cuda_check(cudaMemcpy(static_cast<char*>(buf) + q * chunk, static_cast<char*>(g_->ptrs[q]) + q * chunk,
                                  chunk, cudaMemcpyDefault),
                       "local group: all-gather copy");
        }
        g_->barrier();
    }

    void allreduce_sum_f64(double* buf, size_t count, cudaStream_t s) override {
        reduce(buf, count * sizeof(double), s, [&](const std::vector<std::vector<char>>& all, void* out) {
            double* o = static_cast<double*>(out);
            for (size_t i = 0; i < count; ++i) {
                double acc = 0.0;
                for (const auto& v : all) acc += reinterpret_cast<const double*>(v.data())[i];  // rank order
                o[i] = acc;
            }
        });
    }

    void allreduce_max_u32(unsigned* buf, size_t count, cudaStream_t s) override {
        reduce(buf, count * sizeof(unsigned), s, [&](const std::vector<std::vector<char>>& all, void* out) {
            unsigned* o = static_cast<unsigned*>(out);
            for (size_t i = 0; i < count; ++i) {
                unsigned m = 0;
                for (const auto& v : all) m = std::max(m, reinterpret_cast<const unsigned*>(v.data())[i]);
                o[i] = m;
            }
        });
    }

private:
    template <typename F>
    void reduce(void* buf, size_t bytes, cudaStream_t s, F&& combine) {
        NvtxRange nvtx("local group all-reduce");
        cuda_check(cudaStreamSynchronize(s), "local group: stream sync");
        g_->ptrs[rank_] = buf;
        g_->barrier();
        std::vector<std::vector<char>> all(g_->world, std::vector<char>(bytes));
        for (int q = 0; q < g_->world; ++q)
            cuda_check(cudaMemcpy(all[q].data(), g_->ptrs[q], bytes, cudaMemcpyDefault), "local group: read");
        g_->barrier();  // everyone has read every buffer before anyone overwrites its own
        std::vector<char> out(bytes);
        combine(all, out.data());
        cuda_check(cudaMemcpy(buf, out.data(), bytes, cudaMemcpyDefault), "local group: write");
    }

    std::shared_ptr<LocalGroup> g_;
    int rank_;
};

// ---------------------------------------------------------------- NCCL
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        return a;
    }();
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.all_reduce)
        fail(kNcclError, "libnccl.so.2 could not be loaded");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    const char* msg = nccl().error_string ? nccl().error_string(r) : "?";
    fail(kNcclError, std::string(what) + ": " + msg);
}

class NcclExchange : public Exchange {
public:
    NcclExchange(int rank, int world, const unsigned char* id) : rank_(rank), world_(world) {
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        nccl_check(nccl().comm_init_rank(&comm_, world, uid, rank), "ncclCommInitRank");
    }
    ~NcclExchange() override {
        if (comm_ && nccl().comm_destroy) nccl().comm_destroy(comm_);
    }
    int rank() const override { return rank_; }
    int world() const override { return world_; }
    void allgather_inplace(void* buf, size_t chunk, cudaStream_t s) override {
        NvtxRange nvtx("ncclAllGather");
        nccl_check(nccl().all_gather(static_cast<char*>(buf) + rank_ * chunk, buf, chunk, ncclUint8, comm_, s),
                   "ncclAllGather");
    }
    void allreduce_sum_f64(double* buf, size_t count, cudaStream_t s) override {
        NvtxRange nvtx("ncclAllReduce sum");
        nccl_check(nccl().all_reduce(buf, buf, count, ncclFloat64, ncclSum, comm_, s), "ncclAllReduce");
    }
    void allreduce_max_u32(unsigned* buf, size_t count, cudaStream_t s) override {
        NvtxRange nvtx("ncclAllReduce max");
        nccl_check(nccl().all_reduce(buf, buf, count, ncclUint32, ncclMax, comm_, s), "ncclAllReduce");
    }

private:
    int rank_, world_;
    ncclComm_t comm_ = nullptr;
};

}  // namespace

std::shared_ptr<LocalGroup> make_local_group(int world) {
    if (world < 1) fail(kInvalidArgument, "local group needs world >= 1");
    return std::make_shared<LocalGroup>(world);
}

std::unique_ptr<Exchange> make_local_exchange(std::shared_ptr<LocalGroup> g, int rank) {
    if (rank < 0 || rank >= g->world) fail(kInvalidArgument, "rank out of range");
    return std::make_unique<LocalGroupExchange>(std::move(g), rank);
}

void nccl_unique_id(unsigned char* out) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId uid;
    nccl_check(nccl().get_unique_id(&uid), "ncclGetUniqueId");
    std::memcpy(out, &uid, sizeof(uid));
}

std::unique_ptr<Exchange> make_nccl_exchange(int rank, int world, const unsigned char* id) {
    if (world < 1 || rank < 0 || rank >= world) fail(kInvalidArgument, "bad rank/world");
    return std::make_unique<NcclExchange>(rank, world, id);
}

}  // namespace rb
