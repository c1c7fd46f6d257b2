// Host engine: device context, device-resident kernel matrices, and the
// estimator pipeline (recurrence passes, power iteration, Hutch++, estimate,
// mutual information) driving the sm_100a kernels. This is the C++ host surface
// that mirrors the reference library (proj/include/renyi/*.hpp); the C ABI in
// include/renyi_b200.h wraps it.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <future>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "host_math.h"
#include "kernels.h"

namespace rb {

// NVTX range around one pass, collective or estimator phase (header-only NVTX v3: a no-op unless a
// profiler injects its handler, so the ranges stay compiled in)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// kF64: fp64 A; kF32: A as fp16 hi/lo planes (fp32-class); kMF: matrix-free (bf16 samples, A never stored)
enum Precision : int { kF64 = 0, kF32 = 1, kMF = 2 };

void cuda_check(cudaError_t e, const char* what);

// Device memory comes from a process-wide caching pool (per device): n x n kernel
// storage, panels and scratch are reused across estimates instead of paying
// cudaMalloc/cudaFree (which synchronise the device) inside the estimator loop.
// Blocks are stream-ordered: a block freed while the thread's current engine stream may
// still have queued work is handed to another stream only behind an event recorded at the
// free (cudaStreamWaitEvent), so ranks / contexts on other streams never race on it.
void* pool_alloc(size_t bytes, size_t* capacity, int* device);
void pool_free(void* p, size_t capacity, int device);
void pool_release_all();  // returns every cached block to the driver
// the engine stream of the calling thread (set by Context::stream(); tags pool frees)
void set_current_stream(cudaStream_t s);

class DevBuf {
public:
    DevBuf() = default;
    ~DevBuf();
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), cap_(o.cap_), dev_(o.dev_) { o.p_ = nullptr, o.n_ = 0, o.cap_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept;
    void alloc(size_t bytes);
    void ensure(size_t bytes);  // grow-only
    void release();
    template <typename T>
    T* as() const {
        return static_cast<T*>(p_);
    }
    size_t bytes() const { return n_; }

private:
    void* p_ = nullptr;
    size_t n_ = 0;
    size_t cap_ = 0;
    int dev_ = 0;
};

// Multi-rank exchange (row-sharded A). Context::exchange == nullptr: one rank.
struct Exchange {
    virtual ~Exchange() = default;
    virtual int rank() const = 0;
    virtual int world() const = 0;
    // buf holds `world` chunks of chunk_bytes; this rank's chunk (index rank) is in place
    virtual void allgather_inplace(void* buf, size_t chunk_bytes, cudaStream_t s) = 0;
    virtual void allreduce_sum_f64(double* buf, size_t count, cudaStream_t s) = 0;
    virtual void allreduce_max_u32(unsigned* buf, size_t count, cudaStream_t s) = 0;
};

struct LocalGroup;
std::shared_ptr<LocalGroup> make_local_group(int world);
std::unique_ptr<Exchange> make_local_exchange(std::shared_ptr<LocalGroup> g, int rank);
void nccl_unique_id(unsigned char* out128);
std::unique_ptr<Exchange> make_nccl_exchange(int rank, int world, const unsigned char* id128);

// Row shard of rank `rank` out of `world` for n rows: chunks of rpr rows (rpr a multiple of 256),
// the last chunk shorter. world == 1: row0 = 0, rows = n, rpr = round_up(n, 256).
void shard_rows(int64_t n, int world, int rank, int64_t* row0, int64_t* rows, int64_t* rpr);

// device buffers of one panel session (recurrence state, operand planes, partials, reductions)
struct PanelWorkspace {
    DevBuf partial, partial2, stats, red, cmax, eexp;  // partial2: second K window (row-sharded passes)
    DevBuf state[4], vhi, vlo;
};

class Context {
public:
    explicit Context(int device);
    ~Context();
    int device() const { return device_; }
    cudaStream_t stream() const {
        set_current_stream(stream_);
        return stream_;
    }
    int sms() const { return sms_; }
    void sync();
    // row-sharded passes: the operand all-gather (and the column-maxima all-reduce) run on a second
    // stream, overlapped with the product over the rank's own operand chunk (created on first use)
    cudaStream_t comm_stream();
    void comm_after_main();  // comm stream waits for the work queued so far on the engine stream
    void main_after_comm();  // engine stream waits for the collectives queued so far on the comm stream

    // tuning knobs of the block product
    int grid = 0;  // CTAs of the persistent stream-K kernel (0 = SM count)
    int kc = 16;   // k tiles (x32 columns) per TMEM accumulation chunk
    int mf_kc = 8;  // matrix-free: j-blocks (x128 samples) per TMEM accumulation chunk
    // iterate operand of the fp32 block product: 0 split (default; V as fp16 hi+lo, 3 MMAs),
    // 1 fast (V hi only, 2 MMAs), 2 auto (split where product vectors leave the panel:
    // block_product, apply_panel, the Hutch++ sketch; fast for trace-only passes). Measured
    // trace errors against the oracle: split <= 4e-6, fast / auto up to 2.5e-4 at small probe
    // counts, so only split keeps the 1e-4 fp32 bar everywhere.
    int operand_mode = 0;

    // instrumentation: CUDA-event timing of every block-product launch
    void prof_enable(bool on);
    void prof_begin();
    void prof_end();
    void prof_account(double bytes, double flops);
    // synchronizes; returns launches, summed device milliseconds, algorithmic bytes and flops since enable
    void prof_read(int* launches, double* ms, double* bytes, double* flops);
    long launches = 0;  // kernels launched by the engine (all kinds)
    long long h2d_bytes = 0, d2h_bytes = 0;  // host<->device traffic issued by the engine

    // region timer (CUDA events on the engine stream)
    void timer_begin();
    double timer_end_ms();  // synchronizes

    std::unique_ptr<Exchange> exchange;
    int rank() const { return exchange ? exchange->rank() : 0; }
    int world() const { return exchange ? exchange->world() : 1; }

    // scratch (grow-only)
    PanelWorkspace ws;         // the panel session's buffers
    PanelWorkspace ws_aux[2];  // the second and third operand of a fused mutual-information pass
    bool fused_mi = true;      // mutual information: one pass over A and B for all three terms
    bool feature_groups = true;  // feature tools: candidates' estimates as grouped stacks (fp32)
    // single-column fp32 passes (power iteration, matvec) through the upper-triangle product (symv.cu);
    // RB_SYMV=0 in the environment selects the tensor-core block product for A/B comparisons
    bool symv = true;
    // power iteration: queue pass it+1 behind pass it's dots (its 1/||T|| computed on the device) so the
    // host's readback and convergence test overlap the next product; RB_SPECULATE=0 turns it off
    bool speculate = true;
    // page-locked landing slots for per-pass dots read back without a stream synchronize (grow-only)
    double* pinned_dots(size_t count);
    cudaEvent_t dots_event(int i);  // i in {0, 1}
    // source of seeded Gaussian probes (Rademacher probes are exact on the device either way):
    // 0 device (rng_panel: the reference's substreams with CUDA's log/sin/cos, <= 2 ulp from glibc per
    // draw), 1 host (the reference's own stream arithmetic, bitwise the probes of
    // proj/src/hutchpp.cpp:13-22, generated on the host's threads and copied; mutual information
    // requests its six panels before the kernel builds so the host work overlaps them)
    int probe_source = 0;
    struct ProbeReq {
        int64_t n;
        int cols;
        uint64_t seed;
        std::string label;
        int kind;
    };
    // starts generating the panels on the host threads, columns handed out in request order
    void prefetch_probes(const std::vector<ProbeReq>& reqs);
    std::shared_ptr<std::vector<double>> take_probes(int64_t n, int cols, uint64_t seed, const char* label, int kind);
    void drop_prefetched_probes();  // waits for unused panels, frees them
    DevBuf gram_partial, small, probe_err, gram_ticket;
    DevBuf x0, work, acc;

private:
    int device_ = 0;
    cudaStream_t stream_ = nullptr;
    int sms_ = 148;
    bool prof_ = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> events_;
    size_t prof_used_ = 0;
    double prof_bytes_ = 0.0, prof_flops_ = 0.0;
    cudaEvent_t t0_ = nullptr, t1_ = nullptr;
    cudaStream_t comm_ = nullptr;
    cudaEvent_t ev_main_ = nullptr, ev_comm_ = nullptr;
    double* pin_dots_ = nullptr;
    size_t pin_cap_ = 0;
    cudaEvent_t dots_ev_[2] = {nullptr, nullptr};
    // requested panels, generated one after another in request order (each on all host threads)
    using Panel = std::shared_ptr<std::vector<double>>;
    std::map<std::string, std::shared_future<Panel>> probe_prefetch_;
    std::future<void> probe_job_;
};

struct KernelMatrix {
    int64_t n = 0;      // samples (columns)
    int64_t row0 = 0;   // first row held by this rank
    int64_t rows = 0;   // rows held by this rank
    int64_t rpr = 0;    // rows per rank chunk (multiple of 256)
    int world = 1, rank = 0;
    int64_t ld = 0;     // row pitch (elements)
    int prec = kF32;
    double unscale = 1.0;  // A = stored * unscale (split planes)
    double a_norm = 1.0;   // >= max_i sum_j |A_ij|
    bool normalized = true;
    DevBuf a64, hi, lo;
    // matrix-free storage
    DevBuf xb, xa;  // bf16 [npad][dp] samples, bf16 [2][npad][16] augmented columns (−|x|²/2)
    int dp = 0;
    int dfeat = 0;  // true feature count (algorithmic flops)
    double c2 = 0.0;  // log2(e)/σ²
    // grouped stack (feature tools): `groups` n x n kernels of the same n in one allocation, group g in
    // rows [g·group_rows, g·group_rows + n) (rows past n zero), padded to whole CTA-pair blocks per
    // pair of a `group_grid`-CTA product so every row block is computed whole by one pair
    int groups = 1;
    int64_t group_rows = 0;
    int group_grid = 0;
};

using KernelPtr = std::unique_ptr<KernelMatrix>;

// ---- kernel construction (proj/src/kernel.cpp) ----
// x: host column-major n x d (Eigen layout of the reference), ld >= n.
KernelPtr build_gaussian(Context& ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double sigma, int prec,
                         const double* y = nullptr, int64_t dy = 0, int64_t ldy = 0, double sigma_y = 1.0);
// build_kernel(X, PolynomialKernel{degree, offset}) (kernel.cpp:35-72, ops.cpp:22-28,58-64), host or device samples
KernelPtr build_polynomial(Context& ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int degree, double offset,
                           int prec);
KernelPtr build_polynomial_dev(Context& ctx, const double* d_x, int64_t n, int64_t d, int64_t ldx, int degree,
                               double offset, int prec);
// the raw ops seam (proj/include/renyi/ops.hpp:12-33), host matrices in and out (column-major):
// K = gaussian_gram(X, sigma) / polynomial_gram(X, degree, offset) (n x n, single rank), and
// C = hadamard_scaled(A, B, scale) over rows x cols
void ops_gaussian_gram(Context& ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double sigma, double* k);
void ops_polynomial_gram(Context& ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int degree, double offset,
                         double* k);
void ops_hadamard_scaled(Context& ctx, const double* a, const double* b, int64_t rows, int64_t cols, double scale,
                         double* c);
// device-resident samples (column-major, leading dimension ld)
KernelPtr build_gaussian_dev(Context& ctx, const double* d_x, int64_t n, int64_t d, int64_t ldx, double sigma,
                             int prec, const double* d_y = nullptr, int64_t dy = 0, int64_t ldy = 0,
                             double sigma_y = 1.0);
KernelPtr from_matrix(Context& ctx, const double* a, int64_t n, int prec);

// ---- CSV ingestion (renyi::load_csv, proj/src/csv.cpp:63-115; csv.cu) ----
// Dataset (proj/include/renyi/features.hpp:12-19) with the features resident on the device.
struct Dataset {
    int64_t n = 0, d = 0;
    DevBuf features;  // n x d, column-major fp64
    std::vector<std::string> names, labels;
};
// text: the file's bytes (host); source names the input in messages ('path': ...)
std::unique_ptr<Dataset> load_csv_text(Context& ctx, const char* text, size_t len, const char* label_column,
                                       const std::string& source);
std::unique_ptr<Dataset> load_csv_file(Context& ctx, const std::string& path, const char* label_column);
KernelPtr hadamard_joint(Context& ctx, const KernelMatrix& a, const KernelMatrix& b);
// hadamard_joint of any number of kernels (kernel.cpp:74-101): canonical content order, one scale
KernelPtr hadamard_joint_n(Context& ctx, const std::vector<const KernelMatrix*>& ks);
void download(Context& ctx, const KernelMatrix& k, double* out_colmajor);

// ---- passes ----
struct PanelResult {
    int passes = 0;
    int s = 0;
    std::vector<double> dots;  // [(passes+1)][3][s]: x0·T_k, T_{k-1}·T_k, T_k·T_k
    double dot(int k, int q, int j) const { return dots[(static_cast<size_t>(k) * 3 + q) * s + j]; }
};

// Runs T_0 = X (device fp64 [s][ldx]) through `coeffs.size()` passes.
// acc_coef (optional, size passes+1): acc = sum_k acc_coef[k] T_k into acc_out (device fp64 [s][ldo]).
// last_out (optional): T_passes as fp64 [s][ldo].
PanelResult run_panel(Context& ctx, const KernelMatrix& k, const double* x, int64_t ldx, int s,
                      const std::vector<std::array<double, 3>>& coeffs, const std::vector<double>* acc_coef = nullptr,
                      double* acc_out = nullptr, double* last_out = nullptr, int64_t ldo = 0);

// Y = A V for host panels (ops::matmul_panel seam)
void block_product(Context& ctx, const KernelMatrix& k, const double* v, int s, double* y);
// f(A) V for host panels (apply_panel seam)
void apply_panel(Context& ctx, const KernelMatrix& k, const MatFun& f, const double* v, int s, double* y);
// per-column x_j^T f(A) x_j, host panel
void matfun_traces(Context& ctx, const KernelMatrix& k, const MatFun& f, const double* x, int s, double* out);

// ---- spectrum (proj/src/spectrum.cpp) ----
struct PowerOpts {
    int max_iters = 100;
    double tol = 1e-6;
    uint64_t seed = 0;
    double rank_floor = 1e-12;
};
struct PowerRes {
    double rayleigh = 0.0;
    int iterations = 0;
    bool converged = false;
};
PowerRes power_method(Context& ctx, const KernelMatrix& k, const PowerOpts& o, double shift);
SpectrumBoundsH estimate_bounds(Context& ctx, const KernelMatrix& k, const PowerOpts& o);

// ---- Hutch++ (proj/src/hutchpp.cpp) ----
struct SketchCfg {
    int s_q = 0, s_g = 0;
    uint64_t seed = 0;
    int probe_kind = kProbeGaussian;
    const double* sketch = nullptr;  // optional host n x s_q
    const double* probes = nullptr;  // optional host n x s_g
};
struct TraceEst {
    double value = 0.0, low_rank_part = 0.0, residual_part = 0.0;
    int queries_used = 0, sketch_rank = 0;
    bool exact = false;
};
TraceEst hutchpp(Context& ctx, const KernelMatrix& k, const MatFun& f, const SketchCfg& cfg);

// ---- estimators (proj/src/entropy.cpp, proj/src/measures.cpp) ----
struct EstParams {
    double alpha = 2.0;
    int method = kMethodAuto;
    int s = 0, m = 0;
    double epsilon = 1e-2, delta = 1e-2;
    uint64_t seed = 0;
    PowerOpts power;
    bool has_bounds = false;
    SpectrumBoundsH bounds;
    int probe_kind = kProbeGaussian;
    int s_q = -1, s_g = -1;  // explicit split; -1 = reference split floor(s/4), s-2floor(s/4)
};
struct EntropyEst {
    double entropy = 0.0, trace_estimate = 0.0;
    int method_used = kMethodExact, s_used = 0, m_used = 0;
    bool has_bounds = false;
    SpectrumBoundsH bounds_used;
    double elapsed = 0.0;
    bool deterministic = false;
    TraceEst trace;
};
EntropyEst estimate(Context& ctx, const KernelMatrix& k, const EstParams& p);

// ---- batched trials (proj/src/simulate.cpp:19-72) ----
// trials of estimate() with seeds derive_key(p.seed, t), bounds resolved once, probes of all
// trials sharing the passes over A
std::vector<EntropyEst> estimate_trials(Context& ctx, const KernelMatrix& k, const EstParams& p, int trials);
struct MreCell {
    double alpha = 0.0;
    int s = 0, m = 0, method = kMethodExact;
    double mre = 0.0, sd = 0.0, mean_elapsed = 0.0;
    int trials = 0;
};
MreCell measure_cell(Context& ctx, const KernelMatrix& k, double exact_entropy, const EstParams& p, int trials);

// ---- feature tools (proj/src/features.cpp) ----
struct FeatureData {
    const double* x = nullptr;  // host n x d, column-major, leading dimension ldx
    int64_t n = 0, d = 0, ldx = 0;
    std::vector<std::string> labels, names;
    std::string name(int j) const;
};
struct FeatureRanking {
    std::vector<int> columns;       // top-k, scores non-increasing, ties by ascending column
    std::vector<double> scores;     // I_alpha(X_j; Y)
    std::vector<double> elapsed;    // seconds per scored feature (all d)
};
struct FeatureSelection {
    std::vector<int> columns;       // greedy pick order
    std::vector<double> objective;  // I_alpha(S; Y) after each addition
    std::vector<double> elapsed;    // seconds per greedy step
};
FeatureRanking rank_features(Context& ctx, const FeatureData& data, double sigma, const EstParams& p, int prec, int k);
FeatureSelection select_features(Context& ctx, const FeatureData& data, double sigma, const EstParams& p, int prec,
                                 int k);

struct MutualInfo {
    double value = 0.0, vars_entropy = 0.0, target_entropy = 0.0, joint_entropy = 0.0;
};
MutualInfo mutual_information(Context& ctx, const KernelMatrix& a, const KernelMatrix& b, const EstParams& p);
// memory-lean MI straight from samples: one n x n matrix resident at a time
MutualInfo mutual_information_samples(Context& ctx, const double* x, int64_t n, int64_t dx, int64_t ldx,
                                      double sigma_x, const double* y, int64_t dy, int64_t ldy, double sigma_y,
                                      const EstParams& p, int prec);
MutualInfo mutual_information_samples_dev(Context& ctx, const double* d_x, int64_t n, int64_t dx, int64_t ldx,
                                          double sigma_x, const double* d_y, int64_t dy, int64_t ldy,
                                          double sigma_y, const EstParams& p, int prec);
EstParams with_seed(const EstParams& p, const char* term);

// counted host<->device copies on the engine stream
void h2d(Context& ctx, void* dst, const void* src, size_t bytes);
// large contiguous uploads from pageable memory: page-locked double buffering, several host threads
void h2d_staged(Context& ctx, void* dst, const void* src, size_t bytes);
void d2h(Context& ctx, void* dst, const void* src, size_t bytes);
void h2d_2d(Context& ctx, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height);
void d2h_2d(Context& ctx, void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height);

}  // namespace rb
