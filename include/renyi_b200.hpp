// renyi_b200.hpp — header-only C++ mirror of the reference library's host surface
// (proj/include/renyi/*.hpp) over the C ABI in renyi_b200.h. Names, argument
// meaning and error behaviour follow the reference: failures throw
// renyi::gpu::error carrying the reference's errc kind (is_usage() splits CLI
// exit 2 / 3 as in proj/include/renyi/common.hpp:27-48). Matrices are
// column-major like Eigen::MatrixXd; the kernel matrix lives on the device.
//
//   renyi::gpu::Context ctx(0);
//   auto k = renyi::gpu::build_kernel(ctx, X, renyi::gpu::GaussianKernel{sigma});
//   renyi::gpu::EstimatorParams p; p.alpha = 1.5; p.method = renyi::gpu::Method::chebyshev; ...
//   renyi::gpu::EntropyEstimate e = renyi::gpu::estimate(ctx, k, p);
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "renyi_b200.h"

namespace renyi::gpu {

enum class errc {  // proj/include/renyi/common.hpp:14-25, + device kinds
    invalid_argument = RENYI_E_INVALID_ARGUMENT,
    zero_diagonal = RENYI_E_ZERO_DIAGONAL,
    non_finite = RENYI_E_NON_FINITE,
    size_mismatch = RENYI_E_SIZE_MISMATCH,
    domain_error = RENYI_E_DOMAIN_ERROR,
    rank_collapse = RENYI_E_RANK_COLLAPSE,
    non_positive_trace = RENYI_E_NON_POSITIVE_TRACE,
    alpha_is_one = RENYI_E_ALPHA_IS_ONE,
    degenerate_bounds = RENYI_E_DEGENERATE_BOUNDS,
    parse_error = RENYI_E_PARSE_ERROR,
    cuda_error = RENYI_E_CUDA,
    nccl_error = RENYI_E_NCCL,
    out_of_memory = RENYI_E_OOM,
    no_device = RENYI_E_NO_DEVICE,
    internal = RENYI_E_INTERNAL,
};

class error : public std::runtime_error {
public:
    error(errc kind, const std::string& what) : std::runtime_error(what), kind_(kind) {}
    errc kind() const noexcept { return kind_; }
    bool is_usage() const noexcept { return renyi_status_is_usage(static_cast<int>(kind_)) != 0; }

private:
    errc kind_;
};

inline void check(int status) {
    if (status != RENYI_OK) throw error(static_cast<errc>(status), renyi_last_error());
}

// Column-major dense matrix (Eigen::MatrixXd layout).
struct Matrix {
    int64_t rows = 0, cols = 0;
    std::vector<double> data;
    Matrix() = default;
    Matrix(int64_t r, int64_t c, double v = 0.0) : rows(r), cols(c), data(static_cast<size_t>(r * c), v) {}
    double& operator()(int64_t i, int64_t j) { return data[static_cast<size_t>(i + j * rows)]; }
    double operator()(int64_t i, int64_t j) const { return data[static_cast<size_t>(i + j * rows)]; }
};

enum class Precision { fp64 = RENYI_F64, fp32 = RENYI_F32 };
enum class Method { exact = RENYI_METHOD_EXACT, int_power = RENYI_METHOD_INT, taylor = RENYI_METHOD_TAYLOR,
                    chebyshev = RENYI_METHOD_CHEBYSHEV, auto_select = RENYI_METHOD_AUTO };

class Context {
public:
    explicit Context(int device = 0) {
        renyi_ctx* c = nullptr;
        check(renyi_ctx_create(device, &c));
        h_.reset(c);
    }
    renyi_ctx* get() const { return h_.get(); }
    // RENYI_PROBES_DEVICE (default) or RENYI_PROBES_HOST (bitwise the reference's Gaussian probes)
    void set_probe_source(int source) const { check(renyi_ctx_set_probe_source(get(), source)); }

private:
    struct Del {
        void operator()(renyi_ctx* c) const { renyi_ctx_destroy(c); }
    };
    std::unique_ptr<renyi_ctx, Del> h_;
};

struct GaussianKernel {  // proj/include/renyi/kernel.hpp:12-14
    double sigma = 1.0;
};

struct PolynomialKernel {  // proj/include/renyi/kernel.hpp:16-19
    int degree = 2;
    double offset = 1.0;
};

using KernelSpec = std::variant<GaussianKernel, PolynomialKernel>;  // kernel.hpp:22

// NormalizedKernel (proj/include/renyi/kernel.hpp:27-42), device resident.
class NormalizedKernel {
public:
    NormalizedKernel() = default;
    explicit NormalizedKernel(renyi_kernel* k) : h_(k, Del{}) {}
    renyi_kernel* get() const { return h_.get(); }
    int64_t size() const {
        int64_t n = 0;
        check(renyi_kernel_size(h_.get(), &n));
        return n;
    }
    Matrix matrix(const Context& ctx) const {
        const int64_t n = size();
        Matrix a(n, n);
        check(renyi_kernel_download(ctx.get(), h_.get(), a.data.data()));
        return a;
    }

private:
    struct Del {
        void operator()(renyi_kernel* k) const { renyi_kernel_destroy(k); }
    };
    std::shared_ptr<renyi_kernel> h_{nullptr, Del{}};
};

inline NormalizedKernel build_kernel(const Context& ctx, const Matrix& samples, const GaussianKernel& spec,
                                     Precision prec = Precision::fp64) {  // kernel.cpp:35-72
    renyi_kernel* k = nullptr;
    check(renyi_kernel_build_gaussian(ctx.get(), samples.data.data(), samples.rows, samples.cols, samples.rows,
                                      spec.sigma, static_cast<int>(prec), &k));
    return NormalizedKernel(k);
}

inline NormalizedKernel build_kernel(const Context& ctx, const Matrix& samples, const PolynomialKernel& spec,
                                     Precision prec = Precision::fp64) {  // kernel.cpp:35-72, ops.cpp:22-28
    renyi_kernel* k = nullptr;
    check(renyi_kernel_build_polynomial(ctx.get(), samples.data.data(), samples.rows, samples.cols, samples.rows,
                                        spec.degree, spec.offset, static_cast<int>(prec), &k));
    return NormalizedKernel(k);
}

inline NormalizedKernel build_kernel(const Context& ctx, const Matrix& samples, const KernelSpec& spec,
                                     Precision prec = Precision::fp64) {
    return std::visit([&](const auto& s) { return build_kernel(ctx, samples, s, prec); }, spec);
}

inline NormalizedKernel from_matrix(const Context& ctx, const Matrix& a, Precision prec = Precision::fp64) {
    renyi_kernel* k = nullptr;
    check(renyi_kernel_from_matrix(ctx.get(), a.data.data(), a.rows, static_cast<int>(prec), &k));
    return NormalizedKernel(k);
}

inline NormalizedKernel hadamard_joint(const Context& ctx, const NormalizedKernel& a,
                                       const NormalizedKernel& b) {  // kernel.cpp:74-101
    renyi_kernel* k = nullptr;
    check(renyi_kernel_hadamard_joint(ctx.get(), a.get(), b.get(), &k));
    return NormalizedKernel(k);
}

inline NormalizedKernel hadamard_joint(const Context& ctx, const std::vector<NormalizedKernel>& kernels) {
    std::vector<const renyi_kernel*> hs;
    for (const auto& k : kernels) hs.push_back(k.get());
    renyi_kernel* k = nullptr;
    check(renyi_kernel_hadamard_joint_n(ctx.get(), hs.data(), static_cast<int>(hs.size()), &k));
    return NormalizedKernel(k);
}

namespace ops {  // proj/include/renyi/ops.hpp:23-29
inline Matrix matmul_panel(const Context& ctx, const NormalizedKernel& a, const Matrix& x) {
    Matrix y(x.rows, x.cols);
    check(renyi_matmul_panel(ctx.get(), a.get(), x.data.data(), static_cast<int>(x.cols), y.data.data()));
    return y;
}
inline std::vector<double> matvec(const Context& ctx, const NormalizedKernel& a, const std::vector<double>& x) {
    std::vector<double> y(x.size());
    check(renyi_matvec(ctx.get(), a.get(), x.data(), y.data()));
    return y;
}
// the unnormalised Grams and the scaled Hadamard product (ops.hpp:12-33); samples rows = samples
inline Matrix gaussian_gram(const Context& ctx, const Matrix& samples, double sigma) {
    Matrix k(samples.rows, samples.rows);
    check(renyi_ops_gaussian_gram(ctx.get(), samples.data.data(), samples.rows, samples.cols, samples.rows, sigma,
                                  k.data.data()));
    return k;
}
inline Matrix polynomial_gram(const Context& ctx, const Matrix& samples, int degree, double offset) {
    Matrix k(samples.rows, samples.rows);
    check(renyi_ops_polynomial_gram(ctx.get(), samples.data.data(), samples.rows, samples.cols, samples.rows, degree,
                                    offset, k.data.data()));
    return k;
}
inline Matrix hadamard_scaled(const Context& ctx, const Matrix& a, const Matrix& b, double scale) {
    Matrix c(a.rows, a.cols);
    check(renyi_ops_hadamard_scaled(ctx.get(), a.data.data(), b.data.data(), a.rows, a.cols, scale, c.data.data()));
    return c;
}
}  // namespace ops

// MatrixFunctionSpec factories (proj/include/renyi/poly.hpp:54-70)
struct MatrixFunctionSpec {
    renyi_matfun f{};
    static MatrixFunctionSpec int_power(int alpha) { return {{RENYI_MATFUN_INT_POWER, double(alpha), alpha, 0, 1}}; }
    static MatrixFunctionSpec taylor(double alpha, int m, double v) { return {{RENYI_MATFUN_TAYLOR, alpha, m, 0, v}}; }
    static MatrixFunctionSpec chebyshev(double alpha, int m, double u, double v) {
        return {{RENYI_MATFUN_CHEBYSHEV, alpha, m, u, v}};
    }
    int query_cost() const { return f.kind == RENYI_MATFUN_INT_POWER ? static_cast<int>(f.alpha) : f.degree; }
};

// chebyshev_node_coeffs (proj/src/poly.cpp:18-40) for any f
inline std::vector<double> chebyshev_node_coeffs(const std::function<double(double)>& f, int m, double a, double b) {
    std::vector<double> c(m > 0 ? m + 1 : 1);
    auto tramp = [](double x, void* user) { return (*static_cast<const std::function<double(double)>*>(user))(x); };
    check(renyi_chebyshev_node_coeffs(tramp, const_cast<void*>(static_cast<const void*>(&f)), m, a, b, c.data()));
    return c;
}
inline std::string method_name(int method) { return renyi_method_name(method); }  // entropy.cpp:51-60

inline Matrix apply_panel(const Context& ctx, const MatrixFunctionSpec& spec, const NormalizedKernel& a,
                          const Matrix& x) {  // poly.cpp:158-164
    Matrix y(x.rows, x.cols);
    check(renyi_apply_panel(ctx.get(), a.get(), &spec.f, x.data.data(), static_cast<int>(x.cols), y.data.data()));
    return y;
}

struct SketchConfig {  // proj/include/renyi/hutchpp.hpp:12-18 (+ explicit split and probe injection)
    int s = 8;
    uint64_t seed = 0;
    int s_q = -1, s_g = -1;
    int probe_kind = RENYI_PROBE_GAUSSIAN;
    const Matrix* sketch = nullptr;
    const Matrix* probes = nullptr;
    int sketch_cols() const { return s_q >= 0 ? s_q : s / 4; }
    int probe_cols() const { return s_g >= 0 ? s_g : s - 2 * (s / 4); }
};

using TraceEstimate = renyi_trace_estimate;

inline TraceEstimate hutchpp(const Context& ctx, const MatrixFunctionSpec& f, const NormalizedKernel& a,
                             const SketchConfig& cfg) {  // hutchpp.cpp:69-115
    if (cfg.s_q < 0 && cfg.s_g < 0 && cfg.s < 8)
        throw error(errc::invalid_argument, "hutchpp needs a query budget s >= 8");
    renyi_sketch sk{cfg.sketch_cols(), cfg.probe_cols(), cfg.seed, cfg.probe_kind,
                    cfg.sketch ? cfg.sketch->data.data() : nullptr, cfg.probes ? cfg.probes->data.data() : nullptr};
    TraceEstimate t{};
    check(renyi_hutchpp(ctx.get(), a.get(), &f.f, &sk, &t));
    return t;
}

using PowerOptions = renyi_power_options;
using SpectrumBounds = renyi_spectrum_bounds;

inline PowerOptions default_power_options() {
    PowerOptions o;
    renyi_default_power_options(&o);
    return o;
}

inline SpectrumBounds estimate_bounds(const Context& ctx, const NormalizedKernel& a,
                                      const PowerOptions& o = default_power_options()) {  // spectrum.cpp:80-103
    SpectrumBounds b{};
    check(renyi_estimate_bounds(ctx.get(), a.get(), &o, &b));
    return b;
}

struct EstimatorParams : renyi_estimator_params {  // proj/include/renyi/entropy.hpp:18-30
    EstimatorParams() { renyi_default_params(this); }
};
using EntropyEstimate = renyi_entropy_estimate;
using MutualInformation = renyi_mi_estimate;

inline EntropyEstimate estimate(const Context& ctx, const NormalizedKernel& a,
                                const EstimatorParams& p) {  // entropy.cpp:201-275
    EntropyEstimate e{};
    check(renyi_estimate(ctx.get(), a.get(), &p, &e));
    return e;
}

inline EntropyEstimate entropy_int(const Context& ctx, const NormalizedKernel& a, int alpha, int s, uint64_t seed) {
    EntropyEstimate e{};
    check(renyi_entropy_int(ctx.get(), a.get(), alpha, s, seed, &e));
    return e;
}

inline EntropyEstimate entropy_taylor(const Context& ctx, const NormalizedKernel& a, double alpha, int s, int m,
                                      double v, uint64_t seed) {
    EntropyEstimate e{};
    check(renyi_entropy_taylor(ctx.get(), a.get(), alpha, s, m, v, seed, &e));
    return e;
}

inline EntropyEstimate entropy_chebyshev(const Context& ctx, const NormalizedKernel& a, double alpha, int s, int m,
                                         double u, double v, uint64_t seed) {
    EntropyEstimate e{};
    check(renyi_entropy_chebyshev(ctx.get(), a.get(), alpha, s, m, u, v, seed, &e));
    return e;
}

inline double entropy_from_trace(double trace, double alpha) {  // entropy.cpp:62-69
    double out = 0.0;
    check(renyi_entropy_from_trace(trace, alpha, &out));
    return out;
}

inline MutualInformation mutual_information(const Context& ctx, const NormalizedKernel& vars,
                                            const NormalizedKernel& target,
                                            const EstimatorParams& p) {  // measures.cpp:36-46
    MutualInformation mi{};
    check(renyi_mutual_information(ctx.get(), vars.get(), target.get(), &p, &mi));
    return mi;
}

// Dataset (proj/include/renyi/features.hpp:12-19); features resident on the device
class Dataset {
public:
    explicit Dataset(renyi_dataset* d) : h_(d, Del{}) {
        int hl = 0;
        check(renyi_dataset_shape(d, &n_, &d_, &hl));
        for (int64_t j = 0; j < d_; ++j) names.emplace_back(renyi_dataset_name(d, j));
        if (hl)
            for (int64_t i = 0; i < n_; ++i) labels.emplace_back(renyi_dataset_label(d, i));
    }
    int64_t n() const { return n_; }
    int64_t d() const { return d_; }
    Matrix features(const Context& ctx) const {
        Matrix x(n_, d_);
        check(renyi_dataset_features(ctx.get(), h_.get(), x.data.data(), n_ > 0 ? n_ : 1));
        return x;
    }
    // build_kernel(features(:, columns), spec) without leaving the device
    NormalizedKernel kernel(const Context& ctx, const GaussianKernel& spec, Precision prec = Precision::fp64,
                            const std::vector<int64_t>& columns = {}) const {
        renyi_kernel* k = nullptr;
        check(renyi_kernel_build_gaussian_dataset(ctx.get(), h_.get(), columns.empty() ? nullptr : columns.data(),
                                                  static_cast<int64_t>(columns.size()), spec.sigma,
                                                  static_cast<int>(prec), &k));
        return NormalizedKernel(k);
    }
    std::vector<std::string> names, labels;

private:
    struct Del {
        void operator()(renyi_dataset* d) const { renyi_dataset_destroy(d); }
    };
    std::shared_ptr<renyi_dataset> h_;
    int64_t n_ = 0, d_ = 0;
};

// load_csv (proj/include/renyi/csv.hpp:14-15), parsed on the device
inline Dataset load_csv(const Context& ctx, const std::string& path,
                        const std::optional<std::string>& label_column = std::nullopt) {
    renyi_dataset* d = nullptr;
    check(renyi_csv_load(ctx.get(), path.c_str(), label_column ? label_column->c_str() : nullptr, &d));
    return Dataset(d);
}

// cmd_entropy's composition (proj/tools/renyi_cli.cpp:144-154): build_kernel + estimate
inline EntropyEstimate entropy(const Context& ctx, const Matrix& samples, double sigma, const EstimatorParams& p,
                               Precision prec = Precision::fp32) {
    EntropyEstimate e{};
    check(renyi_entropy(ctx.get(), samples.data.data(), samples.rows, samples.cols, samples.rows, sigma, &p,
                        static_cast<int>(prec), &e));
    return e;
}

}  // namespace renyi::gpu
