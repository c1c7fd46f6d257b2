// Host-side arithmetic of the estimator that stays on the CPU: the
// reference's counter-based RNG (bitwise), polynomial coefficients, parameter
// selection, the μ bound, entropy from a trace, and the tiny dense linear
// algebra used by CholeskyQR2 (s_q x s_q matrices). Every function cites the
// reference routine it restates.
#pragma once

#include <functional>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace rb {

// Status codes: reference errc (proj/include/renyi/common.hpp:14-25) + 1, then
// device/runtime kinds. Mirrored in include/renyi_b200.h.
enum Status : int {
    kOk = 0,
    kInvalidArgument = 1,
    kZeroDiagonal = 2,
    kNonFinite = 3,
    kSizeMismatch = 4,
    kDomainError = 5,
    kRankCollapse = 6,
    kNonPositiveTrace = 7,
    kAlphaIsOne = 8,
    kDegenerateBounds = 9,
    kParseError = 10,
    kCudaError = 20,
    kNcclError = 21,
    kOutOfMemory = 22,
    kNoDevice = 23,
    kInternal = 24,
};

class Error : public std::runtime_error {
public:
    Error(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
    int code() const noexcept { return code_; }

private:
    int code_;
};

[[noreturn]] inline void fail(int code, const std::string& what) { throw Error(code, what); }

// ---- RNG: proj/src/rng.cpp:8-64 ------------------------------------------
uint64_t mix64(uint64_t x);
uint64_t derive_key(uint64_t seed, uint64_t tag);
uint64_t hash_name(const char* name);

class RandomStream {
public:
    explicit RandomStream(uint64_t key) : key_(key) {}
    uint64_t next_u64() { return mix64(key_ ^ mix64(counter_++)); }
    double next_uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double next_gaussian();
    double next_rademacher() { return (next_u64() >> 63) ? -1.0 : 1.0; }
    RandomStream derive(uint64_t tag) const { return RandomStream(derive_key(key_, tag)); }  // rng.cpp:30-32
    uint64_t key() const { return key_; }

private:
    uint64_t key_;
    uint64_t counter_ = 0;
    bool have_spare_ = false;
    double spare_ = 0.0;
};

enum ProbeKind : int { kProbeGaussian = 0, kProbeRademacher = 1 };

// detail::gaussian_panel (proj/src/hutchpp.cpp:13-22), column-major n x cols;
// kind Rademacher uses the same per-column substreams.
void probe_panel(int64_t n, int cols, uint64_t seed, const char* label, int kind, double* out);
// the same panel with its columns (independent substreams) spread over the host's hardware threads
void probe_panel_mt(int64_t n, int cols, uint64_t seed, const char* label, int kind, double* out);
// column j of a panel whose base key is derive_key(seed, hash_name(label))
void probe_column(uint64_t base, int j, int64_t n, int kind, double* col);

// ---- polynomial coefficients: proj/src/poly.cpp:10-58 ----------------------
std::vector<double> binomial_coeffs(double alpha, int m);
std::vector<double> chebyshev_node_coeffs(const std::function<double(double)>& f, int m, double a, double b);
std::vector<double> chebyshev_power_coeffs(double alpha, int m, double a, double b);
double taylor_tail_constant(double alpha, int k_max = 10000);
double chebyshev_safeguard(double u, double v);

enum MatFunKind : int { kIntPower = 0, kTaylor = 1, kChebyshev = 2 };

// MatrixFunctionSpec (proj/include/renyi/poly.hpp:32-70, proj/src/poly.cpp:60-90)
struct MatFun {
    int kind = kIntPower;
    double alpha = 2.0;
    int degree = 2;  // alpha for IntPower, m otherwise
    double u = 0.0, v = 1.0;
    std::vector<double> coeffs;  // binomials (Taylor) or Chebyshev c_k

    static MatFun int_power(int alpha);
    static MatFun taylor(double alpha, int m, double v);
    static MatFun chebyshev(double alpha, int m, double u, double v);
    int query_cost() const { return degree; }
    // recurrence coefficients for pass k (0-based): T_{k+1} = a1 A T_k + a2 T_k + a3 T_{k-1}
    void pass_coeffs(int k, double* a1, double* a2, double* a3) const;
    // trace from per-pass dots x·T_k, k = 0..degree
    double combine(const double* dots_by_pass, int stride) const;
    // the same polynomial at a scalar (scalar_value, proj/src/poly.cpp:166-168)
    double scalar_value(double lambda) const;
};

// ---- entropy.cpp host arithmetic ------------------------------------------
enum Method : int { kMethodExact = 0, kMethodInt = 1, kMethodTaylor = 2, kMethodChebyshev = 3, kMethodAuto = 4 };

void validate_alpha(double alpha);                    // entropy.cpp:16-22
bool integer_alpha(double alpha, int* value);         // entropy.cpp:24-31
void require_non_integer(double alpha, const char* which);
double entropy_from_trace(double trace, double alpha);  // entropy.cpp:62-69

struct SpectrumBoundsH {
    double u = 0.0, v = 1.0, kappa = std::numeric_limits<double>::infinity();
    int iterations_used = 0;
    bool v_converged = true, u_converged = true, rank_deficient = false;
};

struct SelectedParams {
    int s = 0, m = 0;
};
SelectedParams select_params(double alpha, double epsilon, double delta, const SpectrumBoundsH& b, int64_t n,
                             int method);  // entropy.cpp:137-176

struct MuBoundH {
    double u, v, alpha;
    int64_t n;
    double mu, lower, upper;
};
MuBoundH mu_bound(double u, double v, double alpha, int64_t n);  // entropy.cpp:178-199

// ---- small dense linear algebra (column-major) ----------------------------
// Symmetric eigendecomposition (cyclic Jacobi): a (p x p) is destroyed; w descending, v columns.
void sym_eig_desc(int p, std::vector<double>& a, std::vector<double>& w, std::vector<double>& v);
// Cholesky G = R^T R (R upper), returns false if not positive definite
bool cholesky_upper(int p, const std::vector<double>& g, std::vector<double>& r);
// inverse of an upper-triangular p x p
std::vector<double> upper_inverse(int p, const std::vector<double>& r);
// Full orthonormal basis whose first k columns span range(q) (q: n x k orthonormal),
// via Householder QR; returns n x n column-major.
std::vector<double> complete_basis(int64_t n, int k, const std::vector<double>& q);

}  // namespace rb
