#include "host_math.h"

#include <thread>

#include <algorithm>
#include <cmath>
#include <numbers>

namespace rb {

// ---- RNG --------------------------------------------------------------------
uint64_t mix64(uint64_t x) {  // proj/src/rng.cpp:8-14 (splitmix64 finalizer)
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t derive_key(uint64_t seed, uint64_t tag) {  // proj/src/rng.cpp:16-18
    return mix64(seed ^ mix64(tag + 0x6a09e667f3bcc909ULL));
}

uint64_t hash_name(const char* name) {  // proj/src/rng.cpp:20-28 (FNV-1a)
    uint64_t h = 0xcbf29ce484222325ULL;
    for (const char* p = name; *p; ++p) {
        h ^= static_cast<unsigned char>(*p);
        h *= 0x100000001b3ULL;
    }
    return h;
}

double RandomStream::next_gaussian() {  // proj/src/rng.cpp:41-54
    if (have_spare_) {
        have_spare_ = false;
        return spare_;
    }
    double u1 = next_uniform();
    while (u1 <= 0.0) u1 = next_uniform();
    const double u2 = next_uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * std::numbers::pi * u2;
    spare_ = r * std::sin(theta);
    have_spare_ = true;
    return r * std::cos(theta);
}

void probe_panel(int64_t n, int cols, uint64_t seed, const char* label, int kind, double* out) {
    const uint64_t base = derive_key(seed, hash_name(label));
    for (int j = 0; j < cols; ++j) {
        RandomStream s(derive_key(base, static_cast<uint64_t>(j)));
        double* col = out + static_cast<int64_t>(j) * n;
        if (kind == kProbeRademacher)
            for (int64_t i = 0; i < n; ++i) col[i] = s.next_rademacher();
        else
            for (int64_t i = 0; i < n; ++i) col[i] = s.next_gaussian();
    }
}

void probe_column(uint64_t base, int j, int64_t n, int kind, double* col) {
    RandomStream s(derive_key(base, static_cast<uint64_t>(j)));
    if (kind == kProbeRademacher)
        for (int64_t i = 0; i < n; ++i) col[i] = s.next_rademacher();
    else
        for (int64_t i = 0; i < n; ++i) col[i] = s.next_gaussian();
}

void probe_panel_mt(int64_t n, int cols, uint64_t seed, const char* label, int kind, double* out) {
    const uint64_t base = derive_key(seed, hash_name(label));
    const int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    const int nt = std::max(1, std::min(cols, hw));
    auto work = [&](int t) {
        for (int j = t; j < cols; j += nt) probe_column(base, j, n, kind, out + static_cast<int64_t>(j) * n);
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
}

// ---- coefficients -------------------------------------------------------------
std::vector<double> binomial_coeffs(double alpha, int m) {  // proj/src/poly.cpp:10-16
    if (m < 0) fail(kInvalidArgument, "binomial_coeffs needs m >= 0");
    std::vector<double> b(m + 1);
    b[0] = 1.0;
    for (int k = 0; k < m; ++k) b[k + 1] = b[k] * (alpha - k) / (k + 1);
    return b;
}

// chebyshev_node_coeffs + chebyshev_coeffs for f = lambda^alpha (proj/src/poly.cpp:18-46)
std::vector<double> chebyshev_power_coeffs(double alpha, int m, double a, double b) {
    if (a < 0.0 || b <= a) fail(kDomainError, "chebyshev_coeffs needs 0 <= u < v");
    return chebyshev_node_coeffs([alpha](double lam) { return std::pow(lam, alpha); }, m, a, b);
}

// chebyshev_node_coeffs (proj/src/poly.cpp:18-40): c_k = (2/(m+1)) Σ_i f(g(x_i)) T_k(x_i)
std::vector<double> chebyshev_node_coeffs(const std::function<double(double)>& f, int m, double a, double b) {
    if (m < 1) fail(kInvalidArgument, "chebyshev_node_coeffs needs m >= 1");
    const int n_nodes = m + 1;
    std::vector<double> c(m + 1, 0.0);
    for (int i = 0; i < n_nodes; ++i) {
        const double theta = std::numbers::pi * (i + 0.5) / n_nodes;
        const double x = std::cos(theta);
        const double fx = f(a + 0.5 * (b - a) * (x + 1.0));
        double t_prev = 1.0, t_cur = x;
        c[0] += fx;
        if (m >= 1) c[1] += fx * x;
        for (int k = 2; k <= m; ++k) {
            const double t_next = 2.0 * x * t_cur - t_prev;
            c[k] += fx * t_next;
            t_prev = t_cur;
            t_cur = t_next;
        }
    }
    for (double& ck : c) ck *= 2.0 / n_nodes;
    return c;
}

double taylor_tail_constant(double alpha, int k_max) {  // proj/src/poly.cpp:48-58
    const int shift = static_cast<int>(std::ceil(alpha)) + 1;
    double best = 0.0;
    for (int k = 0; k <= k_max; ++k) {
        double ratio = 1.0;
        for (int i = k; i < k + shift; ++i) ratio *= std::abs(alpha - i) / (i + 1);
        best = std::max(best, ratio);
    }
    return best;
}

double chebyshev_safeguard(double u, double v) {  // proj/include/renyi/poly.hpp:27-30
    const double widened = u + 2.0 * std::sqrt(std::max(0.0, 2.0 * u - u * u));
    return std::max(v, widened);
}

MatFun MatFun::int_power(int alpha) {  // proj/src/poly.cpp:60-63
    if (alpha < 1) fail(kInvalidArgument, "int_power needs alpha >= 1");
    MatFun f;
    f.kind = kIntPower;
    f.alpha = alpha;
    f.degree = alpha;
    return f;
}

MatFun MatFun::taylor(double alpha, int m, double v) {  // proj/src/poly.cpp:65-70
    if (m < 1) fail(kInvalidArgument, "taylor spec needs m >= 1");
    if (v <= 0.0 || v > 1.0) fail(kDomainError, "taylor spec needs v in (0, 1]");
    if (alpha <= 0.0) fail(kInvalidArgument, "taylor spec needs alpha > 0");
    MatFun f;
    f.kind = kTaylor;
    f.alpha = alpha;
    f.degree = m;
    f.v = v;
    f.coeffs = binomial_coeffs(alpha, m);
    return f;
}

MatFun MatFun::chebyshev(double alpha, int m, double u, double v) {  // proj/src/poly.cpp:72-80
    if (m < 1) fail(kInvalidArgument, "chebyshev spec needs m >= 1");
    if (alpha <= 0.0) fail(kInvalidArgument, "chebyshev spec needs alpha > 0");
    if (u < 0.0) fail(kDomainError, "chebyshev spec needs u >= 0");
    const double safe_v = chebyshev_safeguard(u, v);
    if (safe_v <= u) fail(kDomainError, "chebyshev spec needs v > u after safeguard");
    MatFun f;
    f.kind = kChebyshev;
    f.alpha = alpha;
    f.degree = m;
    f.u = u;
    f.v = safe_v;
    f.coeffs = chebyshev_power_coeffs(alpha, m, u, safe_v);
    return f;
}

// proj/src/poly.cpp:97-134: the three recurrences as per-pass coefficients.
void MatFun::pass_coeffs(int k, double* a1, double* a2, double* a3) const {
    switch (kind) {
        case kIntPower:
            *a1 = 1.0, *a2 = 0.0, *a3 = 0.0;  // y <- A y
            break;
        case kTaylor:
            *a1 = 1.0 / v, *a2 = -1.0, *a3 = 0.0;  // term <- inv_v*A term - term
            break;
        default: {
            const double scale = 2.0 / (v - u);
            const double center = (v + u) / (v - u);
            if (k == 0) {
                *a1 = scale, *a2 = -center, *a3 = 0.0;  // T1 = mapped(x)
            } else {
                *a1 = 2.0 * scale, *a2 = -2.0 * center, *a3 = -1.0;  // T_{k+1} = 2 mapped(T_k) - T_{k-1}
            }
        }
    }
}

double MatFun::combine(const double* d, int stride) const {
    switch (kind) {
        case kIntPower:
            return d[static_cast<int64_t>(degree) * stride];
        case kTaylor: {
            double acc = coeffs[0] * d[0];
            for (int k = 1; k <= degree; ++k) acc += coeffs[k] * d[static_cast<int64_t>(k) * stride];
            return std::pow(v, alpha) * acc;
        }
        default: {
            double acc = (0.5 * coeffs[0]) * d[0];
            for (int k = 1; k <= degree; ++k) acc += coeffs[k] * d[static_cast<int64_t>(k) * stride];
            return acc;
        }
    }
}

double MatFun::scalar_value(double lambda) const {
    switch (kind) {
        case kIntPower: {
            double y = 1.0;
            for (int k = 0; k < degree; ++k) y = lambda * y;
            return y;
        }
        case kTaylor: {
            const double inv_v = 1.0 / v;
            double term = 1.0, acc = coeffs[0] * 1.0;
            for (int k = 1; k <= degree; ++k) {
                term = inv_v * (lambda * term) - term;
                acc += coeffs[k] * term;
            }
            return std::pow(v, alpha) * acc;
        }
        default: {
            const double scale = 2.0 / (v - u);
            const double center = (v + u) / (v - u);
            auto mapped = [&](double w) { return scale * (lambda * w) - center * w; };
            double t_prev = 1.0, acc = (0.5 * coeffs[0]) * 1.0;
            double t_cur = mapped(1.0);
            acc += coeffs[1] * t_cur;
            for (int k = 2; k <= degree; ++k) {
                const double t_next = 2.0 * mapped(t_cur) - t_prev;
                acc += coeffs[k] * t_next;
                t_prev = t_cur;
                t_cur = t_next;
            }
            return acc;
        }
    }
}

// ---- entropy arithmetic ---------------------------------------------------------
namespace {
constexpr double kAlphaOneTol = 1e-9;
int round_up_multiple_of_4(double x) {
    const long c = static_cast<long>(std::ceil(x));
    return static_cast<int>((c + 3) / 4 * 4);
}
}  // namespace

void validate_alpha(double alpha) {
    if (!(alpha > 0.0)) fail(kInvalidArgument, "alpha must be positive");
    if (std::abs(alpha - 1.0) <= kAlphaOneTol)
        fail(kAlphaIsOne,
             "alpha within 1e-9 of 1 is rejected: the estimators degrade as 1/|alpha-1| and the Shannon limit is "
             "out of scope");
}

bool integer_alpha(double alpha, int* value) {
    const double r = std::round(alpha);
    if (std::abs(alpha - r) <= kAlphaOneTol && r >= 2.0) {
        if (value) *value = static_cast<int>(r);
        return true;
    }
    return false;
}

void require_non_integer(double alpha, const char* which) {
    const double r = std::round(alpha);
    if (std::abs(alpha - r) <= kAlphaOneTol)
        fail(kInvalidArgument, std::string(which) + " handles non-integer alpha; use the integer-power path");
}

double entropy_from_trace(double trace, double alpha) {
    validate_alpha(alpha);
    if (!(trace > 0.0))
        fail(kNonPositiveTrace, "trace estimate is not positive (" + std::to_string(trace) +
                                    "); the query budget s is too small for this matrix");
    return std::log(trace) / (1.0 - alpha);
}

SelectedParams select_params(double alpha, double epsilon, double delta, const SpectrumBoundsH& b, int64_t n,
                             int method) {
    validate_alpha(alpha);
    if (!(epsilon > 0.0 && epsilon < 1.0)) fail(kInvalidArgument, "epsilon must be in (0,1)");
    if (!(delta > 0.0 && delta < 1.0)) fail(kInvalidArgument, "delta must be in (0,1)");
    const double gap = std::abs(alpha - 1.0);
    const double log_inv_delta = std::log(1.0 / delta);
    SelectedParams sel;
    sel.s = round_up_multiple_of_4(std::sqrt(log_inv_delta) / (epsilon * gap) + log_inv_delta);
    const double inv_eps_gap = 1.0 / (epsilon * gap);
    if (method == kMethodTaylor) {
        if (b.u > 0.0) {
            sel.m = static_cast<int>(std::ceil(b.kappa * std::log(inv_eps_gap)));
        } else {
            const double vn = b.v * static_cast<double>(n);
            sel.m = static_cast<int>(
                std::ceil(std::pow(vn, 1.0 / std::min(1.0, alpha)) * std::pow(inv_eps_gap, 1.0 / alpha)));
        }
        sel.m = std::max(sel.m, static_cast<int>(std::ceil(alpha)) + 1);
    } else if (method == kMethodChebyshev) {
        if (b.u > 0.0) {
            sel.m = static_cast<int>(std::ceil(std::sqrt(b.kappa) * std::log(b.kappa * inv_eps_gap)));
        } else {
            const double vn = b.v * static_cast<double>(n);
            sel.m = static_cast<int>(
                std::ceil(std::pow(vn, 0.5 / std::min(1.0, alpha)) * std::pow(inv_eps_gap, 0.5 / alpha)));
        }
        sel.m = std::max(sel.m, 1);
    } else {
        sel.m = 0;
    }
    return sel;
}

MuBoundH mu_bound(double u, double v, double alpha, int64_t n) {
    validate_alpha(alpha);
    const double inv_n = 1.0 / static_cast<double>(n);
    if (u < 0.0 || v > 1.0 || u > inv_n + 1e-12 || v < inv_n - 1e-12)
        fail(kInvalidArgument, "mu_bound needs 0 <= u <= 1/n <= v <= 1");
    MuBoundH b{u, v, alpha, n, 0.0, 0.0, 0.0};
    const double flat = std::pow(static_cast<double>(n), 1.0 - alpha);
    if (v > u) {
        const double nd = static_cast<double>(n);
        const double w_v = (1.0 - u * nd) / (v - u);
        const double w_u = (v * nd - 1.0) / (v - u);
        const double u_pow = u > 0.0 ? std::pow(u, alpha) : 0.0;
        b.mu = w_v * std::pow(v, alpha) + w_u * u_pow;
    } else if (v == u && std::abs(v - inv_n) <= 1e-12) {
        b.mu = flat;
    } else {
        fail(kDegenerateBounds, "mu_bound needs v > u (or the degenerate v = u = 1/n)");
    }
    b.lower = std::min(b.mu, flat);
    b.upper = std::max(b.mu, flat);
    return b;
}

// ---- small dense linear algebra ---------------------------------------------------
void sym_eig_desc(int p, std::vector<double>& a, std::vector<double>& w, std::vector<double>& v) {
    // cyclic Jacobi on a column-major symmetric p x p matrix
    v.assign(static_cast<size_t>(p) * p, 0.0);
    for (int i = 0; i < p; ++i) v[i + static_cast<size_t>(i) * p] = 1.0;
    auto A = [&](int i, int j) -> double& { return a[i + static_cast<size_t>(j) * p]; };
    auto V = [&](int i, int j) -> double& { return v[i + static_cast<size_t>(j) * p]; };
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, total = 0.0;
        for (int j = 0; j < p; ++j)
            for (int i = 0; i < p; ++i) {
                total += A(i, j) * A(i, j);
                if (i != j) off += A(i, j) * A(i, j);
            }
        if (off <= 1e-30 * total || off == 0.0) break;
        for (int pp = 0; pp < p - 1; ++pp)
            for (int q = pp + 1; q < p; ++q) {
                const double apq = A(pp, q);
                if (apq == 0.0) continue;
                const double app = A(pp, pp), aqq = A(q, q);
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < p; ++k) {
                    const double akp = A(k, pp), akq = A(k, q);
                    A(k, pp) = c * akp - s * akq;
                    A(k, q) = s * akp + c * akq;
                }
                for (int k = 0; k < p; ++k) {
                    const double apk = A(pp, k), aqk = A(q, k);
                    A(pp, k) = c * apk - s * aqk;
                    A(q, k) = s * apk + c * aqk;
                }
                for (int k = 0; k < p; ++k) {
                    const double vkp = V(k, pp), vkq = V(k, q);
                    V(k, pp) = c * vkp - s * vkq;
                    V(k, q) = s * vkp + c * vkq;
                }
            }
    }
    std::vector<int> order(p);
    for (int i = 0; i < p; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return A(x, x) > A(y, y); });
    w.resize(p);
    std::vector<double> vs(static_cast<size_t>(p) * p);
    for (int c = 0; c < p; ++c) {
        w[c] = A(order[c], order[c]);
        for (int k = 0; k < p; ++k) vs[k + static_cast<size_t>(c) * p] = V(k, order[c]);
    }
    v.swap(vs);
}

bool cholesky_upper(int p, const std::vector<double>& g, std::vector<double>& r) {
    r.assign(static_cast<size_t>(p) * p, 0.0);
    for (int j = 0; j < p; ++j) {
        for (int i = 0; i <= j; ++i) {
            double s = g[i + static_cast<size_t>(j) * p];
            for (int k = 0; k < i; ++k) s -= r[k + static_cast<size_t>(i) * p] * r[k + static_cast<size_t>(j) * p];
            if (i == j) {
                if (!(s > 0.0)) return false;
                r[j + static_cast<size_t>(j) * p] = std::sqrt(s);
            } else {
                r[i + static_cast<size_t>(j) * p] = s / r[i + static_cast<size_t>(i) * p];
            }
        }
    }
    return true;
}

std::vector<double> upper_inverse(int p, const std::vector<double>& r) {
    std::vector<double> x(static_cast<size_t>(p) * p, 0.0);
    for (int j = 0; j < p; ++j) {
        x[j + static_cast<size_t>(j) * p] = 1.0 / r[j + static_cast<size_t>(j) * p];
        for (int i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int k = i + 1; k <= j; ++k) s += r[i + static_cast<size_t>(k) * p] * x[k + static_cast<size_t>(j) * p];
            x[i + static_cast<size_t>(j) * p] = -s / r[i + static_cast<size_t>(i) * p];
        }
    }
    return x;
}

std::vector<double> complete_basis(int64_t n, int k, const std::vector<double>& q) {
    // Householder QR of q (n x k); Q_full = H_0 ... H_{k-1}
    std::vector<double> a(q);
    std::vector<std::vector<double>> vs;
    std::vector<double> betas;
    for (int j = 0; j < k; ++j) {
        double norm = 0.0;
        for (int64_t i = j; i < n; ++i) norm += a[i + j * n] * a[i + j * n];
        norm = std::sqrt(norm);
        std::vector<double> vv(n, 0.0);
        const double x0 = a[j + j * n];
        const double alpha = x0 >= 0 ? -norm : norm;
        for (int64_t i = j; i < n; ++i) vv[i] = a[i + j * n];
        vv[j] -= alpha;
        double vn = 0.0;
        for (int64_t i = j; i < n; ++i) vn += vv[i] * vv[i];
        const double beta = vn > 0 ? 2.0 / vn : 0.0;
        for (int c = j; c < k; ++c) {
            double s = 0.0;
            for (int64_t i = j; i < n; ++i) s += vv[i] * a[i + c * n];
            s *= beta;
            for (int64_t i = j; i < n; ++i) a[i + c * n] -= s * vv[i];
        }
        vs.push_back(std::move(vv));
        betas.push_back(beta);
    }
    std::vector<double> full(static_cast<size_t>(n) * n, 0.0);
    for (int64_t i = 0; i < n; ++i) full[i + i * n] = 1.0;
    for (int j = k - 1; j >= 0; --j) {
        const std::vector<double>& vv = vs[j];
        for (int64_t c = 0; c < n; ++c) {
            double s = 0.0;
            for (int64_t i = j; i < n; ++i) s += vv[i] * full[i + c * n];
            s *= betas[j];
            for (int64_t i = j; i < n; ++i) full[i + c * n] -= s * vv[i];
        }
    }
    return full;
}

}  // namespace rb
