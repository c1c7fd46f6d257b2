// Builds against include/renyi_b200.hpp and links librenyi_b200.so — the binding
// a reference maintainer would use. On a B200 it runs one estimate; without a GPU
// it exercises the error path (no_device) and the host arithmetic.
#include <cmath>
#include <cstdio>

#include "renyi_b200.hpp"

int main() {
    using namespace renyi::gpu;
    // host arithmetic works everywhere
    const double h = entropy_from_trace(0.38, 2.0);
    if (std::abs(h + std::log(0.38)) > 1e-15) return 2;
    try {
        Context ctx(0);
        Matrix x(500, 4);
        for (int64_t j = 0; j < 4; ++j)
            for (int64_t i = 0; i < 500; ++i) x(i, j) = std::sin(0.37 * i + 1.3 * j);
        NormalizedKernel k = build_kernel(ctx, x, GaussianKernel{2.0}, Precision::fp32);
        EstimatorParams p;
        p.alpha = 1.5;
        p.method = RENYI_METHOD_CHEBYSHEV;
        p.s = 32;
        p.m = 20;
        p.has_bounds = 1;
        p.bounds.u = 0.0;
        p.bounds.v = 1.0;
        const EntropyEstimate e = estimate(ctx, k, p);
        std::printf("entropy %.12f trace %.12f\n", e.entropy, e.trace_estimate);
        // load_csv on the device feeding build_kernel (proj/include/renyi/csv.hpp:14-15)
        const std::string path = "/tmp/renyi_example_host.csv";
        if (FILE* f = std::fopen(path.c_str(), "wb")) {
            std::fprintf(f, "a,b,class\n");
            for (int i = 0; i < 200; ++i) std::fprintf(f, "%g,%g,%s\n", std::sin(0.1 * i), std::cos(0.3 * i), i % 2 ? "x" : "y");
            std::fclose(f);
        }
        const Dataset data = load_csv(ctx, path, std::string("class"));
        if (data.n() != 200 || data.d() != 2 || data.labels.size() != 200 || data.names[1] != "b") return 3;
        const EntropyEstimate e2 = estimate(ctx, data.kernel(ctx, GaussianKernel{1.0}, Precision::fp32), p);
        std::printf("csv entropy %.12f\n", e2.entropy);
        return 0;
    } catch (const error& e) {
        std::printf("error kind=%d usage=%d: %s\n", static_cast<int>(e.kind()), e.is_usage(), e.what());
        return e.kind() == errc::no_device ? 0 : 1;
    }
}
