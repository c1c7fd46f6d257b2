// C ABI (include/renyi_b200.h) over the C++ engine. Exceptions never cross the
// boundary: every entry point maps rb::Error to its status code and stores the
// message for renyi_last_error().
#pragma GCC visibility push(default)
#include "../../include/renyi_b200.h"
#pragma GCC visibility pop

#include <cmath>
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "engine.h"

struct renyi_ctx {
    explicit renyi_ctx(int device) : ctx(device) {}
    rb::Context ctx;
};

struct renyi_kernel {
    rb::KernelPtr k;
};

struct renyi_dataset {
    std::unique_ptr<rb::Dataset> d;
};

struct renyi_local_group {
    std::shared_ptr<rb::LocalGroup> g;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return RENYI_OK;
    } catch (const rb::Error& e) {
        g_last_error = e.what();
        return e.code();
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return RENYI_E_OOM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return RENYI_E_INTERNAL;
    } catch (...) {
        g_last_error = "unknown failure";
        return RENYI_E_INTERNAL;
    }
}

// Builds a handle and releases it to the caller only when construction succeeded.
template <typename H, typename F>
H* make_handle(F&& build) {
    auto h = std::make_unique<H>();
    build(*h);
    return h.release();
}

void need(const void* p, const char* what) {
    if (!p) rb::fail(rb::kInvalidArgument, std::string(what) + " is NULL");
}

rb::MatFun to_matfun(const renyi_matfun* f) {
    need(f, "matrix function");
    switch (f->kind) {
        case RENYI_MATFUN_INT_POWER: {
            const double r = std::round(f->alpha);
            if (std::abs(f->alpha - r) > 1e-9) rb::fail(rb::kInvalidArgument, "int_power needs an integer alpha");
            return rb::MatFun::int_power(static_cast<int>(r));
        }
        case RENYI_MATFUN_TAYLOR:
            return rb::MatFun::taylor(f->alpha, f->degree, f->v);
        case RENYI_MATFUN_CHEBYSHEV:
            return rb::MatFun::chebyshev(f->alpha, f->degree, f->u, f->v);
        default:
            rb::fail(rb::kInvalidArgument, "unknown matrix function kind");
    }
}

rb::PowerOpts to_power(const renyi_power_options* o) {
    rb::PowerOpts p;
    if (o) {
        p.max_iters = o->max_iters;
        p.tol = o->tol;
        p.seed = o->seed;
        p.rank_floor = o->rank_floor;
    }
    return p;
}

rb::SpectrumBoundsH to_bounds(const renyi_spectrum_bounds& b) {
    rb::SpectrumBoundsH h;
    h.u = b.u, h.v = b.v, h.kappa = b.kappa;
    h.iterations_used = b.iterations_used;
    h.v_converged = b.v_converged != 0, h.u_converged = b.u_converged != 0, h.rank_deficient = b.rank_deficient != 0;
    return h;
}

void from_bounds(const rb::SpectrumBoundsH& h, renyi_spectrum_bounds* b) {
    b->u = h.u, b->v = h.v, b->kappa = h.kappa;
    b->iterations_used = h.iterations_used;
    b->v_converged = h.v_converged, b->u_converged = h.u_converged, b->rank_deficient = h.rank_deficient;
}

rb::EstParams to_params(const renyi_estimator_params* p) {
    need(p, "estimator params");
    rb::EstParams q;
    q.alpha = p->alpha;
    q.method = p->method;
    q.s = p->s, q.m = p->m;
    q.epsilon = p->epsilon, q.delta = p->delta;
    q.seed = p->seed;
    q.power = to_power(&p->power);
    q.has_bounds = p->has_bounds != 0;
    q.bounds = to_bounds(p->bounds);
    q.probe_kind = p->probe_kind;
    q.s_q = p->s_q, q.s_g = p->s_g;
    return q;
}

void from_trace(const rb::TraceEst& t, renyi_trace_estimate* o) {
    o->value = t.value, o->low_rank_part = t.low_rank_part, o->residual_part = t.residual_part;
    o->queries_used = t.queries_used, o->sketch_rank = t.sketch_rank, o->exact = t.exact;
}

void from_entropy(const rb::EntropyEst& e, renyi_entropy_estimate* o) {
    o->entropy = e.entropy, o->trace_estimate = e.trace_estimate;
    o->method_used = e.method_used, o->s_used = e.s_used, o->m_used = e.m_used;
    o->has_bounds = e.has_bounds;
    from_bounds(e.bounds_used, &o->bounds_used);
    o->elapsed = e.elapsed;
    o->deterministic = e.deterministic;
    from_trace(e.trace, &o->trace);
}

void check_precision(int precision) {
    if (precision != RENYI_F64 && precision != RENYI_F32 && precision != RENYI_MF) rb::fail(rb::kInvalidArgument, "unknown precision");
}

}  // namespace

extern "C" {

const char* renyi_last_error(void) { return g_last_error.c_str(); }

int renyi_status_is_usage(int s) {
    return s == RENYI_E_INVALID_ARGUMENT || s == RENYI_E_SIZE_MISMATCH || s == RENYI_E_DOMAIN_ERROR ||
           s == RENYI_E_PARSE_ERROR || s == RENYI_E_ALPHA_IS_ONE;
}

int renyi_ctx_create(int device, renyi_ctx** out) {
    return guarded([&] {
        need(out, "out");
        *out = new renyi_ctx(device);
    });
}

int renyi_ctx_destroy(renyi_ctx* ctx) {
    return guarded([&] { delete ctx; });
}

int renyi_ctx_set_tuning(renyi_ctx* ctx, int grid, int kc) {
    return guarded([&] {
        need(ctx, "ctx");
        if (grid < 0 || kc < 1) rb::fail(rb::kInvalidArgument, "grid >= 0 and kc >= 1 required");
        ctx->ctx.grid = grid;
        ctx->ctx.kc = kc;
    });
}

int renyi_ctx_set_matrix_free_chunk(renyi_ctx* ctx, int jblocks) {
    return guarded([&] {
        need(ctx, "ctx");
        if (jblocks < 1) rb::fail(rb::kInvalidArgument, "jblocks >= 1 required");
        ctx->ctx.mf_kc = jblocks;
    });
}

int renyi_shard_rows(int64_t n, int world, int rank, int64_t* row0, int64_t* rows, int64_t* rpr) {
    return guarded([&] {
        need(row0, "row0"), need(rows, "rows"), need(rpr, "rows_per_rank");
        rb::shard_rows(n, world, rank, row0, rows, rpr);
    });
}

int renyi_nccl_unique_id(unsigned char id[128]) {
    return guarded([&] {
        need(id, "id");
        rb::nccl_unique_id(id);
    });
}

int renyi_ctx_init_nccl(renyi_ctx* ctx, int rank, int world, const unsigned char id[128]) {
    return guarded([&] {
        need(ctx, "ctx"), need(id, "id");
        cudaSetDevice(ctx->ctx.device());
        ctx->ctx.exchange = rb::make_nccl_exchange(rank, world, id);
    });
}

int renyi_local_group_create(int world, renyi_local_group** out) {
    return guarded([&] {
        need(out, "out");
        *out = make_handle<renyi_local_group>([&](renyi_local_group& h) { h.g = rb::make_local_group(world); });
    });
}

int renyi_local_group_destroy(renyi_local_group* g) {
    return guarded([&] { delete g; });
}

int renyi_ctx_join_local_group(renyi_ctx* ctx, renyi_local_group* g, int rank) {
    return guarded([&] {
        need(ctx, "ctx"), need(g, "group");
        ctx->ctx.exchange = rb::make_local_exchange(g->g, rank);
    });
}

int renyi_ctx_rank(renyi_ctx* ctx, int* rank, int* world) {
    return guarded([&] {
        need(ctx, "ctx");
        if (rank) *rank = ctx->ctx.rank();
        if (world) *world = ctx->ctx.world();
    });
}

int renyi_ctx_set_operand_mode(renyi_ctx* ctx, int mode) {
    return guarded([&] {
        need(ctx, "ctx");
        if (mode != RENYI_OPERAND_SPLIT && mode != RENYI_OPERAND_FAST && mode != RENYI_OPERAND_AUTO)
            rb::fail(rb::kInvalidArgument, "unknown operand mode");
        ctx->ctx.operand_mode = mode == RENYI_OPERAND_SPLIT ? 0 : (mode == RENYI_OPERAND_FAST ? 1 : 2);
    });
}

int renyi_ctx_set_fused_mi(renyi_ctx* ctx, int on) {
    return guarded([&] {
        need(ctx, "ctx");
        ctx->ctx.fused_mi = on != 0;
    });
}

int renyi_ctx_set_probe_source(renyi_ctx* ctx, int source) {
    return guarded([&] {
        need(ctx, "ctx");
        if (source != RENYI_PROBES_DEVICE && source != RENYI_PROBES_HOST)
            rb::fail(rb::kInvalidArgument, "probe source must be RENYI_PROBES_DEVICE or RENYI_PROBES_HOST");
        ctx->ctx.probe_source = source;
    });
}

int renyi_ctx_set_feature_grouping(renyi_ctx* ctx, int on) {
    return guarded([&] {
        need(ctx, "ctx");
        ctx->ctx.feature_groups = on != 0;
    });
}

int renyi_ctx_sync(renyi_ctx* ctx) {
    return guarded([&] {
        need(ctx, "ctx");
        ctx->ctx.sync();
    });
}

int renyi_release_cached_memory(void) {
    return guarded([&] {
        cudaDeviceSynchronize();
        rb::pool_release_all();
    });
}

int renyi_ctx_profile(renyi_ctx* ctx, int enable) {
    return guarded([&] {
        need(ctx, "ctx");
        ctx->ctx.prof_enable(enable != 0);
    });
}

int renyi_ctx_profile_read(renyi_ctx* ctx, int* launches, double* ms, double* bytes, double* flops) {
    return guarded([&] {
        need(ctx, "ctx");
        need(launches, "launches");
        need(ms, "milliseconds");
        double b = 0.0, f = 0.0;
        ctx->ctx.prof_read(launches, ms, &b, &f);
        if (bytes) *bytes = b;
        if (flops) *flops = f;
    });
}

int renyi_ctx_io_bytes(renyi_ctx* ctx, long long* h2d, long long* d2h) {
    return guarded([&] {
        need(ctx, "ctx");
        if (h2d) *h2d = ctx->ctx.h2d_bytes;
        if (d2h) *d2h = ctx->ctx.d2h_bytes;
    });
}

int renyi_ctx_timer_begin(renyi_ctx* ctx) {
    return guarded([&] {
        need(ctx, "ctx");
        ctx->ctx.timer_begin();
    });
}

int renyi_ctx_timer_end(renyi_ctx* ctx, double* ms) {
    return guarded([&] {
        need(ctx, "ctx");
        need(ms, "milliseconds");
        *ms = ctx->ctx.timer_end_ms();
    });
}

int renyi_ctx_launch_count(renyi_ctx* ctx, long* launches) {
    return guarded([&] {
        need(ctx, "ctx");
        need(launches, "launches");
        *launches = ctx->ctx.launches;
    });
}

int renyi_kernel_build_gaussian(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double sigma,
                                int precision, renyi_kernel** out) {
    return guarded([&] {
        need(ctx, "ctx"), need(x, "samples"), need(out, "out");
        check_precision(precision);
        *out = make_handle<renyi_kernel>([&](renyi_kernel& h) {
            h.k = rb::build_gaussian(ctx->ctx, x, n, d, ldx, sigma, precision);
        });
    });
}

int renyi_ops_gaussian_gram(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double sigma,
                            double* k) {
    return guarded([&] {
        need(ctx, "ctx"), need(x, "samples"), need(k, "out");
        rb::ops_gaussian_gram(ctx->ctx, x, n, d, ldx, sigma, k);
    });
}

int renyi_ops_polynomial_gram(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int degree,
                              double offset, double* k) {
    return guarded([&] {
        need(ctx, "ctx"), need(x, "samples"), need(k, "out");
        rb::ops_polynomial_gram(ctx->ctx, x, n, d, ldx, degree, offset, k);
    });
}

int renyi_ops_hadamard_scaled(renyi_ctx* ctx, const double* a, const double* b, int64_t rows, int64_t cols,
                              double scale, double* c) {
    return guarded([&] {
        need(ctx, "ctx"), need(a, "a"), need(b, "b"), need(c, "out");
        rb::ops_hadamard_scaled(ctx->ctx, a, b, rows, cols, scale, c);
    });
}

int renyi_kernel_build_polynomial(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int degree,
                                  double offset, int precision, renyi_kernel** out) {
    return guarded([&] {
        need(ctx, "ctx"), need(x, "samples"), need(out, "out");
        check_precision(precision);
        *out = make_handle<renyi_kernel>([&](renyi_kernel& h) {
            h.k = rb::build_polynomial(ctx->ctx, x, n, d, ldx, degree, offset, precision);
        });
    });
}

int renyi_kernel_build_polynomial_dev(renyi_ctx* ctx, const double* d_x, int64_t n, int64_t d, int64_t ldx,
                                      int degree, double offset, int precision, renyi_kernel** out) {
    return guarded([&] {
        need(ctx, "ctx"), need(d_x, "samples"), need(out, "out");
        check_precision(precision);
        *out = make_handle<renyi_kernel>([&](renyi_kernel& h) {
            h.k = rb::build_polynomial_dev(ctx->ctx, d_x, n, d, ldx, degree, offset, precision);
        });
    });
}

int renyi_kernel_build_gaussian_joint(renyi_ctx* ctx, const double* x, int64_t n, int64_t dx, int64_t ldx,
                                      double sigma_x, const double* y, int64_t dy, int64_t ldy, double sigma_y,
                                      int precision, renyi_kernel** out) {
    return guarded([&] {
        need(ctx, "ctx"), need(x, "samples"), need(y, "second samples"), need(out, "out");
        check_precision(precision);
        *out = make_handle<renyi_kernel>([&](renyi_kernel& h) {
            h.k = rb::build_gaussian(ctx->ctx, x, n, dx, ldx, sigma_x, precision, y, dy, ldy, sigma_y);
        });
    });
}

int renyi_kernel_build_gaussian_dev(renyi_ctx* ctx, const double* d_x, int64_t n, int64_t d, int64_t ldx,
                                    double sigma, const double* d_y, int64_t dy, int64_t ldy, double sigma_y,
                                    int precision, renyi_kernel** out) {
    return guarded([&] {
        need(ctx, "ctx"), need(d_x, "samples"), need(out, "out");
        check_precision(precision);
        *out = make_handle<renyi_kernel>([&](renyi_kernel& h) {
            h.k = rb::build_gaussian_dev(ctx->ctx, d_x, n, d, ldx, sigma, precision, d_y, dy, ldy, sigma_y);
            ctx->ctx.sync();
        });
    });
}

int renyi_csv_load(renyi_ctx* ctx, const char* path, const char* label_column, renyi_dataset** out) {
    return guarded([&] {
        need(ctx, "ctx"), need(path, "path"), need(out, "out");
        *out = make_handle<renyi_dataset>([&](renyi_dataset& h) {
            h.d = rb::load_csv_file(ctx->ctx, path, label_column);
        });
    });
}

int renyi_csv_parse(renyi_ctx* ctx, const char* text, int64_t len, const char* label_column, const char* source,
                    renyi_dataset** out) {
    return guarded([&] {
        need(ctx, "ctx"), need(out, "out");
        if (len < 0) rb::fail(rb::kInvalidArgument, "negative text length");
        if (len > 0) need(text, "text");
        *out = make_handle<renyi_dataset>([&](renyi_dataset& h) {
            h.d = rb::load_csv_text(ctx->ctx, text, static_cast<size_t>(len), label_column,
                                    source ? source : "<buffer>");
        });
    });
}

int renyi_dataset_shape(const renyi_dataset* ds, int64_t* n, int64_t* d, int* has_labels) {
    return guarded([&] {
        need(ds, "dataset");
        if (n) *n = ds->d->n;
        if (d) *d = ds->d->d;
        if (has_labels) *has_labels = ds->d->labels.empty() ? 0 : 1;
    });
}

int renyi_dataset_features(renyi_ctx* ctx, const renyi_dataset* ds, double* x, int64_t ldx) {
    return guarded([&] {
        need(ctx, "ctx"), need(ds, "dataset");
        const int64_t n = ds->d->n, d = ds->d->d;
        if (n == 0 || d == 0) return;
        need(x, "features");
        if (ldx < n) rb::fail(rb::kInvalidArgument, "leading dimension smaller than the sample count");
        cudaSetDevice(ctx->ctx.device());
        rb::d2h_2d(ctx->ctx, x, static_cast<size_t>(ldx) * sizeof(double), ds->d->features.as<double>(),
                   static_cast<size_t>(n) * sizeof(double), static_cast<size_t>(n) * sizeof(double),
                   static_cast<size_t>(d));
        ctx->ctx.sync();
    });
}

const char* renyi_dataset_name(const renyi_dataset* ds, int64_t j) {
    if (!ds || j < 0 || j >= static_cast<int64_t>(ds->d->names.size())) return nullptr;
    return ds->d->names[static_cast<size_t>(j)].c_str();
}

const char* renyi_dataset_label(const renyi_dataset* ds, int64_t i) {
    if (!ds || i < 0 || i >= static_cast<int64_t>(ds->d->labels.size())) return nullptr;
    return ds->d->labels[static_cast<size_t>(i)].c_str();
}

int renyi_kernel_build_gaussian_dataset(renyi_ctx* ctx, const renyi_dataset* ds, const int64_t* columns,
                                        int64_t ncols, double sigma, int precision, renyi_kernel** out) {
    return guarded([&] {
        need(ctx, "ctx"), need(ds, "dataset"), need(out, "out");
        check_precision(precision);
        const rb::Dataset& data = *ds->d;
        *out = make_handle<renyi_kernel>([&](renyi_kernel& h) {
            cudaSetDevice(ctx->ctx.device());
            if (!columns) {
                h.k = rb::build_gaussian_dev(ctx->ctx, data.features.as<double>(), data.n, data.d, data.n, sigma,
                                            precision);
            } else {
                if (ncols < 1) rb::fail(rb::kInvalidArgument, "need at least one column");
                rb::DevBuf sel;
                sel.alloc(static_cast<size_t>(data.n) * static_cast<size_t>(ncols) * sizeof(double));
                for (int64_t c = 0; c < ncols; ++c) {
                    if (columns[c] < 0 || columns[c] >= data.d)
                        rb::fail(rb::kInvalidArgument, "column " + std::to_string(columns[c]) + " out of range");
                    rb::cuda_check(cudaMemcpyAsync(sel.as<double>() + c * data.n,
                                                   data.features.as<double>() + columns[c] * data.n,
                                                   static_cast<size_t>(data.n) * sizeof(double),
                                                   cudaMemcpyDeviceToDevice, ctx->ctx.stream()),
                                   "column gather");
                }
                h.k = rb::build_gaussian_dev(ctx->ctx, sel.as<double>(), data.n, ncols, data.n, sigma, precision);
            }
            ctx->ctx.sync();
        });
    });
}

int renyi_dataset_destroy(renyi_dataset* ds) {
    return guarded([&] { delete ds; });
}

int renyi_kernel_from_matrix(renyi_ctx* ctx, const double* a, int64_t n, int precision, renyi_kernel** out) {
    return guarded([&] {
        need(ctx, "ctx"), need(a, "matrix"), need(out, "out");
        check_precision(precision);
        *out = make_handle<renyi_kernel>([&](renyi_kernel& h) {
            h.k = rb::from_matrix(ctx->ctx, a, n, precision);
        });
    });
}

int renyi_kernel_hadamard_joint_n(renyi_ctx* ctx, const renyi_kernel* const* kernels, int count,
                                  renyi_kernel** out) {
    return guarded([&] {
        need(ctx, "ctx"), need(kernels, "kernels"), need(out, "out");
        if (count < 2) rb::fail(rb::kInvalidArgument, "hadamard_joint needs at least 2 kernels");
        std::vector<const rb::KernelMatrix*> ks;
        for (int i = 0; i < count; ++i) {
            need(kernels[i], "kernel");
            ks.push_back(kernels[i]->k.get());
        }
        *out = make_handle<renyi_kernel>([&](renyi_kernel& h) { h.k = rb::hadamard_joint_n(ctx->ctx, ks); });
    });
}

int renyi_kernel_hadamard_joint(renyi_ctx* ctx, const renyi_kernel* a, const renyi_kernel* b, renyi_kernel** out) {
    return guarded([&] {
        need(ctx, "ctx"), need(a, "kernel a"), need(b, "kernel b"), need(out, "out");
        *out = make_handle<renyi_kernel>([&](renyi_kernel& h) {
            h.k = rb::hadamard_joint(ctx->ctx, *a->k, *b->k);
        });
    });
}

int renyi_kernel_size(const renyi_kernel* k, int64_t* n) {
    return guarded([&] {
        need(k, "kernel"), need(n, "n");
        *n = k->k->n;
    });
}

int renyi_kernel_download(renyi_ctx* ctx, const renyi_kernel* k, double* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(out, "out");
        rb::download(ctx->ctx, *k->k, out);
    });
}

int renyi_kernel_destroy(renyi_kernel* k) {
    return guarded([&] {
        // storage returns to the engine pool; make sure no queued work still reads it
        if (k) cudaDeviceSynchronize();
        delete k;
    });
}

int renyi_matmul_panel(renyi_ctx* ctx, const renyi_kernel* k, const double* v, int s, double* y) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(v, "panel"), need(y, "out");
        if (s < 1) rb::fail(rb::kInvalidArgument, "panel needs at least one column");
        rb::block_product(ctx->ctx, *k->k, v, s, y);
    });
}

int renyi_matvec(renyi_ctx* ctx, const renyi_kernel* k, const double* x, double* y) {
    return renyi_matmul_panel(ctx, k, x, 1, y);
}

int renyi_apply_panel(renyi_ctx* ctx, const renyi_kernel* k, const renyi_matfun* f, const double* v, int s,
                      double* y) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(v, "panel"), need(y, "out");
        if (s < 1) rb::fail(rb::kInvalidArgument, "panel needs at least one column");
        rb::apply_panel(ctx->ctx, *k->k, to_matfun(f), v, s, y);
    });
}

int renyi_matfun_traces(renyi_ctx* ctx, const renyi_kernel* k, const renyi_matfun* f, const double* x, int s,
                        double* traces) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(x, "panel"), need(traces, "out");
        if (s < 1) rb::fail(rb::kInvalidArgument, "panel needs at least one column");
        rb::matfun_traces(ctx->ctx, *k->k, to_matfun(f), x, s, traces);
    });
}

int renyi_power_method(renyi_ctx* ctx, const renyi_kernel* k, const renyi_power_options* opts, double shift,
                       renyi_power_result* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(out, "out");
        const rb::PowerRes r = rb::power_method(ctx->ctx, *k->k, to_power(opts), shift);
        out->rayleigh = r.rayleigh, out->iterations = r.iterations, out->converged = r.converged;
    });
}

int renyi_estimate_bounds(renyi_ctx* ctx, const renyi_kernel* k, const renyi_power_options* opts,
                          renyi_spectrum_bounds* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(out, "out");
        from_bounds(rb::estimate_bounds(ctx->ctx, *k->k, to_power(opts)), out);
    });
}

int renyi_hutchpp(renyi_ctx* ctx, const renyi_kernel* k, const renyi_matfun* f, const renyi_sketch* cfg,
                  renyi_trace_estimate* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(cfg, "sketch config"), need(out, "out");
        rb::SketchCfg c;
        c.s_q = cfg->s_q, c.s_g = cfg->s_g, c.seed = cfg->seed, c.probe_kind = cfg->probe_kind;
        c.sketch = cfg->sketch, c.probes = cfg->probes;
        from_trace(rb::hutchpp(ctx->ctx, *k->k, to_matfun(f), c), out);
    });
}

int renyi_estimate(renyi_ctx* ctx, const renyi_kernel* k, const renyi_estimator_params* p,
                   renyi_entropy_estimate* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(out, "out");
        from_entropy(rb::estimate(ctx->ctx, *k->k, to_params(p)), out);
    });
}

int renyi_estimate_trials(renyi_ctx* ctx, const renyi_kernel* k, const renyi_estimator_params* p, int trials,
                          renyi_entropy_estimate* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(out, "out");
        const std::vector<rb::EntropyEst> est = rb::estimate_trials(ctx->ctx, *k->k, to_params(p), trials);
        for (int t = 0; t < trials; ++t) from_entropy(est[t], out + t);
    });
}

int renyi_measure_cell(renyi_ctx* ctx, const renyi_kernel* k, double exact_entropy,
                       const renyi_estimator_params* p, int trials, renyi_mre_cell* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(out, "out");
        const rb::MreCell c = rb::measure_cell(ctx->ctx, *k->k, exact_entropy, to_params(p), trials);
        out->alpha = c.alpha, out->s = c.s, out->m = c.m, out->method = c.method;
        out->mre = c.mre, out->sd = c.sd, out->mean_elapsed = c.mean_elapsed, out->trials = c.trials;
    });
}

int renyi_entropy_int(renyi_ctx* ctx, const renyi_kernel* k, int alpha, int s, uint64_t seed,
                      renyi_entropy_estimate* out) {
    renyi_estimator_params p;
    renyi_default_params(&p);
    p.alpha = alpha, p.method = RENYI_METHOD_INT, p.s = s, p.seed = seed;
    if (alpha < 2) {
        g_last_error = "entropy_int needs integer alpha >= 2";
        return RENYI_E_INVALID_ARGUMENT;
    }
    return renyi_estimate(ctx, k, &p, out);
}

int renyi_entropy_taylor(renyi_ctx* ctx, const renyi_kernel* k, double alpha, int s, int m, double v,
                         uint64_t seed, renyi_entropy_estimate* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(out, "out");
        rb::validate_alpha(alpha);
        rb::require_non_integer(alpha, "entropy_taylor");
        const int m_min = static_cast<int>(std::ceil(alpha)) + 1;
        if (m < m_min)
            rb::fail(rb::kInvalidArgument, "entropy_taylor needs m >= ceil(alpha)+1 = " + std::to_string(m_min));
        rb::EstParams p;
        p.alpha = alpha, p.method = rb::kMethodTaylor, p.s = s, p.m = m, p.seed = seed;
        p.has_bounds = true;
        p.bounds.v = v;
        p.bounds.u = 0.0;
        rb::EntropyEst e = rb::estimate(ctx->ctx, *k->k, p);
        e.has_bounds = false;
        from_entropy(e, out);
    });
}

int renyi_entropy_chebyshev(renyi_ctx* ctx, const renyi_kernel* k, double alpha, int s, int m, double u, double v,
                            uint64_t seed, renyi_entropy_estimate* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(k, "kernel"), need(out, "out");
        rb::validate_alpha(alpha);
        rb::require_non_integer(alpha, "entropy_chebyshev");
        rb::EstParams p;
        p.alpha = alpha, p.method = rb::kMethodChebyshev, p.s = s, p.m = m, p.seed = seed;
        p.has_bounds = true;
        p.bounds.u = u;
        p.bounds.v = v;
        rb::EntropyEst e = rb::estimate(ctx->ctx, *k->k, p);
        e.has_bounds = false;
        from_entropy(e, out);
    });
}

int renyi_mutual_information(renyi_ctx* ctx, const renyi_kernel* a, const renyi_kernel* b,
                             const renyi_estimator_params* p, renyi_mi_estimate* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(a, "kernel a"), need(b, "kernel b"), need(out, "out");
        const rb::MutualInfo mi = rb::mutual_information(ctx->ctx, *a->k, *b->k, to_params(p));
        out->value = mi.value, out->vars_entropy = mi.vars_entropy;
        out->target_entropy = mi.target_entropy, out->joint_entropy = mi.joint_entropy;
    });
}

int renyi_mutual_information_samples(renyi_ctx* ctx, const double* x, int64_t n, int64_t dx, int64_t ldx,
                                     double sigma_x, const double* y, int64_t dy, int64_t ldy, double sigma_y,
                                     const renyi_estimator_params* p, int precision, renyi_mi_estimate* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(x, "samples"), need(y, "target samples"), need(out, "out");
        check_precision(precision);
        const rb::MutualInfo mi = rb::mutual_information_samples(ctx->ctx, x, n, dx, ldx, sigma_x, y, dy, ldy,
                                                                 sigma_y, to_params(p), precision);
        out->value = mi.value, out->vars_entropy = mi.vars_entropy;
        out->target_entropy = mi.target_entropy, out->joint_entropy = mi.joint_entropy;
    });
}

int renyi_mutual_information_samples_dev(renyi_ctx* ctx, const double* d_x, int64_t n, int64_t dx, int64_t ldx,
                                         double sigma_x, const double* d_y, int64_t dy, int64_t ldy, double sigma_y,
                                         const renyi_estimator_params* p, int precision, renyi_mi_estimate* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(d_x, "samples"), need(d_y, "target samples"), need(out, "out");
        check_precision(precision);
        const rb::MutualInfo mi = rb::mutual_information_samples_dev(ctx->ctx, d_x, n, dx, ldx, sigma_x, d_y, dy, ldy,
                                                                     sigma_y, to_params(p), precision);
        out->value = mi.value, out->vars_entropy = mi.vars_entropy;
        out->target_entropy = mi.target_entropy, out->joint_entropy = mi.joint_entropy;
    });
}

int renyi_entropy_dev(renyi_ctx* ctx, const double* d_x, int64_t n, int64_t d, int64_t ldx, double sigma,
                      const renyi_estimator_params* p, int precision, renyi_entropy_estimate* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(d_x, "samples"), need(out, "out");
        check_precision(precision);
        rb::KernelPtr k = rb::build_gaussian_dev(ctx->ctx, d_x, n, d, ldx, sigma, precision);
        from_entropy(rb::estimate(ctx->ctx, *k, to_params(p)), out);
    });
}

int renyi_entropy(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double sigma,
                  const renyi_estimator_params* p, int precision, renyi_entropy_estimate* out) {
    return guarded([&] {
        need(ctx, "ctx"), need(x, "samples"), need(out, "out");
        check_precision(precision);
        rb::KernelPtr k = rb::build_gaussian(ctx->ctx, x, n, d, ldx, sigma, precision);
        from_entropy(rb::estimate(ctx->ctx, *k, to_params(p)), out);
    });
}

// ---- host arithmetic ----
void renyi_default_power_options(renyi_power_options* o) {
    if (!o) return;
    o->max_iters = 100;
    o->tol = 1e-6;
    o->seed = 0;
    o->rank_floor = 1e-12;
}

void renyi_default_params(renyi_estimator_params* p) {
    if (!p) return;
    std::memset(p, 0, sizeof(*p));
    p->alpha = 2.0;
    p->method = RENYI_METHOD_AUTO;
    p->epsilon = 1e-2;
    p->delta = 1e-2;
    renyi_default_power_options(&p->power);
    p->bounds.v = 1.0;
    p->bounds.kappa = INFINITY;
    p->bounds.v_converged = p->bounds.u_converged = 1;
    p->probe_kind = RENYI_PROBE_GAUSSIAN;
    p->s_q = p->s_g = -1;
}

uint64_t renyi_mix64(uint64_t x) { return rb::mix64(x); }
uint64_t renyi_derive_key(uint64_t seed, uint64_t tag) { return rb::derive_key(seed, tag); }
uint64_t renyi_hash_name(const char* name) { return name ? rb::hash_name(name) : 0; }

int renyi_probe_panel(int64_t n, int cols, uint64_t seed, const char* label, int kind, double* out) {
    return guarded([&] {
        need(label, "label"), need(out, "out");
        if (n < 0 || cols < 0) rb::fail(rb::kInvalidArgument, "negative panel size");
        rb::probe_panel(n, cols, seed, label, kind, out);
    });
}

namespace {
rb::FeatureData feature_data(const double* x, int64_t n, int64_t d, int64_t ldx, const char* const* labels,
                             int64_t n_labels, const char* const* names) {
    need(x, "x");
    if (n_labels > 0) need(labels, "labels");
    rb::FeatureData data;
    data.x = x, data.n = n, data.d = d, data.ldx = ldx;
    for (int64_t i = 0; i < n_labels; ++i) {
        need(labels[i], "label");
        data.labels.emplace_back(labels[i]);
    }
    if (names)
        for (int64_t j = 0; j < d; ++j) data.names.emplace_back(names[j] ? names[j] : "");
    return data;
}
}  // namespace

int renyi_rank_features(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                        const char* const* labels, int64_t n_labels, const char* const* names, double sigma,
                        const renyi_estimator_params* p, int precision, int k, int* columns, double* scores,
                        double* elapsed) {
    return guarded([&] {
        need(ctx, "ctx"), need(columns, "columns"), need(scores, "scores");
        check_precision(precision);
        const rb::FeatureRanking r = rb::rank_features(
            ctx->ctx, feature_data(x, n, d, ldx, labels, n_labels, names), sigma, to_params(p), precision, k);
        std::copy(r.columns.begin(), r.columns.end(), columns);
        std::copy(r.scores.begin(), r.scores.end(), scores);
        if (elapsed) std::copy(r.elapsed.begin(), r.elapsed.end(), elapsed);
    });
}

int renyi_select_features(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                          const char* const* labels, int64_t n_labels, const char* const* names, double sigma,
                          const renyi_estimator_params* p, int precision, int k, int* columns, double* objective,
                          double* elapsed) {
    return guarded([&] {
        need(ctx, "ctx"), need(columns, "columns"), need(objective, "objective");
        check_precision(precision);
        const rb::FeatureSelection r = rb::select_features(
            ctx->ctx, feature_data(x, n, d, ldx, labels, n_labels, names), sigma, to_params(p), precision, k);
        std::copy(r.columns.begin(), r.columns.end(), columns);
        std::copy(r.objective.begin(), r.objective.end(), objective);
        if (elapsed) std::copy(r.elapsed.begin(), r.elapsed.end(), elapsed);
    });
}

int renyi_mixture_samples(int n, int d, uint64_t seed, double center, double* out) {
    // proj/src/simulate.cpp:9-17: one stream, row by row; out column-major n x d
    return guarded([&] {
        need(out, "out");
        if (n < 0 || d < 0) rb::fail(rb::kInvalidArgument, "negative sample size");
        rb::RandomStream st(rb::derive_key(seed, rb::hash_name("mixture")));
        for (int i = 0; i < n; ++i) {
            const double mu = (st.next_u64() & 1) ? center : -center;
            for (int j = 0; j < d; ++j) out[i + static_cast<int64_t>(j) * n] = mu + st.next_gaussian();
        }
    });
}

int renyi_binomial_coeffs(double alpha, int m, double* out) {
    return guarded([&] {
        need(out, "out");
        const auto b = rb::binomial_coeffs(alpha, m);
        std::copy(b.begin(), b.end(), out);
    });
}

int renyi_chebyshev_coeffs(double alpha, int m, double u, double v, double* out) {
    return guarded([&] {
        need(out, "out");
        const auto c = rb::chebyshev_power_coeffs(alpha, m, u, v);
        std::copy(c.begin(), c.end(), out);
    });
}

struct renyi_rng {
    rb::RandomStream s;
};

int renyi_rng_create(uint64_t key, renyi_rng** out) {
    return guarded([&] {
        need(out, "out");
        *out = new renyi_rng{rb::RandomStream(key)};
    });
}
int renyi_rng_destroy(renyi_rng* r) {
    delete r;
    return 0;
}
int renyi_rng_derive(const renyi_rng* r, uint64_t tag, renyi_rng** out) {
    return guarded([&] {
        need(r, "rng"), need(out, "out");
        *out = new renyi_rng{r->s.derive(tag)};
    });
}
uint64_t renyi_rng_key(const renyi_rng* r) { return r ? r->s.key() : 0; }
uint64_t renyi_rng_next_u64(renyi_rng* r) { return r ? r->s.next_u64() : 0; }
double renyi_rng_next_uniform(renyi_rng* r) { return r ? r->s.next_uniform() : 0.0; }
double renyi_rng_next_gaussian(renyi_rng* r) { return r ? r->s.next_gaussian() : 0.0; }
int renyi_rng_fill_gaussian(renyi_rng* r, int64_t rows, int64_t cols, double* out) {
    return guarded([&] {
        need(r, "rng"), need(out, "out");
        if (rows < 0 || cols < 0) rb::fail(rb::kInvalidArgument, "fill sizes must be non-negative");
        for (int64_t j = 0; j < cols; ++j)  // rng.cpp:60-64: column-wise
            for (int64_t i = 0; i < rows; ++i) out[i + j * rows] = r->s.next_gaussian();
    });
}

int renyi_chebyshev_node_coeffs(renyi_scalar_fn f, void* user, int m, double a, double b, double* out) {
    return guarded([&] {
        need(reinterpret_cast<const void*>(f), "f"), need(out, "out");
        const auto c = rb::chebyshev_node_coeffs([&](double x) { return f(x, user); }, m, a, b);
        std::copy(c.begin(), c.end(), out);
    });
}

const char* renyi_method_name(int method) {
    switch (method) {
        case RENYI_METHOD_EXACT: return "exact";
        case RENYI_METHOD_INT: return "int";
        case RENYI_METHOD_TAYLOR: return "taylor";
        case RENYI_METHOD_CHEBYSHEV: return "chebyshev";
        case RENYI_METHOD_AUTO: return "auto";
        default: return "?";
    }
}

double renyi_chebyshev_safeguard(double u, double v) { return rb::chebyshev_safeguard(u, v); }
double renyi_taylor_tail_constant(double alpha, int k_max) { return rb::taylor_tail_constant(alpha, k_max); }

int renyi_matfun_scalar(const renyi_matfun* f, double lambda, double* out) {
    return guarded([&] {
        need(out, "out");
        *out = to_matfun(f).scalar_value(lambda);
    });
}

long renyi_expected_queries(const renyi_matfun* f, int s) {
    try {
        const rb::MatFun m = to_matfun(f);
        const long s_q = s / 4, s_g = s - 2 * (s / 4);
        return s_q + static_cast<long>(m.query_cost()) * (s_q + s_g) + 2 * s_g;
    } catch (const rb::Error& e) {
        g_last_error = e.what();
        return -1;
    }
}

int renyi_select_params(double alpha, double epsilon, double delta, const renyi_spectrum_bounds* b, int64_t n,
                        int method, int* s, int* m) {
    return guarded([&] {
        need(b, "bounds"), need(s, "s"), need(m, "m");
        const rb::SelectedParams sp = rb::select_params(alpha, epsilon, delta, to_bounds(*b), n, method);
        *s = sp.s, *m = sp.m;
    });
}

int renyi_mu_bound(double u, double v, double alpha, int64_t n, double* mu, double* lower, double* upper) {
    return guarded([&] {
        const rb::MuBoundH b = rb::mu_bound(u, v, alpha, n);
        if (mu) *mu = b.mu;
        if (lower) *lower = b.lower;
        if (upper) *upper = b.upper;
    });
}

int renyi_entropy_from_trace(double trace, double alpha, double* out) {
    return guarded([&] {
        need(out, "out");
        *out = rb::entropy_from_trace(trace, alpha);
    });
}

}  // extern "C"
