/*
 * renyi_b200.h — C ABI of the B200-native randomized matrix-based Rényi
 * entropy hot path (librenyi_b200.so).
 *
 * The reference (arxiv 2205.07426 artifact, proj/) has no FFI: its path sits
 * behind C++ value-semantic functions over Eigen matrices. Each entry point
 * below names the reference function it replaces (file:line, relative to the
 * reference's root). Conventions:
 *   - every call returns an int status: 0 = ok, 1..10 = the reference's errc
 *     kinds + 1 (proj/include/renyi/common.hpp:14-25), 20+ = device/runtime;
 *     renyi_last_error() returns the thread's last message;
 *   - host matrices are column-major (the reference's Eigen layout) with an
 *     explicit leading dimension where noted; kernels (A) are symmetric n x n;
 *   - device state lives behind opaque handles; the caller owns host buffers.
 * Statuses 1,4,5,8,10 are "usage" errors (reference CLI exit 2), the others
 * numerical/runtime (exit 3) — see proj/include/renyi/common.hpp:33-44.
 */
#ifndef RENYI_B200_H
#define RENYI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
enum {
    RENYI_OK = 0,
    RENYI_E_INVALID_ARGUMENT = 1,
    RENYI_E_ZERO_DIAGONAL = 2,
    RENYI_E_NON_FINITE = 3,
    RENYI_E_SIZE_MISMATCH = 4,
    RENYI_E_DOMAIN_ERROR = 5,
    RENYI_E_RANK_COLLAPSE = 6,
    RENYI_E_NON_POSITIVE_TRACE = 7,
    RENYI_E_ALPHA_IS_ONE = 8,
    RENYI_E_DEGENERATE_BOUNDS = 9,
    RENYI_E_PARSE_ERROR = 10,
    RENYI_E_CUDA = 20,
    RENYI_E_NCCL = 21,
    RENYI_E_OOM = 22,
    RENYI_E_NO_DEVICE = 23,
    RENYI_E_INTERNAL = 24
};

/* storage/compute precision of a device kernel matrix. RENYI_MF ("matrix-free") never
 * stores A: each pass recomputes K(x_i, x_j) from bf16 samples on the tensor cores
 * (fp32 accumulation, fp16 kernel values into an fp32-accumulated product). It is built
 * from samples only (renyi_kernel_build_gaussian*, the *_samples and entropy entry
 * points); renyi_kernel_from_matrix / _hadamard_joint / _download reject it. */
enum { RENYI_F64 = 0, RENYI_F32 = 1, RENYI_MF = 2 };
/* fp32 configurations: iterate operand of the block product. SPLIT (default) keeps V as an
 * fp16 hi+lo pair (3 tensor-core products, ~fp32 accuracy per product); FAST rounds V to
 * one fp16 plane (2 products); AUTO uses SPLIT where product vectors are returned
 * (matmul_panel, apply_panel, the Hutch++ sketch) and FAST for trace-only passes. FAST and
 * AUTO are ~10 % faster on config 4 but can miss the 1e-4 trace bar at small probe counts
 * (DESIGN.md). */
enum { RENYI_OPERAND_SPLIT = 0, RENYI_OPERAND_FAST = 1, RENYI_OPERAND_AUTO = 2 };
/* probe distributions */
enum { RENYI_PROBE_GAUSSIAN = 0, RENYI_PROBE_RADEMACHER = 1 };
/* estimator methods (renyi::Method, proj/include/renyi/entropy.hpp:12) */
enum { RENYI_METHOD_EXACT = 0, RENYI_METHOD_INT = 1, RENYI_METHOD_TAYLOR = 2, RENYI_METHOD_CHEBYSHEV = 3,
       RENYI_METHOD_AUTO = 4 };
/* matrix functions (renyi::MatrixFunctionSpec, proj/include/renyi/poly.hpp:32-70) */
enum { RENYI_MATFUN_INT_POWER = 0, RENYI_MATFUN_TAYLOR = 1, RENYI_MATFUN_CHEBYSHEV = 2 };

typedef struct renyi_ctx renyi_ctx;
typedef struct renyi_kernel renyi_kernel;
typedef struct renyi_local_group renyi_local_group;

/* MatrixFunctionSpec::{int_power,taylor,chebyshev} arguments; coefficients
 * (binomials, Chebyshev node sums, safeguard) are derived inside exactly as the
 * reference factories do (proj/src/poly.cpp:60-80). */
typedef struct {
    int kind;     /* RENYI_MATFUN_* */
    double alpha; /* integer value for INT_POWER */
    int degree;   /* m (ignored for INT_POWER) */
    double u, v;  /* Taylor uses v; Chebyshev uses [u, v] before the safeguard */
} renyi_matfun;

/* SketchConfig + probe injection (proj/include/renyi/hutchpp.hpp:12-18). */
typedef struct {
    int s_q, s_g;          /* sketch / residual probe columns (s_q = 0: plain Hutchinson) */
    uint64_t seed;
    int probe_kind;        /* RENYI_PROBE_* when the probes are drawn from the seed */
    const double* sketch;  /* optional n x s_q column-major (NULL: draw) */
    const double* probes;  /* optional n x s_g column-major (NULL: draw) */
} renyi_sketch;

typedef struct { /* TraceEstimate, proj/include/renyi/hutchpp.hpp:20-30 */
    double value, low_rank_part, residual_part;
    int queries_used, sketch_rank, exact;
} renyi_trace_estimate;

typedef struct { /* PowerOptions, proj/include/renyi/spectrum.hpp:22-30 */
    int max_iters;
    double tol;
    uint64_t seed;
    double rank_floor;
} renyi_power_options;

typedef struct { /* SpectrumBounds, proj/include/renyi/spectrum.hpp:12-20 */
    double u, v, kappa;
    int iterations_used, v_converged, u_converged, rank_deficient;
} renyi_spectrum_bounds;

typedef struct { /* PowerResult, proj/include/renyi/spectrum.hpp:35-39 */
    double rayleigh;
    int iterations, converged;
} renyi_power_result;

typedef struct { /* EstimatorParams, proj/include/renyi/entropy.hpp:18-30 (+ probe/split extensions) */
    double alpha;
    int method;
    int s, m;
    double epsilon, delta;
    uint64_t seed;
    renyi_power_options power;
    int has_bounds;
    renyi_spectrum_bounds bounds;
    int probe_kind; /* RENYI_PROBE_*; the reference draws Gaussian probes */
    int s_q, s_g;   /* explicit Hutch++ split; -1 = reference split floor(s/4), s - 2 floor(s/4) */
} renyi_estimator_params;

typedef struct { /* EntropyEstimate, proj/include/renyi/entropy.hpp:32-41 */
    double entropy, trace_estimate;
    int method_used, s_used, m_used;
    int has_bounds;
    renyi_spectrum_bounds bounds_used;
    double elapsed;
    int deterministic;
    renyi_trace_estimate trace;
} renyi_entropy_estimate;

typedef struct { /* MreCell, proj/include/renyi/simulate.hpp:27-37 (oracle_elapsed stays with the caller) */
    double alpha;
    int s, m, method;
    double mre, sd, mean_elapsed; /* mean_elapsed: batched wall time / trials */
    int trials;
} renyi_mre_cell;

typedef struct { /* MutualInformation, proj/include/renyi/measures.hpp:24-29 */
    double value, vars_entropy, target_entropy, joint_entropy;
} renyi_mi_estimate;

/* ---- errors, context ---------------------------------------------------- */
const char* renyi_last_error(void);
int renyi_status_is_usage(int status); /* renyi::error::is_usage, common.hpp:33-44 */
int renyi_ctx_create(int device, renyi_ctx** out);
int renyi_ctx_destroy(renyi_ctx* ctx);
int renyi_ctx_set_tuning(renyi_ctx* ctx, int grid, int kc);
int renyi_ctx_set_operand_mode(renyi_ctx* ctx, int mode);
/* mutual information over fp32 kernels: 1 (default) runs the three terms' passes fused, one read of
 * A and B per pass with the joint kernel n·A∘B formed on the fly (never stored); 0: three separate
 * estimates over a materialised joint (proj/src/measures.cpp:36-46) */
int renyi_ctx_set_fused_mi(renyi_ctx* ctx, int on);
/* rank_features / select_features over fp32 kernels: 1 (default) scores the candidates of a step as
 * grouped stacks (one block product per pass for up to 64 candidates' kernels); 0: one
 * candidate at a time, as the reference's loop (proj/src/features.cpp:95-162) */
int renyi_ctx_set_feature_grouping(renyi_ctx* ctx, int on);
/* seeded Gaussian probes (detail::gaussian_panel, proj/src/hutchpp.cpp:13-22): RENYI_PROBES_DEVICE
 * (default) draws them on the device from the reference's substreams with CUDA's log/sin/cos (<= 2 ulp
 * per draw from glibc's); RENYI_PROBES_HOST draws them with the reference's own arithmetic on the host
 * threads (bitwise the reference's probes) and copies them; mutual information requests its panels
 * before the kernel builds so the host work overlaps them. Rademacher probes are exact either way. */
#define RENYI_PROBES_DEVICE 0
#define RENYI_PROBES_HOST 1
int renyi_ctx_set_probe_source(renyi_ctx* ctx, int source);
/* matrix-free product: j-blocks (of 128 samples) accumulated in TMEM before each fp32 drain */
int renyi_ctx_set_matrix_free_chunk(renyi_ctx* ctx, int jblocks);
int renyi_ctx_sync(renyi_ctx* ctx);
/* returns the engine's cached device blocks (kernel storage, panels, scratch) to the driver */
int renyi_release_cached_memory(void);
/* CUDA-event timing of block-product launches with their algorithmic bytes and
 * flops (SURVEY §8d accounting); bench instrumentation */
int renyi_ctx_profile(renyi_ctx* ctx, int enable);
int renyi_ctx_profile_read(renyi_ctx* ctx, int* launches, double* milliseconds, double* bytes, double* flops);
int renyi_ctx_launch_count(renyi_ctx* ctx, long* launches);
/* host<->device bytes issued by the engine since creation */
int renyi_ctx_io_bytes(renyi_ctx* ctx, long long* h2d, long long* d2h);
/* CUDA-event region timer on the engine stream */
int renyi_ctx_timer_begin(renyi_ctx* ctx);
int renyi_ctx_timer_end(renyi_ctx* ctx, double* milliseconds);

/* ---- multi-rank (row-sharded A) -------------------------------
 * One context per rank. After joining, kernel matrices built on the context hold
 * rows [row0, row0+rows) of A and every estimator call is collective over the
 * group (same arguments on every rank; results identical on every rank). */
int renyi_shard_rows(int64_t n, int world, int rank, int64_t* row0, int64_t* rows, int64_t* rows_per_rank);
int renyi_nccl_unique_id(unsigned char id[128]);
int renyi_ctx_init_nccl(renyi_ctx* ctx, int rank, int world, const unsigned char id[128]);
/* ranks as threads of one process (host-driven collectives; any devices) */
int renyi_local_group_create(int world, renyi_local_group** out);
int renyi_local_group_destroy(renyi_local_group* g);
int renyi_ctx_join_local_group(renyi_ctx* ctx, renyi_local_group* g, int rank);
int renyi_ctx_rank(renyi_ctx* ctx, int* rank, int* world);

/* ---- kernel matrices (proj/include/renyi/kernel.hpp:45-56) --------------- */
/* build_kernel(X, GaussianKernel{sigma}) — proj/src/kernel.cpp:35-72 + ops.cpp:39-47 */
int renyi_kernel_build_gaussian(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double sigma,
                                int precision, renyi_kernel** out);
/* hadamard_joint({build_kernel(X), build_kernel(Y)}) fused from samples — kernel.cpp:74-101 */
int renyi_kernel_build_gaussian_joint(renyi_ctx* ctx, const double* x, int64_t n, int64_t dx, int64_t ldx,
                                      double sigma_x, const double* y, int64_t dy, int64_t ldy, double sigma_y,
                                      int precision, renyi_kernel** out);
/* the same from device-resident samples (column-major, leading dimension ldx; y may be NULL) */
int renyi_kernel_build_gaussian_dev(renyi_ctx* ctx, const double* d_x, int64_t n, int64_t d, int64_t ldx,
                                    double sigma, const double* d_y, int64_t dy, int64_t ldy, double sigma_y,
                                    int precision, renyi_kernel** out);
/* build_kernel(X, PolynomialKernel{degree, offset}) — proj/src/kernel.cpp:35-72 + ops.cpp:22-28,58-64:
 * K_ij = pow(x_i·x_j + offset, degree) in fp64, A_ij = K_ij / (n sqrt(K_ii K_jj)); RENYI_F64 or
 * RENYI_F32 (stored as the split every fp32 product consumes); errors as the reference's: degree < 1
 * or offset < 0 invalid_argument, non-finite kernel values non_finite, K_ii <= 0 zero_diagonal */
int renyi_kernel_build_polynomial(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int degree,
                                  double offset, int precision, renyi_kernel** out);
int renyi_kernel_build_polynomial_dev(renyi_ctx* ctx, const double* d_x, int64_t n, int64_t d, int64_t ldx,
                                      int degree, double offset, int precision, renyi_kernel** out);
/* NormalizedKernel(Matrix) — kernel.hpp:33 (caller asserts the invariants) */
int renyi_kernel_from_matrix(renyi_ctx* ctx, const double* a, int64_t n, int precision, renyi_kernel** out);
/* hadamard_joint({a, b}) — kernel.cpp:74-101 */
int renyi_kernel_hadamard_joint(renyi_ctx* ctx, const renyi_kernel* a, const renyi_kernel* b, renyi_kernel** out);
/* hadamard_joint(kernels) for count >= 2 (kernel.cpp:74-101): factors in a canonical content order, so
 * any permutation of the list gives a bitwise identical joint; n^(count-1) applied once, diag 1/n;
 * count >= 3 is single-rank */
int renyi_kernel_hadamard_joint_n(renyi_ctx* ctx, const renyi_kernel* const* kernels, int count,
                                  renyi_kernel** out);
int renyi_kernel_size(const renyi_kernel* k, int64_t* n);
int renyi_kernel_download(renyi_ctx* ctx, const renyi_kernel* k, double* out);
int renyi_kernel_destroy(renyi_kernel* k);

/* ---- CSV ingestion feeding device X -----------------------------------------
 * renyi::load_csv(path, label_column) — proj/src/csv.cpp:63-115, proj/include/renyi/csv.hpp:8-15
 * (Dataset: proj/include/renyi/features.hpp:12-19). The bytes are parsed on the device: a quote-aware
 * structural scan (read_record, csv.cpp:13-47) and a strtod-exact cell parse (parse_cell, 49-60);
 * the n x d features stay resident for renyi_kernel_build_gaussian_dataset. Errors and their texts
 * are the reference's (RENYI_E_PARSE_ERROR): "cannot open 'p'", "'p': missing header row",
 * "'p': no column named 'c'", "row R: expected H fields, got F", "row R, column C: 't' is not
 * numeric", "'p': need at least 2 data rows, got K". label_column may be NULL. */
typedef struct renyi_dataset renyi_dataset;
int renyi_csv_load(renyi_ctx* ctx, const char* path, const char* label_column, renyi_dataset** out);
/* the same from a host buffer; source names the input in messages (NULL: "<buffer>") */
int renyi_csv_parse(renyi_ctx* ctx, const char* text, int64_t len, const char* label_column, const char* source,
                    renyi_dataset** out);
int renyi_dataset_shape(const renyi_dataset* ds, int64_t* n, int64_t* d, int* has_labels);
/* features (column-major, leading dimension ldx >= n) to a host buffer */
int renyi_dataset_features(renyi_ctx* ctx, const renyi_dataset* ds, double* x, int64_t ldx);
/* names[j] (j < d) and labels[i] (i < n); NULL when out of range */
const char* renyi_dataset_name(const renyi_dataset* ds, int64_t j);
const char* renyi_dataset_label(const renyi_dataset* ds, int64_t i);
/* build_kernel(data.features(:, columns), GaussianKernel{sigma}) from the resident features
 * (columns NULL: all d columns) */
int renyi_kernel_build_gaussian_dataset(renyi_ctx* ctx, const renyi_dataset* ds, const int64_t* columns,
                                        int64_t ncols, double sigma, int precision, renyi_kernel** out);
int renyi_dataset_destroy(renyi_dataset* ds);

/* ---- hot-path seams ------------------------------------------------------- */
/* ops::matmul_panel(a, x) — proj/src/ops.cpp:98-107: Y = A V, V n x s */
int renyi_matmul_panel(renyi_ctx* ctx, const renyi_kernel* k, const double* v, int s, double* y);
/* the raw ops seam (proj/include/renyi/ops.hpp:12-33) on host column-major matrices:
 * ops::gaussian_gram (ops.cpp:9-20,39-47): K n x n, K_ii = 1, exactly symmetric;
 * ops::polynomial_gram (ops.cpp:22-28,58-64): K_ij = pow(x_i·x_j + offset, degree);
 * ops::hadamard_scaled (ops.cpp:116-122): C = scale * (A ∘ B), rows x cols */
int renyi_ops_gaussian_gram(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double sigma,
                            double* k);
int renyi_ops_polynomial_gram(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, int degree,
                              double offset, double* k);
int renyi_ops_hadamard_scaled(renyi_ctx* ctx, const double* a, const double* b, int64_t rows, int64_t cols,
                              double scale, double* c);
/* ops::matvec(a, x) — proj/src/ops.cpp:73-85 */
int renyi_matvec(renyi_ctx* ctx, const renyi_kernel* k, const double* x, double* y);
/* apply_panel(spec, a, x) — proj/src/poly.cpp:158-164 */
int renyi_apply_panel(renyi_ctx* ctx, const renyi_kernel* k, const renyi_matfun* f, const double* v, int s,
                      double* y);
/* fused x_j^T f(A) x_j per column (projected_trace without the vector) — hutchpp.cpp:33-39.
 * Every trace-only entry point (this, renyi_hutchpp, renyi_estimate, the entropy, MI, trials and
 * feature entry points) forms the quadratic forms of a degree-m polynomial from ceil(m/2) passes
 * over A by moment doubling (A symmetric); renyi_apply_panel runs all m. */
int renyi_matfun_traces(renyi_ctx* ctx, const renyi_kernel* k, const renyi_matfun* f, const double* x, int s,
                        double* traces);

/* ---- estimators ------------------------------------------------------------- */
/* power_method — proj/src/spectrum.cpp:25-49 (shift = 0: A, else shift*I - A) */
int renyi_power_method(renyi_ctx* ctx, const renyi_kernel* k, const renyi_power_options* opts, double shift,
                       renyi_power_result* out);
/* estimate_bounds — proj/src/spectrum.cpp:80-103 */
int renyi_estimate_bounds(renyi_ctx* ctx, const renyi_kernel* k, const renyi_power_options* opts,
                          renyi_spectrum_bounds* out);
/* hutchpp — proj/src/hutchpp.cpp:69-115 */
int renyi_hutchpp(renyi_ctx* ctx, const renyi_kernel* k, const renyi_matfun* f, const renyi_sketch* cfg,
                  renyi_trace_estimate* out);
/* estimate — proj/src/entropy.cpp:201-275 */
int renyi_estimate(renyi_ctx* ctx, const renyi_kernel* k, const renyi_estimator_params* p,
                   renyi_entropy_estimate* out);
/* K trials of estimate() with seeds derive_key(p->seed, t), bounds resolved once, as measure_cell
 * runs them (proj/src/simulate.cpp:19-51); the probes of all trials share the passes over A.
 * out[trials]. */
int renyi_estimate_trials(renyi_ctx* ctx, const renyi_kernel* k, const renyi_estimator_params* p, int trials,
                          renyi_entropy_estimate* out);
/* measure_cell — proj/src/simulate.cpp:19-72 (MRE/SD over K trials against a known exact entropy) */
int renyi_measure_cell(renyi_ctx* ctx, const renyi_kernel* k, double exact_entropy,
                       const renyi_estimator_params* p, int trials, renyi_mre_cell* out);
/* rank_features / select_features — proj/src/features.cpp:95-162 (Gaussian kernel of width sigma
 * for every feature and for the one-hot labels; names may be NULL -> "feature_<j>").
 * rank: columns[k], scores[k], elapsed[d]. select: columns[k], objective[k], elapsed[k]. */
int renyi_rank_features(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                        const char* const* labels, int64_t n_labels, const char* const* names, double sigma,
                        const renyi_estimator_params* p, int precision, int k, int* columns, double* scores,
                        double* elapsed);
int renyi_select_features(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx,
                          const char* const* labels, int64_t n_labels, const char* const* names, double sigma,
                          const renyi_estimator_params* p, int precision, int k, int* columns, double* objective,
                          double* elapsed);
/* mixture_samples — proj/src/simulate.cpp:9-17 (host; out column-major n x d) */
int renyi_mixture_samples(int n, int d, uint64_t seed, double center, double* out);
/* entropy_int / entropy_taylor / entropy_chebyshev — proj/src/entropy.cpp:111-135 */
int renyi_entropy_int(renyi_ctx* ctx, const renyi_kernel* k, int alpha, int s, uint64_t seed,
                      renyi_entropy_estimate* out);
int renyi_entropy_taylor(renyi_ctx* ctx, const renyi_kernel* k, double alpha, int s, int m, double v,
                         uint64_t seed, renyi_entropy_estimate* out);
int renyi_entropy_chebyshev(renyi_ctx* ctx, const renyi_kernel* k, double alpha, int s, int m, double u, double v,
                            uint64_t seed, renyi_entropy_estimate* out);
/* mutual_information({a}, b, params) — proj/src/measures.cpp:36-46 */
int renyi_mutual_information(renyi_ctx* ctx, const renyi_kernel* a, const renyi_kernel* b,
                             const renyi_estimator_params* p, renyi_mi_estimate* out);
/* the same from samples, one n x n matrix resident at a time (cmd_mutual_info, renyi_cli.cpp:156-188) */
int renyi_mutual_information_samples(renyi_ctx* ctx, const double* x, int64_t n, int64_t dx, int64_t ldx,
                                     double sigma_x, const double* y, int64_t dy, int64_t ldy, double sigma_y,
                                     const renyi_estimator_params* p, int precision, renyi_mi_estimate* out);
int renyi_mutual_information_samples_dev(renyi_ctx* ctx, const double* d_x, int64_t n, int64_t dx, int64_t ldx,
                                         double sigma_x, const double* d_y, int64_t dy, int64_t ldy, double sigma_y,
                                         const renyi_estimator_params* p, int precision, renyi_mi_estimate* out);
/* north star: build_kernel(X, sigma) + estimate(A, params) (cmd_entropy, renyi_cli.cpp:144-154) */
int renyi_entropy(renyi_ctx* ctx, const double* x, int64_t n, int64_t d, int64_t ldx, double sigma,
                  const renyi_estimator_params* p, int precision, renyi_entropy_estimate* out);
int renyi_entropy_dev(renyi_ctx* ctx, const double* d_x, int64_t n, int64_t d, int64_t ldx, double sigma,
                      const renyi_estimator_params* p, int precision, renyi_entropy_estimate* out);

/* ---- host-side arithmetic (no device) ------------------------------------------ */
void renyi_default_params(renyi_estimator_params* p);      /* EstimatorParams{} defaults */
void renyi_default_power_options(renyi_power_options* o);  /* PowerOptions{} defaults */
uint64_t renyi_mix64(uint64_t x);                            /* rng.cpp:8-14 */
uint64_t renyi_derive_key(uint64_t seed, uint64_t tag);      /* rng.cpp:16-18 */
uint64_t renyi_hash_name(const char* name);                  /* rng.cpp:20-28 */
/* detail::gaussian_panel (hutchpp.cpp:13-22); kind RENYI_PROBE_RADEMACHER = sign of the top bit */
int renyi_probe_panel(int64_t n, int cols, uint64_t seed, const char* label, int kind, double* out);
/* RandomStream (proj/include/renyi/rng.hpp:12-36, rng.cpp:30-64): counter-based splitmix stream,
 * Box-Muller normals with the spare, column-wise fills (prefix-stable in the column count) */
typedef struct renyi_rng renyi_rng;
int renyi_rng_create(uint64_t key, renyi_rng** out);
int renyi_rng_destroy(renyi_rng* r);
int renyi_rng_derive(const renyi_rng* r, uint64_t tag, renyi_rng** out);
uint64_t renyi_rng_key(const renyi_rng* r);
uint64_t renyi_rng_next_u64(renyi_rng* r);
double renyi_rng_next_uniform(renyi_rng* r);
double renyi_rng_next_gaussian(renyi_rng* r);
int renyi_rng_fill_gaussian(renyi_rng* r, int64_t rows, int64_t cols, double* out); /* column-major */
int renyi_binomial_coeffs(double alpha, int m, double* out);                   /* poly.cpp:10-16 */
int renyi_chebyshev_coeffs(double alpha, int m, double u, double v, double* out); /* poly.cpp:42-46 */
/* chebyshev_node_coeffs(f, m, a, b) (poly.cpp:18-40) for a caller-supplied f: out has m + 1 entries */
typedef double (*renyi_scalar_fn)(double x, void* user);
int renyi_chebyshev_node_coeffs(renyi_scalar_fn f, void* user, int m, double a, double b, double* out);
/* method_name (entropy.cpp:51-60): "exact", "int", "taylor", "chebyshev", "auto" ("?" otherwise) */
const char* renyi_method_name(int method);
double renyi_chebyshev_safeguard(double u, double v);                           /* poly.hpp:27-30 */
double renyi_taylor_tail_constant(double alpha, int k_max);                     /* poly.cpp:48-58 */
int renyi_matfun_scalar(const renyi_matfun* f, double lambda, double* out);     /* poly.cpp:166-168 */
long renyi_expected_queries(const renyi_matfun* f, int s);                      /* hutchpp.cpp:117-121 */
int renyi_select_params(double alpha, double epsilon, double delta, const renyi_spectrum_bounds* b, int64_t n,
                        int method, int* s, int* m);                            /* entropy.cpp:137-176 */
int renyi_mu_bound(double u, double v, double alpha, int64_t n, double* mu, double* lower, double* upper);
int renyi_entropy_from_trace(double trace, double alpha, double* out);          /* entropy.cpp:62-69 */

#ifdef __cplusplus
}
#endif

#endif /* RENYI_B200_H */
