// Host-side declarations of the device kernels (launch wrappers). Layout
// conventions, shared by every kernel:
//   * kernel matrix A (n_local x n): row-major, pitch `ld` elements. The fp32
//     configurations store A as two fp16 planes (hi, lo) of A·n·2^14; the fp64
//     configuration stores A itself.
//   * panels (iterates, probes): column-major n x cols, column j at j*ld.
//   * product partials: [slot][npad][128] (tile-column-major) in fp32 / fp64.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace rb {

constexpr double kSplitScale = 16384.0;  // 2^14: A·n lies in [0,1]; stored planes hold A·n·2^14
constexpr int kSplitScaleLog2 = 14;
constexpr int kPanelTarget = 15;  // iterate planes are scaled so max|v| < 2^15 (fp16 max 65504)
constexpr int kMaxPanelCols = 128;

struct SplitMatrixView {
    const __half* hi;
    const __half* lo;
    int64_t rows, cols, ld;
};

// The iterate operand: fp16 hi (+ optional lo) planes laid out [world][cols][rpr]: rank w's
// rows of every column are contiguous (the all-gather output layout); global row k lives
// at chunk k / rpr, offset k % rpr. Single rank: [1][cols][rpr] = column-major with ld rpr.
struct SplitPanelView {
    const __half* v;
    const __half* vlo;  // nullptr: "fast" operand mode (one plane, two MMAs)
    int64_t n;
    int cols;
    int64_t rpr;  // rows per rank chunk (multiple of 256)
    int world;
    // grouped stacked matrices (feature tools, single rank): row block r of A belongs to group
    // r·rows_per_block / group_rows, whose operand rows sit at offset group·group_rows (0: one matrix)
    int64_t group_rows = 0;
    // elements between consecutive ranks' chunks (0: cols·rpr). Row-sharded sessions append a tail per
    // chunk that carries the rank's column maxima through the same all-gather (engine.cu gather_planes)
    int64_t slice = 0;
};

// cudaFuncAttributeMaxDynamicSharedMemorySize for `fn` on the current device, once per (fn, device);
// thread-safe (ranks may drive different devices from different host threads)
cudaError_t ensure_smem_attr(const void* fn, int bytes);

struct StreamKPlan {
    int row_blocks = 0;
    int k_tiles = 0;
    int64_t total_iters = 0;
    int grid = 1;
    int kc = 16;
    int slots = 0;
    int rows_per_block = 256;
    int cluster = 1;  // row blocks per stream-K participant (2: CTA pairs)
    // row blocks [0, dp_blocks) are owned whole, block r by CTA r % grid (data-parallel waves, slot r);
    // the remaining row blocks' iterations are split stream-K over the grid (slot r + CTA)
    int dp_blocks = 0;
    // K window of the launch: its k tile k is global tile (k_off + k) mod k_total (k_total 0: no window,
    // the launch covers every k tile). A row-sharded pass runs two windows: the rank's own chunk of the
    // operand (ready right after its epilogue) and the other ranks' chunks (after the all-gather).
    int k_off = 0;
    int k_total = 0;
};

// window [col0, col0 + cols) (columns of A = rows of the operand, wrapping at n) in a plan's k tiles
struct KWindow {
    int64_t col0 = 0;
    int64_t cols = -1;  // -1: all columns
};

// ---- symmetric single-column product (s = 1 passes, symv.cu) ---------------
// 128-row blocks of an n x n matrix
int64_t symv_blocks(int64_t n);
// partials of y = A·x from the upper triangle: slot I·nb + J holds block I's share from tile (I, J) or
// (J, I); partial [nb·nb][128] floats, one column
cudaError_t launch_symv_split(const SplitMatrixView& a, const __half* xhi, const __half* xlo, float* partial,
                              int grid, cudaStream_t stream);

// ---- block product -------------------------------------------------------
int tc_block_rows();
int tc_block_k();
int tc_npad(int cols);
// sets p.k_tiles / k_off / k_total for window w over n columns in tiles of `tile` columns
void apply_window(StreamKPlan& p, int64_t n, int tile, KWindow w);
StreamKPlan make_streamk_plan(int64_t rows, int64_t cols, int grid, int kc, KWindow w = {});
cudaError_t launch_block_av_tc(const SplitMatrixView& a, const SplitPanelView& v, const StreamKPlan& plan,
                               float* partial, cudaStream_t stream);
// fused mutual-information pass: Y_A = A·V[0], Y_B = B·V[1], Y_J = J·V[2] with J = n·(A∘B) (J_ii = 1/n)
// formed from the staged A and B tiles (stored J = factor·stored A·stored B, stored J_ii = diag);
// 128-row blocks (make_tri_plan), all three panels of the same width <= tri_max_cols()
StreamKPlan make_tri_plan(int64_t rows, int64_t cols, int grid, int kc, KWindow w = {});
int tri_max_cols();
cudaError_t launch_block_av_tri(const SplitMatrixView& a, const SplitMatrixView& b, const SplitPanelView* v,
                                const StreamKPlan& plan, float* const* partial, int64_t row0, double factor,
                                double diag, cudaStream_t stream);

// matrix-free: bf16 samples [n][dp] (dp = 64 or 128, zero padded) and negated bias −b = −c·|x|² [n_pad]
struct MfMatrixView {
    const __nv_bfloat16* x;   // bf16 samples [n][dp] (dp = 64 or 128, zero padded)
    const __nv_bfloat16* xa;  // augmented columns [2][npad][16]: row side, column side (block_av_mf.cu)
    int64_t n;
    int64_t npad;             // round_up(n, 128)
    int dp;
    int64_t row0;
    double c2;  // log2(e)/σ²
};
StreamKPlan make_mf_plan(int64_t rows, int64_t n, int grid, int kc, KWindow w = {});
int mf_aug_cols();
cudaError_t launch_block_av_mf(const MfMatrixView& a, const SplitPanelView& v, const StreamKPlan& plan,
                               float* partial, cudaStream_t stream);
// x (fp64, element (i,k) at x[i*rs + k*cs]) -> bf16 [n][dp] and the augmented columns
// carrying −|bf16(x)|²/2 as three bf16 terms
cudaError_t launch_mf_prepare(const double* x, int64_t n, int d, int64_t rs, int64_t cs, int dp, int64_t npad,
                              __nv_bfloat16* xb, __nv_bfloat16* xa, cudaStream_t stream);

StreamKPlan make_f64_plan(int64_t rows, int64_t cols, int grid);
int f64_npad(int cols);
cudaError_t launch_block_av_f64(const double* a, int64_t rows, int64_t cols, int64_t lda, const double* v, int s,
                                int64_t ldv, const StreamKPlan& plan, double* partial, cudaStream_t stream);

// ---- pass epilogue (recurrence + fused fp64 trace partials) --------------
template <typename PT, typename ST>
struct EpiArgs {
    const PT* partial;
    int npad;
    int64_t total_iters;
    int k_tiles;
    int grid;
    int cluster;   // slot(r, p) = cluster*(r/cluster + p) + r%cluster
    int dp_blocks;  // row blocks owned whole (slot r); stream-K over the rest (StreamKPlan)
    int64_t rows;  // local rows (product rows)
    int rows_per_block;  // 256 (tensor-core path) or 128 (fp64 path)
    int s;
    int64_t ld;
    const int* e_cur;  // split only
    int* e_next;       // split only
    double unscale;    // product scale: 2^-14/n (split) or 1
    const unsigned* cmax_cur;
    const unsigned* cmax_prev;  // may be null when a3 == 0
    unsigned* cmax_new;
    double a1, a2, a3;
    double a_norm;  // bound on max_i sum_j |A_ij|
    const ST* t_cur;
    const ST* t_prev;
    ST* t_new;
    const ST* x0;
    __half* vop;    // fp16 operand plane(s) for the next pass (split only)
    __half* vop_lo; // optional low plane (operand split mode)
    double* stats;  // [3][row_blocks][s]
    double* acc;    // optional vector accumulator (fp64, [s][ld])
    double acc_coef;
    // second K window of a row-sharded pass (the other ranks' operand chunks, see StreamKPlan::k_off):
    // its slots are summed after the first window's, in the same fixed order; partial2 == nullptr: none
    const PT* partial2 = nullptr;
    // symmetric single-column product (launch_symv_split): nb partial slots per row block, [I·nb, I·nb + nb)
    int64_t symv_nb = 0;
    // optional device scale of a1, a2, a3 (the power iteration's 1/||T||, computed on the device from the
    // previous pass's dots so the next pass can be queued before the host reads them)
    const double* gscale = nullptr;
    int64_t total_iters2 = 0;
    int k_tiles2 = 0;
    int grid2 = 1;
    int dp_blocks2 = 0;
};

cudaError_t launch_epilogue_split(const EpiArgs<float, float>& a, cudaStream_t stream);
// g = 1 / sqrt(red[2]) (red: one pass's [3][1] dots): the power iteration's next normalisation
cudaError_t launch_power_norm(const double* red, double* g, cudaStream_t stream);
cudaError_t launch_epilogue_f64(const EpiArgs<double, double>& a, cudaStream_t stream);

// T0 <- X0 (fp64 input); stats[0] and cmax[0]; then planes with exponent e0.
template <typename ST>
struct PrepArgs {
    const double* x;  // [s][ldx]
    int64_t ldx;
    int64_t rows;
    int rows_per_block;
    int s;
    int64_t ld;
    ST* t0;
    unsigned* cmax0;
    double* stats;  // [3][row_blocks][s]
    int* e0;
    __half* vop;
    __half* vop_lo;
    double* acc;  // optional: acc = acc_coef * t0
    double acc_coef;
};
// split into stats (T0, cmax0, dots) and planes (exponent from the — possibly all-reduced — cmax0)
cudaError_t launch_prepare_split_stats(const PrepArgs<float>& a, cudaStream_t stream);
cudaError_t launch_prepare_split_planes(const PrepArgs<float>& a, cudaStream_t stream);
cudaError_t launch_prepare_f64(const PrepArgs<double>& a, cudaStream_t stream);

// out[p][q][j] = sum_r stats[p][q][r][j] (fixed order)
// out[j] = max over ranks q of the uint32 tail at planes + q·slice_elems + tail_off (j < s): the
// column maxima every rank appended to its operand chunk, merged after the all-gather
cudaError_t launch_merge_tails(const __half* planes, int64_t slice_elems, int64_t tail_off, int world, int s,
                               unsigned* out, cudaStream_t stream);
// (row blocks [r0, r0 + count) only, count < 0: to the end -- one group of a grouped stack)
cudaError_t launch_reduce_stats(const double* stats, int passes, int row_blocks, int s, double* out,
                                cudaStream_t stream, int r0 = 0, int count = -1);

// state (fp32/fp64, [s][ld]) -> fp64 [s][ldo]
cudaError_t launch_state_to_f64(const void* state, bool is_f32, int64_t rows, int s, int64_t ld, double* out,
                                int64_t ldo, cudaStream_t stream);

// ---- small dense panel algebra (fp64) ------------------------------------
// C[p x q] = X^T Z over rows; partial buffer must hold grid*p*q doubles.
// ticket: a zeroed device counter (reset by the kernel): the last CTA reduces the partials in CTA order
// instead of a separate reduction launch; nullptr: separate reduction kernel
cudaError_t launch_panel_gram(const double* x, int p, int64_t ldx, const double* z, int q, int64_t ldz,
                              int64_t rows, double* partial, int grid, double* out, cudaStream_t stream,
                              unsigned* ticket = nullptr);
// W = beta*G + X*C   (X: rows x p, C: p x q column-major, W/G: rows x q)
cudaError_t launch_panel_update(double beta, const double* g, int64_t ldg, const double* x, int p, int64_t ldx,
                                const double* c, int q, int64_t rows, double* w, int64_t ldw, cudaStream_t stream);

// ---- probes ----------------------------------------------------------------
// Column j of the panel draws from RandomStream(derive_key(base_key, j0 + j)),
// or from RandomStream(base_key) itself when derive == false (single column).
// kind 0 = Gaussian (Box-Muller, reference stream order), 1 = Rademacher.
// Rows [row0, row0 + rows) of the panel (row0 even: Gaussian draws come in Box-Muller pairs).
cudaError_t launch_rng_panel(uint64_t base_key, bool derive, int kind, int64_t row0, int64_t rows, int cols, int j0,
                             double* out, int64_t ld, int* err_flag, cudaStream_t stream);

// ---- kernel-matrix construction --------------------------------------------
// Gaussian Gram + trace normalisation (reference build_kernel for sigma):
// A_ij = fl(1/n) * exp(-max(0, |x_i|^2+|x_j|^2-2 x_i.x_j) / (2 sigma^2)), A_ii = 1/n.
// Optional second sample set (Y) gives the normalised Hadamard joint
// n * A^X_ij * A^Y_ij with diag 1/n.
struct GramArgs {
    const double* x;  // samples n x dx (fp64; fp32 configs pass fp32-rounded values), element (i,k) at x[i*x_rs + k*x_cs]
    int dx;
    int64_t x_rs, x_cs;
    double inv_two_sigma2_x;
    const double* y;  // optional second variable (nullptr)
    int dy;
    int64_t y_rs, y_cs;
    double inv_two_sigma2_y;
    int64_t n;        // samples (= columns of A)
    int64_t row0;     // first row of this shard
    int64_t rows;     // rows in this shard
    int64_t ld;       // pitch of the output
    double inv_n;
    int f32_compute;  // 1: distances/exponentials in fp32 (fp32 configs); 0: fp64
};
// scratch (device bytes) the split Gram needs for staged operands; the caller provides it from its
// caching pool (no allocation on the launch path: stream-ordered allocations stalled up to 150 ms)
size_t gram_split_scratch_bytes(const GramArgs& g);
cudaError_t launch_gram_split(const GramArgs& g, __half* hi, __half* lo, void* scratch, cudaStream_t stream);
// tensor-core (3xTF32) Gram for single-rank fp32 builds with at most 128 features (gram_tc.cu)
bool gram_tc_supported(const GramArgs& g);
size_t gram_tc_scratch_bytes(const GramArgs& g);
cudaError_t launch_gram_tc(const GramArgs& g, __half* hi, __half* lo, void* scratch, cudaStream_t stream);
cudaError_t launch_gram_f64(const GramArgs& g, double* a, cudaStream_t stream);
// polynomial kernel build (x, n, dx, strides, rows/row0/ld, inv_n of g): isd [n] scratch; hi/lo (fp32
// configuration) or a64 (fp64); flags[0] |= 1 on a non-finite entry, flags[1] = min i with K_ii <= 0
// hadamard_joint of L >= 3 stored factors in a given order (kernel.cpp:74-101): fp64 factors by a64, split
// factors by hi/lo with their unscale; the output fp64 (c64) or split (chi/clo, stored = value / out_unscale)
constexpr int kMaxJoint = 16;
struct HadamardFactors {
    const double* a64[kMaxJoint];
    const __half* hi[kMaxJoint];
    const __half* lo[kMaxJoint];
    double unscale[kMaxJoint];
    int count;
};
cudaError_t launch_hadamard_n(const HadamardFactors& h, int64_t rows, int64_t cols, int64_t ld, int64_t row0,
                              double scale, double inv_n, double out_unscale, double* c64, __half* chi, __half* clo,
                              cudaStream_t stream);
// one content hash per stored row (the canonical factor order of hadamard_joint)
cudaError_t launch_row_hash(const double* a64, const __half* hi, const __half* lo, int64_t rows, int64_t cols,
                            int64_t ld, uint64_t* out, cudaStream_t stream);
// c = scale * (a ∘ b) elementwise over count entries (ops::hadamard_scaled, ops.cpp:116-122)
cudaError_t launch_scaled_product(const double* a, const double* b, int64_t count, double scale, double* c,
                                  cudaStream_t stream);
cudaError_t launch_poly_gram(const GramArgs& g, int degree, double offset, double* isd, __half* hi, __half* lo,
                             double* a64, unsigned* flags, cudaStream_t stream);

// A (fp64 row-major) -> planes holding A*scale.
cudaError_t launch_matrix_to_split(const double* a, int64_t rows, int64_t cols, int64_t lda, double scale,
                                   __half* hi, __half* lo, int64_t ld, cudaStream_t stream);
// Elementwise normalised Hadamard on split planes: stored C = factor*sA*sB, diagonal = diag_value.
cudaError_t launch_hadamard_split(const __half* ahi, const __half* alo, const __half* bhi, const __half* blo,
                                  int64_t rows, int64_t cols, int64_t ld, int64_t row0, double factor,
                                  double diag_value, __half* chi, __half* clo, cudaStream_t stream);
cudaError_t launch_hadamard_f64(const double* a, const double* b, int64_t rows, int64_t cols, int64_t ld,
                                int64_t row0, double n, double* c, cudaStream_t stream);
// out (column-major [d][n]) = scale * x
cudaError_t launch_scale_columns(const double* x, int64_t n, int d, int64_t rs, int64_t cs, double scale, double* out,
                                 cudaStream_t stream);
// samples check: flag[0] |= non-finite, flag[1] = float bits of max |x| (atomic max)
cudaError_t launch_check_samples(const double* x, int64_t n, int d, int64_t rs, int64_t cs, unsigned* flags,
                                 cudaStream_t stream);
// split planes -> fp64 (A = (hi+lo) * unscale)
cudaError_t launch_split_to_f64(const __half* hi, const __half* lo, int64_t rows, int64_t cols, int64_t ld,
                                double unscale, double* out, int64_t ldo, cudaStream_t stream);

}  // namespace rb
