// fp64 block product Y = A·V for the fp64 configuration (config 1, n=2000:
// A is 32 MB and L2-resident, so this is a latency/correctness path, not a
// roofline path). Same partial layout as the tensor-core kernel with one slot
// per 128-row block, so the shared pass epilogue consumes both.
// Reference: ops::matmul_panel / panel_block, proj/src/ops.cpp:30-35,98-107.
#include <algorithm>

#include "kernels.h"

namespace rb {

namespace {

constexpr int FM = 128;  // rows per CTA (matches the epilogue's row block)
constexpr int FN = 32;   // columns per CTA
constexpr int FK = 32;   // K per smem tile

// Stream-K over (row block, 32-column k tile) iterations: CTA c owns iterations
// [T·c/G, T·(c+1)/G) and writes one partial per row block it touches to slot rb + c (the pass
// epilogue sums a row block's slots in CTA order, so results are run-to-run identical). At
// n = 2000 this spreads the 32 MB of A over every SM instead of 16 row-block CTAs.
__global__ void __launch_bounds__(256, 2) block_av_f64_kernel(const double* __restrict__ a, int64_t rows, int64_t cols,
                                                           int64_t lda, const double* __restrict__ v, int s,
                                                           int64_t ldv, int npad, double* __restrict__ partial,
                                                           int64_t total_iters, int k_tiles) {
    __shared__ double as[FK][FM + 1];
    __shared__ double vs[FK][FN + 1];
    const int tx = threadIdx.x % 8;  // columns tx + 8j
    const int ty = threadIdx.x / 8;  // rows ty + 32i
    const int G = gridDim.x, c = blockIdx.x;
    const int col0 = blockIdx.y * FN;
    int64_t it = total_iters * c / G;
    const int64_t it_end = total_iters * (c + 1) / G;
    while (it < it_end) {
        const int64_t rb = it / k_tiles;
        const int64_t seg_end = min(it_end, (rb + 1) * k_tiles);
        const int64_t row0 = rb * FM;
        // 4x4 register tile per thread: rows ty + 32i, columns tx + 8j (8 shared loads per 16 DFMA; each
        // output's k sum runs in the same order as before, so results are bitwise unchanged)
        double acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
        // software pipeline: the next k tile's loads are in flight in registers while this one computes
        // (A is L2-resident: each tile is an L2 round trip, which the compute of the previous tile hides)
        constexpr int NA = FM * FK / 256, NV = FN * FK / 256;
        double ra[NA], rv[NV];
        auto load = [&](int64_t t) {
            const int64_t k0 = (t - rb * k_tiles) * FK;
#pragma unroll
            for (int q = 0; q < NA; ++q) {
                const int idx = threadIdx.x + 256 * q;
                const int rr = idx / FK, kk = idx % FK;
                const int64_t gr = row0 + rr, gk = k0 + kk;
                ra[q] = (gr < rows && gk < cols) ? a[gr * lda + gk] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const int idx = threadIdx.x + 256 * q;
                const int cc = idx / FK, kk = idx % FK;
                const int gc = col0 + cc;
                const int64_t gk = k0 + kk;
                rv[q] = (gc < s && gk < cols) ? v[static_cast<int64_t>(gc) * ldv + gk] : 0.0;
            }
        };
        load(it);
        for (; it < seg_end; ++it) {
#pragma unroll
            for (int q = 0; q < NA; ++q) {
                const int idx = threadIdx.x + 256 * q;
                as[idx % FK][idx / FK] = ra[q];
            }
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const int idx = threadIdx.x + 256 * q;
                vs[idx % FK][idx / FK] = rv[q];
            }
            __syncthreads();
            if (it + 1 < seg_end) load(it + 1);
#pragma unroll 4
            for (int kk = 0; kk < FK; ++kk) {
                double ar[4], vr[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) ar[i] = as[kk][ty + 32 * i];
#pragma unroll
                for (int j = 0; j < 4; ++j) vr[j] = vs[kk][tx + 8 * j];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fma(ar[i], vr[j], acc[i][j]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = col0 + tx + 8 * j;
            if (col < s) {
                double* dst = partial + ((rb + c) * npad + col) * FM;
#pragma unroll
                for (int i = 0; i < 4; ++i) dst[ty + 32 * i] = acc[i][j];
            }
        }
    }
}

}  // namespace

int f64_npad(int cols) { return ((cols + FN - 1) / FN) * FN; }

StreamKPlan make_f64_plan(int64_t rows, int64_t cols, int grid) {
    StreamKPlan p;
    p.row_blocks = static_cast<int>((rows + FM - 1) / FM);
    p.k_tiles = static_cast<int>((cols + FK - 1) / FK);
    p.total_iters = static_cast<int64_t>(p.row_blocks) * p.k_tiles;
    p.grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(grid, p.total_iters)));
    p.kc = 1;
    p.cluster = 1;
    p.dp_blocks = 0;
    p.slots = p.row_blocks + p.grid;
    p.rows_per_block = FM;
    return p;
}

cudaError_t launch_block_av_f64(const double* a, int64_t rows, int64_t cols, int64_t lda, const double* v, int s,
                                int64_t ldv, const StreamKPlan& plan, double* partial, cudaStream_t stream) {
    const int npad = f64_npad(s);
    dim3 grid(static_cast<unsigned>(plan.grid), static_cast<unsigned>(npad / FN));
    block_av_f64_kernel<<<grid, 256, 0, stream>>>(a, rows, cols, lda, v, s, ldv, npad, partial, plan.total_iters,
                                                  plan.k_tiles);
    return cudaGetLastError();
}

}  // namespace rb
