// y = A·x for one column (s = 1: the power iteration of spectrum.cpp:25-49 on fp32 kernels) reading
// only the upper triangle of the symmetric A: each 128 x 128 tile (I, J), I <= J, is streamed once and
// gives both its row sums A_IJ·x_J (rows of block I) and, off the diagonal, its column sums
// A_IJᵀ·x_I (rows of block J) -- 2 B of HBM per entry instead of 4 B. The reference's matvec
// (proj/src/ops.cpp:73-85) reads every entry; A is symmetric by construction (ops.cpp:9-20, mirrored
// Gram), so the result is the same product in a different summation order.
//
// Each CTA takes tiles of the upper triangle in row-major order (persistent stride); a half-warp owns
// a tile row (16 lanes x 8 columns, two 16-byte loads per plane), rows in fp32 FMA chains of 8 reduced
// by shuffles in a fixed tree, columns accumulated per thread over its 8 rows and summed across the 16
// row groups in a fixed order through shared memory. Every row block I receives exactly nb partials
// (row sums of tiles (I, J >= I), column sums of tiles (I' < I, I)) in slot I·nb + (other tile index):
// the pass epilogue sums them in slot order (fp64), so the result is run-to-run bitwise identical.
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rb {

namespace {

constexpr int ST = 128;  // tile rows / columns
constexpr int kSymvThreads = 256;

__device__ __forceinline__ void upper_tile(int64_t t, int64_t nb, int64_t* bi, int64_t* bj) {
    // tile t of the row-major upper triangle: row I holds nb - I tiles
    auto start = [nb](int64_t b) { return b * nb - b * (b - 1) / 2; };
    const double q = 2.0 * nb + 1.0;
    int64_t i = static_cast<int64_t>((q - sqrt(q * q - 8.0 * static_cast<double>(t))) * 0.5);
    i = i < 0 ? 0 : (i > nb - 1 ? nb - 1 : i);
    while (i + 1 < nb && start(i + 1) <= t) ++i;
    while (i > 0 && start(i) > t) --i;
    *bi = i;
    *bj = i + (t - start(i));
}

__device__ __forceinline__ void unpack8(uint4 h, uint4 l, float* out) {
    const __half2* hh = reinterpret_cast<const __half2*>(&h);
    const __half2* ll = reinterpret_cast<const __half2*>(&l);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float2 a = __half22float2(hh[q]), b = __half22float2(ll[q]);
        out[2 * q] = a.x + b.x;  // hi + lo: exact in fp32 (22 significant bits)
        out[2 * q + 1] = a.y + b.y;
    }
}

__global__ void __launch_bounds__(kSymvThreads) symv_split_kernel(const __half* __restrict__ ahi,
                                                                  const __half* __restrict__ alo, int64_t n,
                                                                  int64_t lda, const __half* __restrict__ xhi,
                                                                  const __half* __restrict__ xlo, int64_t nb,
                                                                  float* __restrict__ partial) {
    __shared__ float xs_i[ST], xs_j[ST];
    __shared__ float cs[16][ST + 1];  // column partials of the 16 row groups
    const int tid = threadIdx.x;
    const int lane = tid % 32, warp = tid / 32;
    const int half = lane / 16, c = lane % 16;  // tile row parity inside the warp, 8-column chunk
    const int rg = warp * 2 + half;             // row group 0..15: rows rg, rg + 16, ...
    const int64_t tiles = nb * (nb + 1) / 2;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        int64_t bi, bj;
        upper_tile(t, nb, &bi, &bj);
        const int64_t i0 = bi * ST, j0 = bj * ST;
        const bool diag = bi == bj;
        __syncthreads();  // the previous tile's shared arrays are consumed
        if (tid < ST) {
            const int64_t gi = i0 + tid, gj = j0 + tid;
            xs_i[tid] = gi < n ? __half2float(xhi[gi]) + (xlo ? __half2float(xlo[gi]) : 0.f) : 0.f;
            xs_j[tid] = gj < n ? __half2float(xhi[gj]) + (xlo ? __half2float(xlo[gj]) : 0.f) : 0.f;
        }
        __syncthreads();
        float xj[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) xj[e] = xs_j[c * 8 + e];
        float cacc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) cacc[e] = 0.f;
        const int64_t gc = j0 + c * 8;  // first column of this thread's chunk
        const bool cols_full = gc + 8 <= n;
        // the 8 rows of this row group: loads first (16 independent 16-byte loads in flight)
        uint4 rh[8], rl[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int64_t gi = i0 + rg + 16 * q;
            if (gi < n && cols_full) {
                rh[q] = *reinterpret_cast<const uint4*>(ahi + gi * lda + gc);
                rl[q] = *reinterpret_cast<const uint4*>(alo + gi * lda + gc);
            } else {
                __half hv[8], lv[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const bool ok = gi < n && gc + e < n;
                    hv[e] = ok ? ahi[gi * lda + gc + e] : __float2half(0.f);
                    lv[e] = ok ? alo[gi * lda + gc + e] : __float2half(0.f);
                }
                rh[q] = *reinterpret_cast<const uint4*>(hv);
                rl[q] = *reinterpret_cast<const uint4*>(lv);
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int row = rg + 16 * q;
            float a[8];
            unpack8(rh[q], rl[q], a);
            float r = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) r = fmaf(a[e], xj[e], r);
            // the row's 16 chunks: fixed xor tree inside the half-warp
#pragma unroll
            for (int o = 8; o >= 1; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
            if (c == 0) partial[(bi * nb + bj) * ST + row] = r;  // row sums of tile (I, J): slot I·nb + J
            if (!diag) {
                const float xi = xs_i[row];
#pragma unroll
                for (int e = 0; e < 8; ++e) cacc[e] = fmaf(a[e], xi, cacc[e]);
            }
        }
        if (!diag) {
#pragma unroll
            for (int e = 0; e < 8; ++e) cs[rg][c * 8 + e] = cacc[e];
            __syncthreads();
            if (tid < ST) {
                float v = 0.f;
#pragma unroll
                for (int g = 0; g < 16; ++g) v += cs[g][tid];
                partial[(bj * nb + bi) * ST + tid] = v;  // column sums of tile (I, J): slot J·nb + I
            }
        }
    }
}

}  // namespace

int64_t symv_blocks(int64_t n) { return (n + ST - 1) / ST; }

cudaError_t launch_symv_split(const SplitMatrixView& a, const __half* xhi, const __half* xlo, float* partial,
                              int grid, cudaStream_t stream) {
    if (a.rows != a.cols) return cudaErrorInvalidValue;
    if (a.ld % 8 != 0) return cudaErrorInvalidValue;  // 16-byte row chunks
    const int64_t nb = symv_blocks(a.cols);
    const int64_t tiles = nb * (nb + 1) / 2;
    const int64_t g = std::min<int64_t>(std::max(grid, 1), tiles);
    symv_split_kernel<<<static_cast<unsigned>(g), kSymvThreads, 0, stream>>>(a.hi, a.lo, a.cols, a.ld, xhi, xlo, nb,
                                                                             partial);
    return cudaGetLastError();
}

}  // namespace rb
