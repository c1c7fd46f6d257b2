// y = A·x for one column (s = 1: the power iteration of spectrum.cpp:25-49 on fp32 kernels) reading
// only the upper triangle of the symmetric A: each 128 x 128 tile (I, J), I <= J, is streamed once and
// gives both its row sums A_IJ·x_J (rows of block I) and, off the diagonal, its column sums
// A_IJᵀ·x_I (rows of block J) -- 2 B of HBM per entry instead of 4 B. The reference's matvec
// (proj/src/ops.cpp:73-85) reads every entry; A is symmetric by construction (ops.cpp:9-20, mirrored
// Gram), so the result is the same product in a different summation order.
//
// Each CTA takes tiles of the upper triangle in row-major order (persistent, one CTA per SM, tiles
// streamed by TMA through a 3-stage ring); a half-warp owns a tile row (16 lanes x 8 columns, one
// 16-byte shared-memory read per plane), rows in fp32 FMA chains of 8 reduced
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

// Streaming structure: one producer thread keeps kStages tiles in flight by TMA (A_hi and A_lo 128 x 128
// boxes, zero-filled past n, plus the tile's 128-entry slices of the operand planes by 1-D bulk copies);
// eight consumer warps compute from shared memory and release each stage when their reads are done.
constexpr int kStages = 3;
constexpr int kPlaneBytes = ST * ST * 2;                // one fp16 plane of a tile
constexpr int kXBytes = ST * 2;                         // one fp16 operand slice
constexpr int kStageBytes = 2 * kPlaneBytes + 4 * kXBytes;  // A_hi, A_lo, x_i hi/lo, x_j hi/lo
constexpr int kSymvSmem = kStages * kStageBytes + 1024;
constexpr int kConsumers = 8;
constexpr int kSymvThreadsTma = 32 * (kConsumers + 1);

__global__ void __launch_bounds__(kSymvThreadsTma, 1)
    symv_split_kernel(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
                      const __half* __restrict__ xhi, const __half* __restrict__ xlo, int64_t nb,
                      float* __restrict__ partial) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    __shared__ float cs[16][ST + 1];  // column partials of the 16 row groups
    const int tid = threadIdx.x;
    const int warp = tid / 32, lane = tid % 32;
    const int64_t tiles = nb * (nb + 1) / 2;
    if (tid == 0) {
        prefetch_tmap(&map_hi);
        prefetch_tmap(&map_lo);
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kConsumers);
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (warp == kConsumers) {  // producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int st = 0;
            uint32_t ph = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                int64_t bi, bj;
                upper_tile(t, nb, &bi, &bj);
                mbar_wait(&empty[st], ph ^ 1u);
                uint8_t* dst = smem + st * kStageBytes;
                mbar_arrive_expect_tx(&full[st], kStageBytes);
                tma_load_2d(dst, &map_hi, &full[st], static_cast<int>(bj * ST), static_cast<int>(bi * ST), pol);
                tma_load_2d(dst + kPlaneBytes, &map_lo, &full[st], static_cast<int>(bj * ST), static_cast<int>(bi * ST),
                            pol);
                uint8_t* xd = dst + 2 * kPlaneBytes;
                bulk_load_1d(xd, xhi + bi * ST, kXBytes, &full[st], pol);
                bulk_load_1d(xd + kXBytes, xlo + bi * ST, kXBytes, &full[st], pol);
                bulk_load_1d(xd + 2 * kXBytes, xhi + bj * ST, kXBytes, &full[st], pol);
                bulk_load_1d(xd + 3 * kXBytes, xlo + bj * ST, kXBytes, &full[st], pol);
                if (++st == kStages) st = 0, ph ^= 1u;
            }
        }
        return;
    }
    // consumers: a half-warp owns a tile row (16 lanes x 8 columns), rows rg, rg + 16, ...
    const int half = lane / 16, c = lane % 16;
    const int rg = warp * 2 + half;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        int64_t bi, bj;
        upper_tile(t, nb, &bi, &bj);
        const bool diag = bi == bj;
        mbar_wait(&full[st], ph);
        const uint8_t* tile = smem + st * kStageBytes;
        const __half* xs = reinterpret_cast<const __half*>(tile + 2 * kPlaneBytes);  // [x_i hi | lo | x_j hi | lo]
        float xj[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
            xj[e] = __half2float(xs[2 * ST + c * 8 + e]) + __half2float(xs[3 * ST + c * 8 + e]);
        float cacc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) cacc[e] = 0.f;
        uint4 rh[8], rl[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int row = rg + 16 * q;
            rh[q] = *reinterpret_cast<const uint4*>(tile + row * (ST * 2) + c * 16);
            rl[q] = *reinterpret_cast<const uint4*>(tile + kPlaneBytes + row * (ST * 2) + c * 16);
        }
        float xi[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int row = rg + 16 * q;
            xi[q] = __half2float(xs[row]) + __half2float(xs[ST + row]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);  // this warp's reads of the stage are in registers
        if (++st == kStages) st = 0, ph ^= 1u;
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
#pragma unroll
                for (int e = 0; e < 8; ++e) cacc[e] = fmaf(a[e], xi[q], cacc[e]);
            }
        }
        if (!diag) {
            asm volatile("bar.sync 1, 256;" ::: "memory");  // the previous tile's column sums are read
#pragma unroll
            for (int e = 0; e < 8; ++e) cs[rg][c * 8 + e] = cacc[e];
            asm volatile("bar.sync 1, 256;" ::: "memory");
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
    if (a.rows != a.cols || !xlo) return cudaErrorInvalidValue;
    const int64_t nb = symv_blocks(a.cols);
    const int64_t tiles = nb * (nb + 1) / 2;
    TensorMapEncodeFn enc = tensor_map_encoder();
    if (!enc) return cudaErrorInvalidValue;
    CUtensorMap mh, ml;
    for (int p = 0; p < 2; ++p) {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.cols), static_cast<cuuint64_t>(a.rows)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld) * 2};
        cuuint32_t box[2] = {ST, ST};
        cuuint32_t estr[2] = {1, 1};
        if (enc(p ? &ml : &mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half*>(p ? a.lo : a.hi), dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(symv_split_kernel), kSymvSmem); e != cudaSuccess)
        return e;
    const int64_t g = std::min<int64_t>(std::max(grid, 1), tiles);
    symv_split_kernel<<<static_cast<unsigned>(g), kSymvThreadsTma, kSymvSmem, stream>>>(mh, ml, xhi, xlo, nb, partial);
    return cudaGetLastError();
}

}  // namespace rb
