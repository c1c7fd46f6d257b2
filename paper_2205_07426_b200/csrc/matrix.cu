// Kernel-matrix construction on the device.
//
// K1+K2 (+K4): Gaussian Gram, trace normalisation and the normalised
// Hadamard joint, fused into one pass that writes A straight into its HBM
// storage format. Reference: ops::gaussian_gram / gaussian_row
// (proj/src/ops.cpp:9-20,39-47), build_kernel (proj/src/kernel.cpp:35-72),
// hadamard_joint / hadamard_scaled (proj/src/kernel.cpp:74-101,
// proj/src/ops.cpp:116-122).
//
// Arithmetic per entry follows the reference: d2 = (|x_i|^2 + |x_j|^2) − 2·x_i·x_j,
// clamp at 0, K = exp(−d2 · 1/(2σ²)), K_ii = 1 exactly; A = fl(1/n)·K. The
// fp32 configurations compute d2 and exp in fp32 (inputs are fp32 samples) and
// store K·2^14 (= A·n·2^14) as an fp16 hi/lo pair; the fp64 configuration
// stores fl(1/n)·K in fp64. Both are exactly symmetric (the formula is).
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace rb {

namespace {

constexpr int TM = 64;  // output tile rows
constexpr int TN = 64;  // output tile cols
constexpr int TKd = 32; // feature chunk

template <typename T>
struct GramTile {
    // accumulates dot products and squared norms of one 64x64 tile over a feature block
    __device__ static void accumulate(const double* __restrict__ x, int d, int64_t rs, int64_t cs, int64_t n,
                                      int64_t row0, int64_t col0, T (&dot)[4][4], T (&sqr)[4], T (&sqc)[4],
                                      T (*xr)[TM + 1], T (*xc)[TN + 4]) {
        const int tid = threadIdx.x;
        const int tx = tid % 16, ty = tid / 16;
        for (int k0 = 0; k0 < d; k0 += TKd) {
            const int kc = min(TKd, d - k0);
            for (int idx = tid; idx < TM * TKd; idx += blockDim.x) {
                const int rr = idx % TM, kk = idx / TM;  // consecutive threads: consecutive samples
                const int64_t gr = row0 + rr;
                xr[kk][rr] = (kk < kc && gr < n) ? static_cast<T>(x[gr * rs + (k0 + kk) * cs]) : T(0);
                const int64_t gc = col0 + rr;
                xc[kk][rr] = (kk < kc && gc < n) ? static_cast<T>(x[gc * rs + (k0 + kk) * cs]) : T(0);
            }
            __syncthreads();
            for (int kk = 0; kk < kc; ++kk) {
                T a[4], b[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) a[u] = xr[kk][ty + 16 * u];
#pragma unroll
                for (int v = 0; v < 4; ++v) b[v] = xc[kk][4 * tx + v];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    sqr[u] = fma(a[u], a[u], sqr[u]);
#pragma unroll
                    for (int v = 0; v < 4; ++v) dot[u][v] = fma(a[u], b[v], dot[u][v]);
                }
#pragma unroll
                for (int v = 0; v < 4; ++v) sqc[v] = fma(b[v], b[v], sqc[v]);
            }
            __syncthreads();
        }
    }
};

__device__ __forceinline__ float kexp(float x) { return expf(x); }
__device__ __forceinline__ double kexp(double x) { return exp(x); }

template <typename T, bool SPLIT>
__global__ void __launch_bounds__(256) gram_kernel(GramArgs g, __half* __restrict__ hi, __half* __restrict__ lo,
                                                   double* __restrict__ a64) {
    __shared__ T xr[TKd][TM + 1];
    __shared__ T xc[TKd][TN + 4];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t row0 = g.row0 + static_cast<int64_t>(blockIdx.y) * TM;  // global sample index of tile rows
    const int64_t col0 = static_cast<int64_t>(blockIdx.x) * TN;

    T dot[4][4], sqr[4], sqc[4];
    T kval[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        sqr[u] = sqc[u] = T(0);
#pragma unroll
        for (int v = 0; v < 4; ++v) dot[u][v] = T(0);
    }
    GramTile<T>::accumulate(g.x, g.dx, g.x_rs, g.x_cs, g.n, row0, col0, dot, sqr, sqc, xr, xc);
    const T ax = static_cast<T>(g.inv_two_sigma2_x);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            T d2 = (sqr[u] + sqc[v]) - T(2) * dot[u][v];
            if (d2 < T(0)) d2 = T(0);
            kval[u][v] = kexp(-d2 * ax);
        }
    if (g.y) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            sqr[u] = sqc[u] = T(0);
#pragma unroll
            for (int v = 0; v < 4; ++v) dot[u][v] = T(0);
        }
        GramTile<T>::accumulate(g.y, g.dy, g.y_rs, g.y_cs, g.n, row0, col0, dot, sqr, sqc, xr, xc);
        const T ay = static_cast<T>(g.inv_two_sigma2_y);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                T d2 = (sqr[u] + sqc[v]) - T(2) * dot[u][v];
                if (d2 < T(0)) d2 = T(0);
                const T ky = kexp(-d2 * ay);
                if (SPLIT) {
                    kval[u][v] = kval[u][v] * ky;
                } else {
                    // reference op order: n * ((inv_n*Kx) * (inv_n*Ky)); finished below
                    kval[u][v] = kval[u][v];
                    dot[u][v] = ky;  // stash Ky
                }
            }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t gi = row0 + ty + 16 * u;  // sample index
        if (gi >= g.row0 + g.rows || gi >= g.n) continue;
        const int64_t li = gi - g.row0;         // local row
        const int64_t gj0 = col0 + 4 * tx;
        if (SPLIT) {
            __half h[4], l[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                float kv = static_cast<float>(kval[u][v]);
                if (gi == gj0 + v) kv = 1.0f;
                const float s = kv * static_cast<float>(kSplitScale);
                h[v] = __float2half_rn(s);
                l[v] = __float2half_rn(s - __half2float(h[v]));
            }
            __half* ph = hi + li * g.ld + gj0;
            __half* pl = lo + li * g.ld + gj0;
            if (gj0 + 3 < g.n) {
                *reinterpret_cast<uint2*>(ph) = make_uint2(
                    (static_cast<uint32_t>(__half_as_ushort(h[1])) << 16) | __half_as_ushort(h[0]),
                    (static_cast<uint32_t>(__half_as_ushort(h[3])) << 16) | __half_as_ushort(h[2]));
                *reinterpret_cast<uint2*>(pl) = make_uint2(
                    (static_cast<uint32_t>(__half_as_ushort(l[1])) << 16) | __half_as_ushort(l[0]),
                    (static_cast<uint32_t>(__half_as_ushort(l[3])) << 16) | __half_as_ushort(l[2]));
            } else {
                for (int v = 0; v < 4; ++v)
                    if (gj0 + v < g.n) {
                        ph[v] = h[v];
                        pl[v] = l[v];
                    }
            }
        } else {
            double* pa = a64 + li * g.ld + gj0;
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const int64_t gj = gj0 + v;
                if (gj >= g.n) continue;
                double val;
                if (gi == gj) {
                    val = g.inv_n;
                } else if (g.y) {
                    const double ax_ = g.inv_n * static_cast<double>(kval[u][v]);
                    const double ay_ = g.inv_n * static_cast<double>(dot[u][v]);
                    val = static_cast<double>(g.n) * (ax_ * ay_);
                } else {
                    val = g.inv_n * static_cast<double>(kval[u][v]);
                }
                pa[v] = val;
            }
        }
    }
}

// fp64 storage, whole matrix on one rank: only tiles with column tile >= row tile are evaluated
// (the per-entry arithmetic of gram_kernel<double, false>, which is symmetric bit for bit: the dot is a
// chain of fma(x_ik, x_jk, .) and the norm sum is commutative), and each off-diagonal tile is also
// written mirrored through shared memory with coalesced row stores. Halves the exp work of config 1.
constexpr int kSymF64Smem = (TKd * (TM + 1) + TKd * (TN + 4)) > TM * (TN + 1) ? (TKd * (TM + 1) + TKd * (TN + 4))
                                                                               : TM * (TN + 1);

__global__ void __launch_bounds__(256) gram_sym_f64_kernel(GramArgs g, double* __restrict__ a64, int tiles) {
    __shared__ double buf[kSymF64Smem];
    auto xr = reinterpret_cast<double(*)[TM + 1]>(buf);
    auto xc = reinterpret_cast<double(*)[TN + 4]>(buf + TKd * (TM + 1));
    auto stg = reinterpret_cast<double(*)[TN + 1]>(buf);  // reused after the accumulation
    // upper-triangle tile b -> (bi, bj), bi <= bj, row-major over the triangle
    int bi = 0, rem = blockIdx.x;
    while (rem >= tiles - bi) rem -= tiles - bi, ++bi;
    const int bj = bi + rem;
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t row0 = static_cast<int64_t>(bi) * TM, col0 = static_cast<int64_t>(bj) * TN;

    double dot[4][4], sqr[4], sqc[4], kval[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        sqr[u] = sqc[u] = 0.0;
#pragma unroll
        for (int v = 0; v < 4; ++v) dot[u][v] = 0.0;
    }
    GramTile<double>::accumulate(g.x, g.dx, g.x_rs, g.x_cs, g.n, row0, col0, dot, sqr, sqc, xr, xc);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            double d2 = (sqr[u] + sqc[v]) - 2.0 * dot[u][v];
            if (d2 < 0.0) d2 = 0.0;
            kval[u][v] = exp(-d2 * g.inv_two_sigma2_x);
        }
    if (g.y) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            sqr[u] = sqc[u] = 0.0;
#pragma unroll
            for (int v = 0; v < 4; ++v) dot[u][v] = 0.0;
        }
        GramTile<double>::accumulate(g.y, g.dy, g.y_rs, g.y_cs, g.n, row0, col0, dot, sqr, sqc, xr, xc);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                double d2 = (sqr[u] + sqc[v]) - 2.0 * dot[u][v];
                if (d2 < 0.0) d2 = 0.0;
                dot[u][v] = exp(-d2 * g.inv_two_sigma2_y);  // Ky
            }
    }
    // accumulate() ends with a barrier: the feature tiles are dead, buf is the mirror staging now
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int r = ty + 16 * u;
        const int64_t gi = row0 + r;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t gj = col0 + 4 * tx + v;  // (entries past n are staged but never stored)
            double val;
            if (gi == gj) {
                val = g.inv_n;
            } else if (g.y) {  // reference op order: n * ((inv_n*Kx) * (inv_n*Ky))
                val = static_cast<double>(g.n) * ((g.inv_n * kval[u][v]) * (g.inv_n * dot[u][v]));
            } else {
                val = g.inv_n * kval[u][v];
            }
            stg[r][4 * tx + v] = val;
        }
    }
    __syncthreads();
    // both the tile and its mirror leave shared memory as whole 512-byte row segments
    for (int idx = tid; idx < TM * TN; idx += blockDim.x) {
        const int r = idx / TN, c = idx % TN;  // tile row row0 + r, consecutive threads: consecutive columns
        const int64_t gi = row0 + r, gj = col0 + c;
        if (gi < g.n && gj < g.n) a64[gi * g.ld + gj] = stg[r][c];
    }
    if (bi == bj) return;
    for (int idx = tid; idx < TM * TN; idx += blockDim.x) {
        const int c = idx / TM, r = idx % TM;  // mirror row col0 + c, consecutive threads: consecutive columns
        const int64_t gi = col0 + c, gj = row0 + r;
        if (gi < g.n && gj < g.n) a64[gi * g.ld + gj] = stg[r][c];
    }
}

// fp32 configurations: symmetric tiles. Only tiles with column tile >= row tile are
// evaluated; the mirrored tile is written through shared memory (coalesced), so the
// distance/exp work halves while every entry of A is still written once.
// The joint uses one exp2 of the summed exponents (exp(a)·exp(b) = exp(a+b)).
__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void store_split4(__half* ph, __half* pl, const float* kv, int64_t gj0, int64_t n) {
    __half h[4], l[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        const float s = kv[v] * static_cast<float>(kSplitScale);
        h[v] = __float2half_rn(s);
        l[v] = __float2half_rn(s - __half2float(h[v]));
    }
    if (gj0 + 3 < n) {
        *reinterpret_cast<uint2*>(ph) =
            make_uint2((static_cast<uint32_t>(__half_as_ushort(h[1])) << 16) | __half_as_ushort(h[0]),
                       (static_cast<uint32_t>(__half_as_ushort(h[3])) << 16) | __half_as_ushort(h[2]));
        *reinterpret_cast<uint2*>(pl) =
            make_uint2((static_cast<uint32_t>(__half_as_ushort(l[1])) << 16) | __half_as_ushort(l[0]),
                       (static_cast<uint32_t>(__half_as_ushort(l[3])) << 16) | __half_as_ushort(l[2]));
    } else {
        for (int v = 0; v < 4; ++v)
            if (gj0 + v < n) {
                ph[v] = h[v];
                pl[v] = l[v];
            }
    }
}

// 128x128 output tile per CTA (256 threads, 8x8 entries each); samples pre-converted to fp32
// column-major [d][n] (xf, yf) so each tile reads 2·128·d·4 bytes from L2 (d/16 B per entry).
// 128x128 output tile per CTA (512 threads, 4x8 entries each); samples pre-converted to fp32
// column-major [d][n] (xf, yf) so each tile reads 2·128·d·4 bytes from L2 (d/16 B per entry).
constexpr int ST = 128;  // symmetric tile
constexpr int SK = 16;   // feature chunk

__device__ __forceinline__ void store_split8(__half* ph, __half* pl, const float* kv, int64_t gj0, int64_t n) {
    __align__(16) __half2 h[4];
    __align__(16) __half2 l[4];
    const float2 sc = make_float2(static_cast<float>(kSplitScale), static_cast<float>(kSplitScale));
#pragma unroll
    for (int v = 0; v < 4; ++v) {  // packed: cvt.rn.f16x2.f32 for hi, the residual in fp32 pairs, cvt again
        const float2 s2 = __fmul2_rn(make_float2(kv[2 * v], kv[2 * v + 1]), sc);
        h[v] = __float22half2_rn(s2);
        const float2 back = __half22float2(h[v]);
        l[v] = __float22half2_rn(__fadd2_rn(s2, make_float2(-back.x, -back.y)));
    }
    if (gj0 + 7 < n && ((reinterpret_cast<uintptr_t>(ph) | reinterpret_cast<uintptr_t>(pl)) & 15) == 0) {
        *reinterpret_cast<uint4*>(ph) = *reinterpret_cast<const uint4*>(h);
        *reinterpret_cast<uint4*>(pl) = *reinterpret_cast<const uint4*>(l);
    } else {
        const __half* hh = reinterpret_cast<const __half*>(h);
        const __half* ll = reinterpret_cast<const __half*>(l);
        for (int v = 0; v < 8; ++v)
            if (gj0 + v < n) {
                ph[v] = hh[v];
                pl[v] = ll[v];
            }
    }
}

constexpr int SU = 4;      // rows per thread (rows ty + 32u)
constexpr int SThreads = 512;

__device__ __forceinline__ void sym_accumulate(const float* __restrict__ xf, int d, int64_t n, int64_t row0,
                                               int64_t col0, float (&dot)[SU][8], float (&sqr)[SU], float (&sqc)[8],
                                               float (*xr)[ST], float (*xc)[ST]) {
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    for (int k0 = 0; k0 < d; k0 += SK) {
        const int kc = min(SK, d - k0);
        for (int idx = tid; idx < SK * ST; idx += blockDim.x) {
            const int kk = idx / ST, rr = idx % ST;  // consecutive threads: consecutive samples (coalesced)
            const int64_t gr = row0 + rr, gc = col0 + rr;
            xr[kk][rr] = (kk < kc && gr < n) ? xf[static_cast<int64_t>(k0 + kk) * n + gr] : 0.f;
            xc[kk][rr] = (kk < kc && gc < n) ? xf[static_cast<int64_t>(k0 + kk) * n + gc] : 0.f;
        }
        __syncthreads();
        for (int kk = 0; kk < kc; ++kk) {
            float a[SU], b[8];
#pragma unroll
            for (int u = 0; u < SU; ++u) a[u] = xr[kk][ty + 32 * u];
            const float4 b0 = *reinterpret_cast<const float4*>(&xc[kk][8 * tx]);
            const float4 b1 = *reinterpret_cast<const float4*>(&xc[kk][8 * tx + 4]);
            b[0] = b0.x, b[1] = b0.y, b[2] = b0.z, b[3] = b0.w, b[4] = b1.x, b[5] = b1.y, b[6] = b1.z, b[7] = b1.w;
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                sqr[u] = fmaf(a[u], a[u], sqr[u]);
                const float2 au = make_float2(a[u], a[u]);
#pragma unroll
                for (int v = 0; v < 8; v += 2) {  // packed FFMA2: two columns per instruction
                    const float2 r = __ffma2_rn(au, make_float2(b[v], b[v + 1]), make_float2(dot[u][v], dot[u][v + 1]));
                    dot[u][v] = r.x, dot[u][v + 1] = r.y;
                }
            }
#pragma unroll
            for (int v = 0; v < 8; ++v) sqc[v] = fmaf(b[v], b[v], sqc[v]);
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(SThreads) gram_sym_f32_kernel(GramArgs g, const float* __restrict__ xf,
                                                           const float* __restrict__ yf, int nb,
                                                           __half* __restrict__ hi, __half* __restrict__ lo) {
    extern __shared__ float gsm[];
    float(*xr)[ST] = reinterpret_cast<float(*)[ST]>(gsm);             // [SK][ST]
    float(*xc)[ST] = reinterpret_cast<float(*)[ST]>(gsm + SK * ST);    // [SK][ST]
    float(*tt)[ST + 1] = reinterpret_cast<float(*)[ST + 1]>(gsm + 2 * SK * ST);  // [ST][ST+1]
    // linear upper-triangle tile index -> (bi, bj), bi <= bj
    const int64_t t = blockIdx.x;
    auto start = [nb](int64_t b) { return b * nb - b * (b - 1) / 2; };
    const double q = 2.0 * nb + 1.0;
    int64_t bi = static_cast<int64_t>((q - sqrt(q * q - 8.0 * static_cast<double>(t))) * 0.5);
    if (bi < 0) bi = 0;
    if (bi > nb - 1) bi = nb - 1;
    while (bi + 1 < nb && start(bi + 1) <= t) ++bi;
    while (bi > 0 && start(bi) > t) --bi;
    const int64_t bj = bi + (t - start(bi));
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t row0 = bi * ST, col0 = bj * ST;
    const float l2e = 1.4426950408889634f;

    float e[SU][8];
    {
        float dot[SU][8], sqr[SU], sqc[8];
#pragma unroll
        for (int u = 0; u < SU; ++u) {
            sqr[u] = 0.f;
#pragma unroll
            for (int v = 0; v < 8; ++v) dot[u][v] = 0.f;
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) sqc[v] = 0.f;
        sym_accumulate(xf, g.dx, g.n, row0, col0, dot, sqr, sqc, xr, xc);
        const float ax = static_cast<float>(g.inv_two_sigma2_x) * l2e;
#pragma unroll
        for (int u = 0; u < SU; ++u)
#pragma unroll
            for (int v = 0; v < 8; ++v) e[u][v] = -fmaxf((sqr[u] + sqc[v]) - 2.f * dot[u][v], 0.f) * ax;
    }
    if (yf) {
        float dot[SU][8], sqr[SU], sqc[8];
#pragma unroll
        for (int u = 0; u < SU; ++u) {
            sqr[u] = 0.f;
#pragma unroll
            for (int v = 0; v < 8; ++v) dot[u][v] = 0.f;
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) sqc[v] = 0.f;
        sym_accumulate(yf, g.dy, g.n, row0, col0, dot, sqr, sqc, xr, xc);
        const float ay = static_cast<float>(g.inv_two_sigma2_y) * l2e;
#pragma unroll
        for (int u = 0; u < SU; ++u)
#pragma unroll
            for (int v = 0; v < 8; ++v) e[u][v] -= fmaxf((sqr[u] + sqc[v]) - 2.f * dot[u][v], 0.f) * ay;
    }
#pragma unroll
    for (int u = 0; u < SU; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) e[u][v] = fast_exp2(e[u][v]);  // e now holds K
    if (bi == bj) {  // K_ii = 1 exactly (ops.cpp:12) on the diagonal tiles only
#pragma unroll
        for (int u = 0; u < SU; ++u)
#pragma unroll
            for (int v = 0; v < 8; ++v)
                if (ty + 32 * u == 8 * tx + v) e[u][v] = 1.0f;
    }
    // direct tile: rows gi, columns gj
#pragma unroll
    for (int u = 0; u < SU; ++u) {
        const int64_t gi = row0 + ty + 32 * u;
        if (gi < g.n) store_split8(hi + gi * g.ld + col0 + 8 * tx, lo + gi * g.ld + col0 + 8 * tx, e[u], col0 + 8 * tx, g.n);
    }
    if (bi == bj) return;
    // mirrored tile: rows gj, columns gi (transposed through shared memory)
#pragma unroll
    for (int u = 0; u < SU; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) tt[8 * tx + v][ty + 32 * u] = e[u][v];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < SU; ++u) {
        const int rr = ty + 32 * u;
        const int64_t gr = col0 + rr;
        if (gr >= g.n) continue;
        float w[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) w[v] = tt[rr][8 * tx + v];
        store_split8(hi + gr * g.ld + row0 + 8 * tx, lo + gr * g.ld + row0 + 8 * tx, w, row0 + 8 * tx, g.n);
    }
}

__global__ void to_f32_colmajor_kernel(const double* __restrict__ x, int64_t n, int d, int64_t rs, int64_t cs,
                                       float* __restrict__ out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n * d) return;
    const int64_t i = t % n, k = t / n;
    out[t] = static_cast<float>(x[i * rs + k * cs]);
}

__global__ void matrix_to_split_kernel(const double* __restrict__ a, int64_t rows, int64_t cols, int64_t lda,
                                       double scale, __half* __restrict__ hi, __half* __restrict__ lo, int64_t ld) {
    const int64_t i = blockIdx.y;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = a[i * lda + j] * scale;
        const __half h = __double2half(v);
        hi[i * ld + j] = h;
        lo[i * ld + j] = __double2half(v - static_cast<double>(__half2float(h)));
    }
}

__global__ void split_to_f64_kernel(const __half* __restrict__ hi, const __half* __restrict__ lo, int64_t rows,
                                    int64_t cols, int64_t ld, double unscale, double* __restrict__ out,
                                    int64_t ldo) {
    const int64_t i = blockIdx.y;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i * ldo + j] = (static_cast<double>(__half2float(hi[i * ld + j])) +
                            static_cast<double>(__half2float(lo[i * ld + j]))) *
                           unscale;
}

__global__ void hadamard_split_kernel(const __half* __restrict__ ahi, const __half* __restrict__ alo,
                                      const __half* __restrict__ bhi, const __half* __restrict__ blo, int64_t rows,
                                      int64_t cols, int64_t ld, int64_t row0, double factor, double diag_value,
                                      __half* __restrict__ chi, __half* __restrict__ clo) {
    const int64_t i = blockIdx.y;
    // stored values S = X / unscale_X; stored C = n·uA·uB/uC · Sa·Sb = factor · Sa·Sb
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = i * ld + j;
        double v;
        if (row0 + i == j) {
            v = diag_value;
        } else {
            const double sa = static_cast<double>(__half2float(ahi[k])) + static_cast<double>(__half2float(alo[k]));
            const double sb = static_cast<double>(__half2float(bhi[k])) + static_cast<double>(__half2float(blo[k]));
            v = factor * (sa * sb);
        }
        const __half h = __double2half(v);
        chi[k] = h;
        clo[k] = __double2half(v - static_cast<double>(__half2float(h)));
    }
}

__global__ void hadamard_f64_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t rows,
                                    int64_t cols, int64_t ld, int64_t row0, double n, double* __restrict__ c) {
    const int64_t i = blockIdx.y;
    const double inv_n = 1.0 / n;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = i * ld + j;
        c[k] = (row0 + i == j) ? inv_n : n * (a[k] * b[k]);
    }
}

__global__ void check_samples_kernel(const double* __restrict__ x, int64_t n, int d, int64_t rs, int64_t cs,
                                     unsigned* flags) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t total = n * d;
    float mx = 0.f;
    bool bad = false;
    for (int64_t e = t; e < total; e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % n, k = e / n;
        const double v = x[i * rs + k * cs];
        if (!isfinite(v)) bad = true;
        else mx = fmaxf(mx, static_cast<float>(fabs(v)));
    }
    mx = warp_max(mx);
    const unsigned b = __any_sync(0xffffffffu, bad);
    if ((threadIdx.x & 31) == 0) {
        if (b) atomicOr(flags, 1u);
        atomicMax(flags + 1, __float_as_uint(mx));
    }
}

inline dim3 row_grid(int64_t rows, int64_t cols) {
    const int64_t bx = (cols + 255) / 256;
    return dim3(static_cast<unsigned>(bx > 64 ? 64 : bx), static_cast<unsigned>(rows));
}

}  // namespace

size_t gram_split_scratch_bytes(const GramArgs& g) {
    if (gram_tc_supported(g)) return gram_tc_scratch_bytes(g);
    if (g.f32_compute && g.row0 == 0 && g.rows == g.n && g.ld % 8 == 0)
        return static_cast<size_t>(g.n) * (g.dx + (g.y ? g.dy : 0)) * sizeof(float);
    return 0;
}

cudaError_t launch_gram_split(const GramArgs& g, __half* hi, __half* lo, void* scratch, cudaStream_t stream) {
    if (gram_tc_supported(g)) return launch_gram_tc(g, hi, lo, scratch, stream);
    if (g.f32_compute && g.row0 == 0 && g.rows == g.n && g.ld % 8 == 0) {
        // fp32 copies of the samples, column-major [d][n], for the symmetric tiles
        float* xf = static_cast<float*>(scratch);
        cudaError_t e = cudaSuccess;
        const int64_t nx = g.n * g.dx;
        to_f32_colmajor_kernel<<<static_cast<unsigned>((nx + 255) / 256), 256, 0, stream>>>(g.x, g.n, g.dx, g.x_rs,
                                                                                         g.x_cs, xf);
        float* yf = nullptr;
        if (g.y) {
            yf = xf + nx;
            const int64_t ny = g.n * g.dy;
            to_f32_colmajor_kernel<<<static_cast<unsigned>((ny + 255) / 256), 256, 0, stream>>>(
                g.y, g.n, g.dy, g.y_rs, g.y_cs, yf);
        }
        const int nb = static_cast<int>((g.n + ST - 1) / ST);
        const int64_t tiles = static_cast<int64_t>(nb) * (nb + 1) / 2;
        const size_t smem = (2 * SK * ST + ST * (ST + 1)) * sizeof(float);
        e = ensure_smem_attr(reinterpret_cast<const void*>(gram_sym_f32_kernel), static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        gram_sym_f32_kernel<<<static_cast<unsigned>(tiles), SThreads, smem, stream>>>(g, xf, yf, nb, hi, lo);
        e = cudaGetLastError();
        return e;
    }
    dim3 grid(static_cast<unsigned>((g.n + TN - 1) / TN), static_cast<unsigned>((g.rows + TM - 1) / TM));
    if (g.f32_compute)
        gram_kernel<float, true><<<grid, 256, 0, stream>>>(g, hi, lo, nullptr);
    else
        gram_kernel<double, true><<<grid, 256, 0, stream>>>(g, hi, lo, nullptr);
    return cudaGetLastError();
}

namespace {
// ---------------------------------------------------------------- polynomial kernel
// build_kernel(X, PolynomialKernel{degree, offset}) (proj/src/kernel.cpp:35-72, ops.cpp:22-28,58-64):
// K_ij = pow(x_i·x_j + offset, degree) in fp64 (dots summed over the features in order), normalised
// A_ij = ((fl(1/n)·K_ij)·isd_i)·isd_j with isd_i = 1/sqrt(K_ii), A_ii = 1/n. Stored as fp64 (fp64
// configuration) or as the fp16 hi/lo split of A·n·2^14 = K_ij·isd_i·isd_j·2^14 (|.| <= 2^14 by
// Cauchy-Schwarz: the kernel is PSD), the format every block product consumes.
// flags[0]: a non-finite K entry; flags[1]: the smallest i with K_ii <= 0 (n when none).
__global__ void poly_diag_kernel(const double* __restrict__ x, int64_t n, int d, int64_t rs, int64_t cs, double deg,
                                 double offset, double* __restrict__ isd, unsigned* __restrict__ flags) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double dot = 0.0;
    for (int k = 0; k < d; ++k) {
        const double v = x[i * rs + k * cs];
        dot = fma(v, v, dot);
    }
    const double kii = pow(dot + offset, deg);
    if (!isfinite(kii)) atomicOr(flags, 1u);
    if (!(kii > 0.0)) atomicMin(flags + 1, static_cast<unsigned>(i));
    isd[i] = 1.0 / sqrt(kii);
}

template <bool SPLIT>
__global__ void __launch_bounds__(256) poly_gram_kernel(GramArgs g, double deg, double offset,
                                                        const double* __restrict__ isd, __half* __restrict__ hi,
                                                        __half* __restrict__ lo, double* __restrict__ a64,
                                                        unsigned* __restrict__ flags) {
    __shared__ double xr[TKd][TM + 1];
    __shared__ double xc[TKd][TN + 4];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int64_t row0 = g.row0 + static_cast<int64_t>(blockIdx.y) * TM;
    const int64_t col0 = static_cast<int64_t>(blockIdx.x) * TN;
    double dot[4][4], sqr[4], sqc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        sqr[u] = sqc[u] = 0.0;
#pragma unroll
        for (int v = 0; v < 4; ++v) dot[u][v] = 0.0;
    }
    GramTile<double>::accumulate(g.x, g.dx, g.x_rs, g.x_cs, g.n, row0, col0, dot, sqr, sqc, xr, xc);
    bool bad = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t gi = row0 + ty + 16 * u;
        if (gi >= g.row0 + g.rows || gi >= g.n) continue;
        const int64_t li = gi - g.row0;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t gj = col0 + 4 * tx + v;
            if (gj >= g.n) continue;
            const double k = pow(dot[u][v] + offset, deg);
            bad |= !isfinite(k);
            if (!isd) {  // ops::polynomial_gram: the raw K (no normalisation)
                a64[li * g.ld + gj] = k;
                continue;
            }
            // the reference evaluates each pair once, i < j: ((inv_n·K)·isd_i)·isd_j, mirrored (exact symmetry)
            const double s1 = isd[gi < gj ? gi : gj], s2 = isd[gi < gj ? gj : gi];
            if (SPLIT) {
                const double s = gi == gj ? static_cast<double>(kSplitScale) : k * s1 * s2 * kSplitScale;
                const __half h = __double2half(s);
                hi[li * g.ld + gj] = h;
                lo[li * g.ld + gj] = __double2half(s - static_cast<double>(__half2float(h)));
            } else {
                a64[li * g.ld + gj] = gi == gj ? g.inv_n : g.inv_n * k * s1 * s2;
            }
        }
    }
    if (bad) atomicOr(flags, 1u);
}

}  // namespace

cudaError_t launch_poly_gram(const GramArgs& g, int degree, double offset, double* isd, __half* hi, __half* lo,
                             double* a64, unsigned* flags, cudaStream_t stream) {
    const double deg = static_cast<double>(degree);
    if (isd)  // isd == nullptr: the raw K of ops::polynomial_gram into a64
        poly_diag_kernel<<<static_cast<unsigned>((g.n + 255) / 256), 256, 0, stream>>>(g.x, g.n, g.dx, g.x_rs, g.x_cs,
                                                                                      deg, offset, isd, flags);
    dim3 grid(static_cast<unsigned>((g.n + TN - 1) / TN), static_cast<unsigned>((g.rows + TM - 1) / TM));
    if (hi) poly_gram_kernel<true><<<grid, 256, 0, stream>>>(g, deg, offset, isd, hi, lo, nullptr, flags);
    else poly_gram_kernel<false><<<grid, 256, 0, stream>>>(g, deg, offset, isd, nullptr, nullptr, a64, flags);
    return cudaGetLastError();
}

cudaError_t launch_gram_f64(const GramArgs& g, double* a, cudaStream_t stream) {
    if (g.row0 == 0 && g.rows == g.n) {  // whole matrix: symmetric tiles
        const int64_t tiles = (g.n + TM - 1) / TM;
        if (tiles * (tiles + 1) / 2 <= 0x7FFFFFFF) {
            gram_sym_f64_kernel<<<static_cast<unsigned>(tiles * (tiles + 1) / 2), 256, 0, stream>>>(
                g, a, static_cast<int>(tiles));
            return cudaGetLastError();
        }
    }
    dim3 grid(static_cast<unsigned>((g.n + TN - 1) / TN), static_cast<unsigned>((g.rows + TM - 1) / TM));
    gram_kernel<double, false><<<grid, 256, 0, stream>>>(g, nullptr, nullptr, a);
    return cudaGetLastError();
}

__global__ void scale_columns_kernel(const double* __restrict__ x, int64_t n, int d, int64_t rs, int64_t cs,
                                     double scale, double* __restrict__ out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n * d) return;
    const int64_t i = t % n, k = t / n;
    out[t] = x[i * rs + k * cs] * scale;
}

cudaError_t launch_scale_columns(const double* x, int64_t n, int d, int64_t rs, int64_t cs, double scale, double* out,
                                 cudaStream_t stream) {
    const int64_t total = n * d;
    if (total == 0) return cudaSuccess;
    scale_columns_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, stream>>>(x, n, d, rs, cs, scale, out);
    return cudaGetLastError();
}

cudaError_t launch_check_samples(const double* x, int64_t n, int d, int64_t rs, int64_t cs, unsigned* flags,
                                 cudaStream_t stream) {
    const int64_t total = n * d;
    const int64_t blocks = std::min<int64_t>(1184, (total + 255) / 256);
    check_samples_kernel<<<static_cast<unsigned>(blocks > 0 ? blocks : 1), 256, 0, stream>>>(x, n, d, rs, cs, flags);
    return cudaGetLastError();
}

cudaError_t launch_matrix_to_split(const double* a, int64_t rows, int64_t cols, int64_t lda, double scale,
                                   __half* hi, __half* lo, int64_t ld, cudaStream_t stream) {
    matrix_to_split_kernel<<<row_grid(rows, cols), 256, 0, stream>>>(a, rows, cols, lda, scale, hi, lo, ld);
    return cudaGetLastError();
}

cudaError_t launch_split_to_f64(const __half* hi, const __half* lo, int64_t rows, int64_t cols, int64_t ld,
                                double unscale, double* out, int64_t ldo, cudaStream_t stream) {
    split_to_f64_kernel<<<row_grid(rows, cols), 256, 0, stream>>>(hi, lo, rows, cols, ld, unscale, out, ldo);
    return cudaGetLastError();
}

cudaError_t launch_hadamard_split(const __half* ahi, const __half* alo, const __half* bhi, const __half* blo,
                                  int64_t rows, int64_t cols, int64_t ld, int64_t row0, double factor,
                                  double diag_value, __half* chi, __half* clo, cudaStream_t stream) {
    hadamard_split_kernel<<<row_grid(rows, cols), 256, 0, stream>>>(ahi, alo, bhi, blo, rows, cols, ld, row0, factor,
                                                                      diag_value, chi, clo);
    return cudaGetLastError();
}

namespace {
__global__ void scaled_product_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t count,
                                      double scale, double* __restrict__ c) {
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        c[k] = scale * (a[k] * b[k]);
}
}  // namespace

cudaError_t launch_scaled_product(const double* a, const double* b, int64_t count, double scale, double* c,
                                  cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    const int64_t blocks = std::min<int64_t>(148 * 8, (count + 255) / 256);
    scaled_product_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(a, b, count, scale, c);
    return cudaGetLastError();
}

namespace {
// hadamard_joint of L >= 3 factors (proj/src/kernel.cpp:74-101) in the caller's canonical order:
// p = M_0; p = 1.0·(p·M_l) for the middle factors (= p·M_l exactly); p = scale·(p·M_{L-1}); diag 1/n
__global__ void hadamard_n_kernel(HadamardFactors h, int64_t rows, int64_t cols, int64_t ld, int64_t row0,
                                  double scale, double inv_n, double out_unscale, double* __restrict__ c64,
                                  __half* __restrict__ chi, __half* __restrict__ clo) {
    const int64_t i = blockIdx.y;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < cols;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k = i * ld + j;
        auto val = [&](int l) {
            return h.a64[l] ? h.a64[l][k]
                            : (static_cast<double>(__half2float(h.hi[l][k])) +
                               static_cast<double>(__half2float(h.lo[l][k]))) * h.unscale[l];
        };
        double v;
        if (row0 + i == j) {
            v = inv_n;
        } else {
            v = val(0);
            for (int l = 1; l + 1 < h.count; ++l) v = v * val(l);
            v = scale * (v * val(h.count - 1));
        }
        if (c64) {
            c64[k] = v;
        } else {
            const double s = v / out_unscale;
            const __half hh = __double2half(s);
            chi[k] = hh;
            clo[k] = __double2half(s - static_cast<double>(__half2float(hh)));
        }
    }
}

// order key material: one 64-bit hash per row of the stored entries (fp64 values or the hi/lo
// fp16 pairs), lanes of a warp hashing interleaved elements, folded in lane order
__global__ void row_hash_kernel(const double* __restrict__ a64, const __half* __restrict__ hi,
                                const __half* __restrict__ lo, int64_t rows, int64_t cols, int64_t ld,
                                uint64_t* __restrict__ out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    if (r >= rows) return;
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int64_t j = lane; j < cols; j += 32) {
        uint64_t w;
        if (a64) {
            w = static_cast<uint64_t>(__double_as_longlong(a64[r * ld + j]));
        } else {
            w = (static_cast<uint64_t>(__half_as_ushort(hi[r * ld + j])) << 16) | __half_as_ushort(lo[r * ld + j]);
        }
        h = (h ^ w) * 0x100000001b3ULL;
    }
    uint64_t acc = 0;
    for (int l = 0; l < 32; ++l) {  // fold the lanes' hashes in lane order
        const uint64_t hl = __shfl_sync(0xffffffffu, h, l);
        acc = l == 0 ? hl : ((acc ^ hl) * 0x100000001b3ULL);
    }
    if (lane == 0) out[r] = acc;
}
}  // namespace

cudaError_t launch_hadamard_n(const HadamardFactors& h, int64_t rows, int64_t cols, int64_t ld, int64_t row0,
                              double scale, double inv_n, double out_unscale, double* c64, __half* chi, __half* clo,
                              cudaStream_t stream) {
    hadamard_n_kernel<<<row_grid(rows, cols), 256, 0, stream>>>(h, rows, cols, ld, row0, scale, inv_n, out_unscale,
                                                                 c64, chi, clo);
    return cudaGetLastError();
}

cudaError_t launch_row_hash(const double* a64, const __half* hi, const __half* lo, int64_t rows, int64_t cols,
                            int64_t ld, uint64_t* out, cudaStream_t stream) {
    if (rows <= 0) return cudaSuccess;
    row_hash_kernel<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, stream>>>(a64, hi, lo, rows, cols, ld, out);
    return cudaGetLastError();
}

cudaError_t launch_hadamard_f64(const double* a, const double* b, int64_t rows, int64_t cols, int64_t ld,
                                int64_t row0, double n, double* c, cudaStream_t stream) {
    hadamard_f64_kernel<<<row_grid(rows, cols), 256, 0, stream>>>(a, b, rows, cols, ld, row0, n, c);
    return cudaGetLastError();
}

}  // namespace rb
