// Pass epilogue and small panel kernels.
//
// The pass epilogue is where the reference's recurrence arithmetic
// (proj/src/poly.cpp:97-134) and trace dots (proj/src/hutchpp.cpp:33-51) go:
//   T_new = a1·(A·T_cur) + a2·T_cur + a3·T_prev
// covers IntPower (1,0,0), Taylor (1/v,-1,0), Chebyshev first step
// (scale,-center,0) and later steps (2·scale,-2·center,-1), and the shifted
// power iteration (−g, v·g, 0). Per probe column it accumulates, in fp64,
// x0·T_new (trace form), T_cur·T_new (Rayleigh) and T_new·T_new, and the
// column max |T_new| that sets the next pass's fp16 plane scale.
#include <cuda_fp16.h>

#include <algorithm>

#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"
#include "kernels.h"

namespace rb {

namespace {


__device__ __forceinline__ int64_t streamk_owner(int64_t i, int64_t total, int grid) {
    return ((i + 1) * grid + total - 1) / total - 1;
}

__device__ __forceinline__ double cm_value(const unsigned* cm, int j) {
    return cm ? static_cast<double>(__uint_as_float(cm[j])) : 0.0;
}

// exponent e with bound * 2^e < 2^kPanelTarget
__device__ __forceinline__ int plane_exponent(double bound) {
    if (!(bound > 0.0) || !isfinite(bound)) return 0;
    int E;
    frexp(bound, &E);  // bound < 2^E
    int e = kPanelTarget - E;
    e = max(-120, min(120, e));
    return e;
}

// 2^e as an exact double for the exponents the planes use (|e| <= 120): scaling by it equals ldexp
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double(static_cast<long long>(1023 + e) << 52); }

// fp16 operand (+ optional low plane carrying the rounding residual)
__device__ __forceinline__ void split_store(double v, __half* hi, __half* lo, int64_t idx) {
    const __half h = __double2half(v);
    hi[idx] = h;
    if (lo) lo[idx] = __double2half(v - static_cast<double>(__half2float(h)));
}

// columns per epilogue CTA (grid = row blocks x column groups). Measured on the config-4 fused MI step
// (93 epilogues, ncu launch list): 16 columns 29.3 ms, 8: 14.8 ms, 4: 9.0 ms, 2: 8.4 ms -- short CTAs
// keep more loads in flight per SM than long per-thread column loops
constexpr int kEpiCols = 2;

// y += base[c·stride] for c = 0 .. n-1, in slot order (fp64), 16 loads in flight: the symmetric product
// leaves nb ≈ 400 slots per row block, which a load-add chain walked one L2 round trip at a time
// (96 us per s = 1 epilogue at n = 50k)
template <typename PT>
__device__ __forceinline__ void sum_slots(double& y, const PT* base, int64_t stride, int64_t n) {
    int64_t c = 0;
    for (; c + 16 <= n; c += 16) {
        PT v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = base[(c + u) * stride];
#pragma unroll
        for (int u = 0; u < 16; ++u) y += static_cast<double>(v[u]);
    }
    for (; c < n; ++c) y += static_cast<double>(base[c * stride]);
}

template <typename PT, typename ST, bool SPLIT, int ER>
__global__ void __launch_bounds__(ER) epilogue_kernel(EpiArgs<PT, ST> p) {
    constexpr int NW = ER / 32;
    __shared__ double red[3][NW][kEpiCols];
    __shared__ float mxs[NW][kEpiCols];
    __shared__ int64_t sown[4];                        // the row block's partial slot ranges
    __shared__ double sscale[kEpiCols], snext[kEpiCols];  // 2^-e_cur·unscale and 2^e_next per column
    const int jb0 = blockIdx.y * kEpiCols, jb1 = min(p.s, jb0 + kEpiCols);
    const int r = blockIdx.x;
    const int tid = threadIdx.x;
    const int warp = tid / 32, lane = tid % 32;
    const int64_t i = static_cast<int64_t>(r) * ER + tid;
    const bool valid = i < p.rows;
    const int64_t cl = p.cluster, rb = r / cl, rr = r % cl;
    const double gs = p.gscale ? *p.gscale : 1.0;  // fl(1.0·a) = a: no device scale, same coefficients
    const double a1 = p.a1 * gs, a2 = p.a2 * gs, a3 = p.a3 * gs;
    // block-uniform work once per block (the 64-bit stream-K owner divisions and the plane exponents
    // were ~40 % of the kernel's instructions when every thread repeated them)
    if (tid == 0) {
        // slots [c_lo, c_hi] of row block rb under a plan (whole row blocks: slot rb)
        auto owners = [&](int64_t KT, int64_t total_iters, int grid, int64_t dp, int64_t* out) {
            out[0] = 0, out[1] = 0;
            if (rb >= dp) {
                const int64_t rt = rb - dp, tail = total_iters - dp * KT;
                out[0] = streamk_owner(rt * KT, tail, grid);
                out[1] = streamk_owner((rt + 1) * KT - 1, tail, grid);
            }
        };
        if (p.symv_nb > 0) {  // slots rb·nb .. rb·nb + nb - 1 (cluster 1: slot = rb + c)
            sown[0] = rb * (p.symv_nb - 1), sown[1] = sown[0] + p.symv_nb - 1;
        } else {
            owners(p.k_tiles, p.total_iters, p.grid, p.dp_blocks, sown);
        }
        if (p.partial2) owners(p.k_tiles2, p.total_iters2, p.grid2, p.dp_blocks2, sown + 2);
        else sown[2] = 0, sown[3] = -1;
    }
    if (SPLIT && tid < kEpiCols && jb0 + tid < jb1) {
        const int j = jb0 + tid;
        const double growth = fabs(a1) * p.a_norm + fabs(a2);
        const double bound = growth * cm_value(p.cmax_cur, j) + fabs(a3) * cm_value(p.cmax_prev, j);
        const int e = plane_exponent(bound);
        if (r == 0) p.e_next[j] = e;
        sscale[tid] = pow2(-p.e_cur[j]);
        snext[tid] = pow2(e);
    }
    __syncthreads();
    const int64_t c_lo = sown[0], c_hi = sown[1], c2_lo = sown[2], c2_hi = sown[3];

    // all of this block's loads first (kEpiCols independent columns in flight per thread: the loop
    // below was latency-bound, one column's loads at a time -- 150 us per config-4 epilogue), then
    // the arithmetic in the same order as before
    double ys[kEpiCols];
    ST tcs[kEpiCols], tps[kEpiCols], x0s[kEpiCols];
#pragma unroll
    for (int jj = 0; jj < kEpiCols; ++jj) {
        const int j = jb0 + jj;
        ys[jj] = 0.0;
        tcs[jj] = tps[jj] = x0s[jj] = ST(0);
        if (j >= jb1) continue;
        double y = 0.0;
        const int64_t stride = cl * p.npad * ER;
        sum_slots(y, p.partial + ((cl * (rb + c_lo) + rr) * p.npad + j) * ER + tid, stride, c_hi - c_lo + 1);
        if (c2_hi >= c2_lo)
            sum_slots(y, p.partial2 + ((cl * (rb + c2_lo) + rr) * p.npad + j) * ER + tid, stride, c2_hi - c2_lo + 1);
        ys[jj] = y;
        const int64_t idx = static_cast<int64_t>(j) * p.ld + i;
        if (valid) {
            tcs[jj] = p.t_cur[idx];
            if (p.t_prev) tps[jj] = p.t_prev[idx];
            x0s[jj] = p.x0[idx];
        }
    }
#pragma unroll
    for (int jj = 0; jj < kEpiCols; ++jj) {
        const int j = jb0 + jj;
        if (j >= jb1) break;
        double y = ys[jj];
        if (SPLIT) y = (y * p.unscale) * sscale[jj];  // = ldexp(y·unscale, −e_cur) (exact power of two)
        const double tc = static_cast<double>(tcs[jj]), tp = static_cast<double>(tps[jj]),
                     x0 = static_cast<double>(x0s[jj]);
        const int64_t idx = static_cast<int64_t>(j) * p.ld + i;
        double tn = a1 * y + a2 * tc + a3 * tp;
        const ST tns = static_cast<ST>(tn);
        tn = static_cast<double>(tns);
        if (!valid) tn = 0.0;
        if (valid) {
            p.t_new[idx] = tns;
            if (p.acc) p.acc[idx] += p.acc_coef * tn;
        }
        if (SPLIT && valid) split_store(tn * snext[jj], p.vop, p.vop_lo, idx);
        const double d1 = warp_sum(x0 * tn);
        const double d2 = warp_sum(tc * tn);
        const double d3 = warp_sum(tn * tn);
        const float mx = warp_max(static_cast<float>(fabs(tn)));
        if (lane == 0) {
            red[0][warp][j - jb0] = d1;
            red[1][warp][j - jb0] = d2;
            red[2][warp][j - jb0] = d3;
            mxs[warp][j - jb0] = mx;
        }
    }
    __syncthreads();
    const int R = gridDim.x, w = jb1 - jb0;
    if (tid < w) {  // one atomic per column and block (the per-warp atomics contended on s addresses)
        float m = mxs[0][tid];
#pragma unroll
        for (int ww = 1; ww < NW; ++ww) m = fmaxf(m, mxs[ww][tid]);
        atomicMax(p.cmax_new + jb0 + tid, __float_as_uint(m));
    }
    for (int t = tid; t < 3 * w; t += blockDim.x) {
        const int q = t / w, jj = t % w;
        double v = red[q][0][jj];
#pragma unroll
        for (int ww = 1; ww < NW; ++ww) v += red[q][ww][jj];
        p.stats[(static_cast<int64_t>(q) * R + r) * p.s + jb0 + jj] = v;
    }
}

// grid = row blocks x column groups of kEpiCols (as the pass epilogue: a serial loop over every column
// in one block left the first pass's statistics latency-bound, 21-108 us per launch); each block's
// per-column sums are the same warp sums added in the same warp order as before
template <typename ST, int ER>
__global__ void __launch_bounds__(ER) prep_stats_kernel(PrepArgs<ST> p) {
    constexpr int NW = ER / 32;
    __shared__ double red[NW][kEpiCols];
    const int r = blockIdx.x;
    const int jb0 = blockIdx.y * kEpiCols, jb1 = min(p.s, jb0 + kEpiCols);
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int64_t i = static_cast<int64_t>(r) * ER + tid;
    const bool valid = i < p.rows;
    ST xs[kEpiCols];
#pragma unroll
    for (int jj = 0; jj < kEpiCols; ++jj)  // every column's load in flight first
        xs[jj] = (valid && jb0 + jj < jb1) ? static_cast<ST>(p.x[static_cast<int64_t>(jb0 + jj) * p.ldx + i]) : ST(0);
#pragma unroll
    for (int jj = 0; jj < kEpiCols; ++jj) {
        const int j = jb0 + jj;
        if (j >= jb1) break;
        double v = 0.0;
        if (valid) {
            const ST vs = xs[jj];
            v = static_cast<double>(vs);
            p.t0[static_cast<int64_t>(j) * p.ld + i] = vs;
            if (p.acc) p.acc[static_cast<int64_t>(j) * p.ld + i] = p.acc_coef * v;
        }
        const double d = warp_sum(v * v);
        const float mx = warp_max(static_cast<float>(fabs(v)));
        if (lane == 0) {
            red[warp][jj] = d;
            atomicMax(p.cmax0 + j, __float_as_uint(mx));
        }
    }
    __syncthreads();
    const int R = gridDim.x;
    if (tid < jb1 - jb0) {
        const int j = jb0 + tid;
        double v = red[0][tid];
#pragma unroll
        for (int w = 1; w < NW; ++w) v += red[w][tid];
        // q = 0 (x0·T0), 1 (T0·T0 as "Rayleigh" slot), 2 (T0·T0)
        p.stats[(0 * static_cast<int64_t>(R) + r) * p.s + j] = v;
        p.stats[(1 * static_cast<int64_t>(R) + r) * p.s + j] = v;
        p.stats[(2 * static_cast<int64_t>(R) + r) * p.s + j] = v;
    }
}

__global__ void prep_planes_kernel(PrepArgs<float> p) {
    const int j = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int e = plane_exponent(static_cast<double>(__uint_as_float(p.cmax0[j])));
    if (blockIdx.x == 0 && threadIdx.x == 0) p.e0[j] = e;
    if (i >= p.rows) return;
    const int64_t idx = static_cast<int64_t>(j) * p.ld + i;
    split_store(ldexp(static_cast<double>(p.t0[idx]), e), p.vop, p.vop_lo, idx);
}

// out[p][q][j] = sum over row blocks [r0, r0 + count) of stats[p][q][r][j] (R row blocks per (p, q))
// one warp per output: lane l sums row blocks l, l + 32, ... of the range in order, then a fixed xor
// tree (the order depends only on the count and the blocks' positions in the range, so a group of a
// grouped stack reduces exactly as the same rows in their own session); a thread per output walked
// the ~400 row blocks of an s = 1 pass one L2 round trip at a time (35 us per launch)
__global__ void reduce_stats_kernel(const double* __restrict__ stats, int passes, int R, int r0, int count, int s,
                                    double* __restrict__ out) {
    const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    const int64_t total = static_cast<int64_t>(passes) * 3 * s;
    if (t >= total) return;  // warp-uniform
    const int64_t j = t % s;
    const int64_t pq = t / s;  // pass*3 + q
    const double* src = stats + (pq * R + r0) * s + j;
    double acc = 0.0;
    for (int r = lane; r < count; r += 32) acc += src[static_cast<int64_t>(r) * s];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[t] = acc;
}

template <typename ST>
__global__ void state_to_f64_kernel(const ST* __restrict__ st, int64_t rows, int64_t ld, double* __restrict__ out,
                                    int64_t ldo) {
    const int j = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < rows) out[static_cast<int64_t>(j) * ldo + i] = static_cast<double>(st[static_cast<int64_t>(j) * ld + i]);
}

// ---- panel gram: partial[cta][a][b] = sum_{rows of cta} X[i][a] Z[i][b] ----
constexpr int GR = 32;  // rows per smem chunk
__global__ void __launch_bounds__(256) panel_gram_kernel(const double* __restrict__ x, int p, int64_t ldx,
                                                         const double* __restrict__ z, int q, int64_t ldz,
                                                         int64_t rows, double* __restrict__ partial,
                                                         unsigned* __restrict__ ticket, double* __restrict__ out) {
    extern __shared__ double sm[];
    double* xs = sm;            // [GR][p]
    double* zs = sm + GR * p;   // [GR][q]
    const int G = gridDim.x;
    const int64_t per = (rows + G - 1) / G;
    const int64_t r0 = per * blockIdx.x;
    const int64_t r1 = min(rows, r0 + per);
    const int outs = p * q;
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.0;
    for (int64_t c0 = r0; c0 < r1; c0 += GR) {
        for (int idx = threadIdx.x; idx < GR * p; idx += blockDim.x) {
            const int a = idx / GR, rr = idx % GR;
            const int64_t gi = c0 + rr;
            xs[rr * p + a] = gi < r1 ? x[static_cast<int64_t>(a) * ldx + gi] : 0.0;
        }
        for (int idx = threadIdx.x; idx < GR * q; idx += blockDim.x) {
            const int b = idx / GR, rr = idx % GR;
            const int64_t gi = c0 + rr;
            zs[rr * q + b] = gi < r1 ? z[static_cast<int64_t>(b) * ldz + gi] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int o = threadIdx.x + u * blockDim.x;
            if (o < outs) {
                const int a = o % p, b = o / p;
                double t = acc[u];
                for (int rr = 0; rr < GR; ++rr) t = fma(xs[rr * p + a], zs[rr * q + b], t);
                acc[u] = t;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int o = threadIdx.x + u * blockDim.x;
        if (o < outs) partial[static_cast<int64_t>(blockIdx.x) * outs + o] = acc[u];
    }
    // the last CTA to finish sums every CTA's partial in CTA order (the separate reduce kernel's
    // order: bitwise the same Gram), saving a launch per Gram of the latency-bound QR steps
    if (!ticket) return;
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == static_cast<unsigned>(G - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int o = threadIdx.x; o < outs; o += blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < G; ++c) s += __ldcg(partial + static_cast<int64_t>(c) * outs + o);
        out[o] = s;
    }
    if (threadIdx.x == 0) *ticket = 0u;  // ready for the next Gram on this stream
}

__global__ void panel_gram_reduce_kernel(const double* __restrict__ partial, int G, int outs,
                                         double* __restrict__ out) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= outs) return;
    double acc = 0.0;
    for (int c = 0; c < G; ++c) acc += partial[static_cast<int64_t>(c) * outs + o];
    out[o] = acc;
}

__global__ void panel_update_kernel(double beta, const double* __restrict__ g, int64_t ldg,
                                    const double* __restrict__ x, int p, int64_t ldx, const double* __restrict__ c,
                                    int q, int64_t rows, double* __restrict__ w, int64_t ldw) {
    extern __shared__ double cs[];  // [p][q] column-major c[a + b*p]
    for (int t = threadIdx.x; t < p * q; t += blockDim.x) cs[t] = c[t];
    __syncthreads();
    const int b = blockIdx.y;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= rows) return;
    double acc = 0.0;
    for (int a = 0; a < p; ++a) acc = fma(x[static_cast<int64_t>(a) * ldx + i], cs[a + b * p], acc);
    const double base = (beta != 0.0 && g) ? beta * g[static_cast<int64_t>(b) * ldg + i] : 0.0;
    w[static_cast<int64_t>(b) * ldw + i] = base + acc;
}

// ---- reference RNG (proj/src/rng.cpp:8-54) on the device ----
__device__ __forceinline__ uint64_t dmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t dderive(uint64_t seed, uint64_t tag) {
    return dmix64(seed ^ dmix64(tag + 0x6a09e667f3bcc909ULL));
}

__global__ void rng_panel_kernel(uint64_t base_key, bool derive, int kind, int64_t row0, int64_t rows, int j0,
                                 double* __restrict__ out, int64_t ld, int* err) {
    const int j = blockIdx.y;
    const uint64_t key = derive ? dderive(base_key, static_cast<uint64_t>(j0 + j)) : base_key;
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double* col = out + static_cast<int64_t>(j) * ld;
    if (kind == 1) {
        if (t >= rows) return;
        const uint64_t u = dmix64(key ^ dmix64(static_cast<uint64_t>(row0 + t)));
        col[t] = (u >> 63) ? -1.0 : 1.0;
        return;
    }
    // Gaussian: local pair t covers elements 2t (cos) and 2t+1 (sin); global counters row0+2t, row0+2t+1.
    const int64_t i0 = 2 * t;
    if (i0 >= rows) return;
    const uint64_t w1 = dmix64(key ^ dmix64(static_cast<uint64_t>(row0 + 2 * t)));
    const uint64_t w2 = dmix64(key ^ dmix64(static_cast<uint64_t>(row0 + 2 * t + 1)));
    const double u1 = static_cast<double>(w1 >> 11) * 0x1.0p-53;
    const double u2 = static_cast<double>(w2 >> 11) * 0x1.0p-53;
    if (u1 <= 0.0) atomicExch(err, 1);  // the reference would redraw (p = 2^-53 per pair)
    const double rr = sqrt(-2.0 * log(u1));
    const double theta = 2.0 * 3.141592653589793 * u2;
    col[i0] = rr * cos(theta);
    if (i0 + 1 < rows) col[i0 + 1] = rr * sin(theta);
}

}  // namespace

TensorMapEncodeFn tensor_map_encoder() {
    static const TensorMapEncodeFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<TensorMapEncodeFn>(p);
        return static_cast<TensorMapEncodeFn>(nullptr);
    }();
    return fn;
}

cudaError_t ensure_smem_attr(const void* fn, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({fn, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({fn, dev});
    return e;
}

namespace {
__global__ void power_norm_kernel(const double* __restrict__ red, double* __restrict__ g) {
    if (threadIdx.x == 0 && blockIdx.x == 0) g[0] = 1.0 / sqrt(red[2]);  // spectrum.cpp:45-47 (x = y/||y||)
}
}  // namespace

cudaError_t launch_power_norm(const double* red, double* g, cudaStream_t stream) {
    power_norm_kernel<<<1, 32, 0, stream>>>(red, g);
    return cudaGetLastError();
}

cudaError_t launch_epilogue_split(const EpiArgs<float, float>& a, cudaStream_t stream) {
    if (a.s > kMaxPanelCols) return cudaErrorInvalidValue;
    const unsigned groups = static_cast<unsigned>((a.s + kEpiCols - 1) / kEpiCols);
    if (a.rows_per_block == 256) {
        const unsigned R = static_cast<unsigned>((a.rows + 255) / 256);
        epilogue_kernel<float, float, true, 256><<<dim3(R, groups), 256, 0, stream>>>(a);
    } else if (a.rows_per_block == 128) {
        const unsigned R = static_cast<unsigned>((a.rows + 127) / 128);
        epilogue_kernel<float, float, true, 128><<<dim3(R, groups), 128, 0, stream>>>(a);
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_epilogue_f64(const EpiArgs<double, double>& a, cudaStream_t stream) {
    if (a.s > kMaxPanelCols || a.rows_per_block != 128) return cudaErrorInvalidValue;
    const unsigned R = static_cast<unsigned>((a.rows + 127) / 128);
    const unsigned groups = static_cast<unsigned>((a.s + kEpiCols - 1) / kEpiCols);
    epilogue_kernel<double, double, false, 128><<<dim3(R, groups), 128, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_prepare_split_stats(const PrepArgs<float>& a, cudaStream_t stream) {
    if (a.s > kMaxPanelCols) return cudaErrorInvalidValue;
    const unsigned groups = static_cast<unsigned>((a.s + kEpiCols - 1) / kEpiCols);
    if (a.rows_per_block == 256) {
        const int R = static_cast<int>((a.rows + 255) / 256);
        if (R > 0) prep_stats_kernel<float, 256><<<dim3(R, groups), 256, 0, stream>>>(a);
    } else if (a.rows_per_block == 128) {
        const int R = static_cast<int>((a.rows + 127) / 128);
        if (R > 0) prep_stats_kernel<float, 128><<<dim3(R, groups), 128, 0, stream>>>(a);
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_prepare_split_planes(const PrepArgs<float>& a, cudaStream_t stream) {
    dim3 grid(static_cast<unsigned>(std::max<int64_t>(1, (a.rows + 255) / 256)), a.s);
    prep_planes_kernel<<<grid, 256, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_prepare_f64(const PrepArgs<double>& a, cudaStream_t stream) {
    if (a.s > kMaxPanelCols || a.rows_per_block != 128) return cudaErrorInvalidValue;
    const int R = static_cast<int>((a.rows + 127) / 128);
    const unsigned groups = static_cast<unsigned>((a.s + kEpiCols - 1) / kEpiCols);
    prep_stats_kernel<double, 128><<<dim3(R, groups), 128, 0, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_reduce_stats(const double* stats, int passes, int row_blocks, int s, double* out,
                                cudaStream_t stream, int r0, int count) {
    const int64_t total = static_cast<int64_t>(passes) * 3 * s;
    if (total == 0) return cudaSuccess;
    if (count < 0) count = row_blocks - r0;
    reduce_stats_kernel<<<static_cast<unsigned>((total + 3) / 4), 128, 0, stream>>>(stats, passes, row_blocks, r0,
                                                                                    count, s, out);
    return cudaGetLastError();
}

__global__ void merge_tails_kernel(const __half* planes, int64_t slice_elems, int64_t tail_off, int world, int s,
                                   unsigned* out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= s) return;
    unsigned m = 0;
    for (int q = 0; q < world; ++q)
        m = max(m, reinterpret_cast<const unsigned*>(planes + q * slice_elems + tail_off)[j]);
    out[j] = m;
}

cudaError_t launch_merge_tails(const __half* planes, int64_t slice_elems, int64_t tail_off, int world, int s,
                               unsigned* out, cudaStream_t stream) {
    merge_tails_kernel<<<(s + 127) / 128, 128, 0, stream>>>(planes, slice_elems, tail_off, world, s, out);
    return cudaGetLastError();
}

cudaError_t launch_state_to_f64(const void* state, bool is_f32, int64_t rows, int s, int64_t ld, double* out,
                                int64_t ldo, cudaStream_t stream) {
    dim3 grid(static_cast<unsigned>((rows + 255) / 256), s);
    if (is_f32)
        state_to_f64_kernel<float><<<grid, 256, 0, stream>>>(static_cast<const float*>(state), rows, ld, out, ldo);
    else
        state_to_f64_kernel<double><<<grid, 256, 0, stream>>>(static_cast<const double*>(state), rows, ld, out, ldo);
    return cudaGetLastError();
}

cudaError_t launch_panel_gram(const double* x, int p, int64_t ldx, const double* z, int q, int64_t ldz,
                              int64_t rows, double* partial, int grid, double* out, cudaStream_t stream,
                              unsigned* ticket) {
    if (p <= 0 || q <= 0) return cudaSuccess;
    if (p * q > 8 * 256) return cudaErrorInvalidValue;
    const size_t smem = static_cast<size_t>(GR) * (p + q) * sizeof(double);
    if (smem > 48 * 1024) return cudaErrorInvalidValue;
    if (!ticket) {  // no completion counter: separate reduction
        panel_gram_kernel<<<grid, 256, smem, stream>>>(x, p, ldx, z, q, ldz, rows, partial, nullptr, nullptr);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        const int outs = p * q;
        panel_gram_reduce_kernel<<<(outs + 127) / 128, 128, 0, stream>>>(partial, grid, outs, out);
        return cudaGetLastError();
    }
    panel_gram_kernel<<<grid, 256, smem, stream>>>(x, p, ldx, z, q, ldz, rows, partial, ticket, out);
    return cudaGetLastError();
}

cudaError_t launch_panel_update(double beta, const double* g, int64_t ldg, const double* x, int p, int64_t ldx,
                                const double* c, int q, int64_t rows, double* w, int64_t ldw, cudaStream_t stream) {
    if (q <= 0) return cudaSuccess;
    const size_t smem = static_cast<size_t>(p) * q * sizeof(double);
    if (smem > 48 * 1024) return cudaErrorInvalidValue;
    dim3 grid(static_cast<unsigned>((rows + 255) / 256), q);
    panel_update_kernel<<<grid, 256, smem, stream>>>(beta, g, ldg, x, p, ldx, c, q, rows, w, ldw);
    return cudaGetLastError();
}

cudaError_t launch_rng_panel(uint64_t base_key, bool derive, int kind, int64_t row0, int64_t rows, int cols, int j0,
                             double* out, int64_t ld, int* err_flag, cudaStream_t stream) {
    if (cols <= 0 || rows <= 0) return cudaSuccess;
    if (kind != 1 && (row0 & 1)) return cudaErrorInvalidValue;
    const int64_t work = kind == 1 ? rows : (rows + 1) / 2;
    dim3 grid(static_cast<unsigned>((work + 255) / 256), cols);
    rng_panel_kernel<<<grid, 256, 0, stream>>>(base_key, derive, kind, row0, rows, j0, out, ld, err_flag);
    return cudaGetLastError();
}

}  // namespace rb
