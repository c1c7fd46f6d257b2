// Tensor-core Gram for the fp32 configurations (north star subsystem (1); SURVEY §8 a1+a2+a4):
//   K_ij = exp(−‖x_i − x_j‖² / (2σ²)),   A = K/n stored as the fp16 hi/lo planes of K·2^14,
// with ‖x_i − x_j‖² formed from a tcgen05 X·Xᵀ contraction instead of per-entry FFMA chains
// (the reference's expanded form, proj/src/ops.cpp:9-20,39-47, sq_i + sq_j − 2 x_i·x_j).
//
// fp32-class accuracy from the tf32 tensor cores by the 3xTF32 split: with z = x/(σ√2) (both
// variables concatenated for a joint kernel), z = hi + lo (hi, lo tf32), the K-concatenated operands
//   A_i = [hi_i | lo_i | hi_i],   B_j = [hi_j | hi_j | lo_j]
// give S = hi·hi + lo·hi + hi·lo ≈ z_i·z_j (the dropped lo·lo is 2^-22 relative), accumulated in
// fp32 in TMEM. The epilogue forms arg = log2(e)·(2S − sq_i − sq_j) (sq from fp64), exp2, K_ii = 1,
// the K·2^14 hi/lo split, and writes the tile and (through shared memory) its mirror: only the
// upper-triangle tiles are computed.
//
// Warp roles: 0 TMA (A/B K sub-tiles, 2-stage ring), 1 MMA issuer (M=128, N=128, K=8 tf32
// steps into one of two TMEM accumulators), 2-17 epilogue (four warpgroups: column quarters) whose
// staged tiles leave through TMA stores.
// Persistent CTAs walk the upper-triangle tiles row-major (consecutive tiles share A in L2).
#include <algorithm>
#include <cmath>
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace rb {

namespace {

constexpr int GT = 128;           // tile (rows and columns)
constexpr int KS = 32;            // fp32 per K sub-tile: one 128-byte SW128 row
constexpr int kGStages = 2;
constexpr int kGEpiWarps = 16;  // epilogue warps: 4 groups of 32 columns x 4 TMEM lane quarters
constexpr int kGThreads = 32 * (2 + kGEpiWarps);
constexpr int kSub = GT * KS * 4;  // 16 KB per operand sub-tile
constexpr int kPlane = GT * GT * 2;  // one staged [128][128] fp16 plane: two 128B-swizzled boxes of 64 columns
// ring | D (tile, row-major: hi, lo) | T (transposed tile: hi, lo)
constexpr int kGSmem = kGStages * 2 * kSub + 4 * kPlane + 1024;

// byte offset of fp16 element (r, c) in a staged plane (TMA SWIZZLE_128B boxes of 128 rows x 64 columns)
__device__ __forceinline__ uint32_t sw_off(int r, int c) {
    return static_cast<uint32_t>((c >> 6) * (GT * 128) + r * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4) + ((c & 7) << 1));
}

struct GtArgs {
    int64_t nb, tiles;  // column blocks; tiles (upper triangle, or shard row blocks x nb)
    int rect;           // 1: a row shard [row0, row0 + rows): all its tiles, no mirroring
    int64_t row0, row_end;
    int ksub;           // K sub-tiles (KP / 32)
    int64_t n, ld;
    const float* sq;    // ‖z_i‖², [round_up(n,128)]
    __half* hi;
    __half* lo;
};

__device__ __forceinline__ void tile_of(int64_t t, int64_t nb, int64_t* bi, int64_t* bj) {
    auto start = [nb](int64_t b) { return b * nb - b * (b - 1) / 2; };
    const double q = 2.0 * nb + 1.0;
    int64_t i = static_cast<int64_t>((q - sqrt(q * q - 8.0 * static_cast<double>(t))) * 0.5);
    i = i < 0 ? 0 : (i > nb - 1 ? nb - 1 : i);
    while (i + 1 < nb && start(i + 1) <= t) ++i;
    while (i > 0 && start(i) > t) --i;
    *bi = i;
    *bj = i + (t - start(i));
}

__device__ __forceinline__ float tf32_round(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

__device__ __forceinline__ void map_tile(const GtArgs& a, int64_t t, int64_t* bi, int64_t* bj) {
    if (a.rect) {
        *bi = a.row0 / GT + t / a.nb;
        *bj = t % a.nb;
    } else {
        tile_of(t, a.nb, bi, bj);
    }
}


__global__ void __launch_bounds__(kGThreads, 1)
    gram_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo, GtArgs args) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t full[kGStages], empty[kGStages], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_base_smem;
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
    const uint32_t ring = base_u32;                            // [stage][A | B]
    uint8_t* dd = base + kGStages * 2 * kSub;                  // D: [hi | lo] staged planes (sw_off layout)
    uint8_t* tt = dd + 2 * kPlane;                             // T: [hi | lo], the transposed tile

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&map_a);
        prefetch_tmap(&map_b);
        prefetch_tmap(&map_hi);
        prefetch_tmap(&map_lo);
        for (int s = 0; s < kGStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], kGEpiWarps);  // one arrival per epilogue warp
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&tmem_base_smem, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_smem;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer ----------------
            // the staged operands (a few MB) are re-read by every tile: keep them in L2 against the
            // 40 GB output stream (ncu r2: with evict_normal 4.4 GB of DRAM re-reads per n = 100k build)
            const uint64_t pol = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < args.tiles; t += gridDim.x) {
                int64_t bi, bj;
                map_tile(args, t, &bi, &bj);
                for (int ks = 0; ks < args.ksub; ++ks) {
                    mbar_wait(&empty[stage], phase ^ 1u);
                    mbar_arrive_expect_tx(&full[stage], 2 * kSub);
                    uint8_t* st = base + stage * 2 * kSub;
                    tma_load_2d(st, &map_a, &full[stage], ks * KS, static_cast<int>(bi * GT), pol);
                    tma_load_2d(st + kSub, &map_b, &full[stage], ks * KS, static_cast<int>(bj * GT), pol);
                    if (++stage == kGStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer ----------------
            constexpr uint32_t idesc = umma_idesc_tf32_f32(GT, GT);
            int stage = 0;
            uint32_t phase = 0, lt = 0;
            for (int64_t t = blockIdx.x; t < args.tiles; t += gridDim.x, ++lt) {
                const uint32_t buf = lt & 1u;
                mbar_wait(&acc_empty[buf], ((lt >> 1) & 1u) ^ 1u);
                tc_fence_after();
                for (int ks = 0; ks < args.ksub; ++ks) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a = ring + stage * 2 * kSub, b = a + kSub;
#pragma unroll
                    for (int k = 0; k < KS / 8; ++k)
                        umma_tf32(tmem + buf * GT, umma_desc_sw128(a + k * 32), umma_desc_sw128(b + k * 32), idesc,
                                  (ks > 0 || k > 0) ? 1u : 0u);
                    umma_commit(&empty[stage]);
                    if (++stage == kGStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                umma_commit(&acc_full[buf]);
            }
        }
    } else {
        // ---------------- epilogue: warps 2-17, columns [32h, 32h+32) of the tile ----------------
        // Phase A: TMEM -> K -> fp16 hi/lo in registers (overlapping the previous tile's TMA stores),
        // then staged row-major (D) and transposed (T) in shared memory in the TMA 128B-swizzled box
        // layout (conflict-free row writes and transposed 2-byte writes).
        // Phase B: one thread stores the boxes with TMA (full-line writes; the global writes drain
        // asynchronously while the next tile is computed). On a diagonal tile the lower triangle of D
        // is first replaced from T so A is exactly symmetric like the reference's mirrored Gram
        // (ops.cpp:9-20).
        const int h = (warp - 2) >> 2, q = warp & 3;
        const int row = q * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        const float l2e = 1.4426950408889634f, scale = static_cast<float>(kSplitScale);
        const int et = threadIdx.x - 2 * kWarp;  // 0..511
        uint32_t lt = 0;
        for (int64_t t = blockIdx.x; t < args.tiles; t += gridDim.x, ++lt) {
            int64_t bi, bj;
            map_tile(args, t, &bi, &bj);
            const uint32_t buf = lt & 1u;
            const bool diag = bi == bj;
            const int64_t gi = bi * GT + row;
            const float sqi = __ldg(args.sq + gi);
            mbar_wait(&acc_full[buf], (lt >> 1) & 1u);
            tc_fence_after();
            // (1) the tile's 32 columns of this thread's row -> fp16 hi/lo pairs in registers, while the
            //     TMA engine may still be reading the previous tile's staging
            uint32_t ph[16], pl[16];
#pragma unroll
            for (int c0 = 0; c0 < 32; c0 += 16) {
                float sv[16];
                tmem_ld16(tmem + lane_off + buf * GT + h * 32 + c0, sv);
                tmem_ld_wait();
                const float4* sqj4 = reinterpret_cast<const float4*>(args.sq + bj * GT + h * 32 + c0);
#pragma unroll
                for (int e = 0; e < 16; e += 4) {
                    const float4 sj = __ldg(sqj4 + e / 4);
                    const float sjv[4] = {sj.x, sj.y, sj.z, sj.w};
#pragma unroll
                    for (int u = 0; u < 4; u += 2) {
                        float kk[2];
#pragma unroll
                        for (int w = 0; w < 2; ++w) {
                            const int c = c0 + e + u + w;
                            const float arg = fminf(l2e * (2.f * sv[e + u + w] - sqi - sjv[u + w]), 0.f);
                            float kv;
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(kv) : "f"(arg));
                            if (diag && h * 32 + c == row) kv = 1.0f;  // K_ii = 1 exactly (ops.cpp:12)
                            kk[w] = kv * scale;
                        }
                        const __half2 hh = __floats2half2_rn(kk[0], kk[1]);
                        const float2 back = __half22float2(hh);
                        const __half2 ll = __floats2half2_rn(kk[0] - back.x, kk[1] - back.y);
                        ph[(c0 + e + u) / 2] = *reinterpret_cast<const uint32_t*>(&hh);
                        pl[(c0 + e + u) / 2] = *reinterpret_cast<const uint32_t*>(&ll);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);  // TMEM buffer free for the tile after next
            // (2) staging free (the previous tile's TMA stores have read it), then D rows and T columns
            if (et == 0) bulk_wait_read_all();
            asm volatile("bar.sync 1, 512;" ::: "memory");
#pragma unroll
            for (int c8 = 0; c8 < 32; c8 += 8) {
                const int cc = h * 32 + c8;
                *reinterpret_cast<uint4*>(dd + sw_off(row, cc)) =
                    make_uint4(ph[c8 / 2], ph[c8 / 2 + 1], ph[c8 / 2 + 2], ph[c8 / 2 + 3]);
                *reinterpret_cast<uint4*>(dd + kPlane + sw_off(row, cc)) =
                    make_uint4(pl[c8 / 2], pl[c8 / 2 + 1], pl[c8 / 2 + 2], pl[c8 / 2 + 3]);
            }
#pragma unroll
            for (int p = 0; p < 16; ++p) {  // transposed copy: T[c][row], T[c + 1][row]
                const int c = h * 32 + 2 * p;
                const __half2 hh = *reinterpret_cast<const __half2*>(&ph[p]);
                const __half2 ll = *reinterpret_cast<const __half2*>(&pl[p]);
                *reinterpret_cast<__half*>(tt + sw_off(c, row)) = __low2half(hh);
                *reinterpret_cast<__half*>(tt + kPlane + sw_off(c, row)) = __low2half(ll);
                *reinterpret_cast<__half*>(tt + sw_off(c + 1, row)) = __high2half(hh);
                *reinterpret_cast<__half*>(tt + kPlane + sw_off(c + 1, row)) = __high2half(ll);
            }
            if (diag && !args.rect) {  // D[i][j] <- K(j, i) = T[i][j] below the diagonal
                asm volatile("bar.sync 1, 512;" ::: "memory");
                for (int idx = et; idx < GT * GT; idx += 32 * kGEpiWarps) {
                    const int i = idx >> 7, j = idx & 127;
                    if (j < i) {
                        const uint32_t o = sw_off(i, j);
                        *reinterpret_cast<__half*>(dd + o) = *reinterpret_cast<const __half*>(tt + o);
                        *reinterpret_cast<__half*>(dd + kPlane + o) = *reinterpret_cast<const __half*>(tt + kPlane + o);
                    }
                }
            }
            fence_proxy_async_smem();  // this thread's staging writes -> visible to the TMA engine
            asm volatile("bar.sync 1, 512;" ::: "memory");
            if (et == 0) {
                const uint64_t wpol = policy_evict_first();  // A is written once here, read next pass
                const int ri = static_cast<int>(bi * GT - args.row0), ci = static_cast<int>(bj * GT);
                for (int b = 0; b < 2; ++b) {
                    tma_store_2d_hint(&map_hi, dd + b * (GT * 128), ci + 64 * b, ri, wpol);
                    tma_store_2d_hint(&map_lo, dd + kPlane + b * (GT * 128), ci + 64 * b, ri, wpol);
                }
                if (!diag && !args.rect) {  // the mirror tile (bj, bi)
                    for (int b = 0; b < 2; ++b) {
                        tma_store_2d_hint(&map_hi, tt + b * (GT * 128), static_cast<int>(bi * GT) + 64 * b,
                                          static_cast<int>(bj * GT), wpol);
                        tma_store_2d_hint(&map_lo, tt + kPlane + b * (GT * 128), static_cast<int>(bi * GT) + 64 * b,
                                          static_cast<int>(bj * GT), wpol);
                    }
                }
                bulk_commit_group();  // read completion is awaited before the next tile's staging writes
            }
        }
        if (et == 0) bulk_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 256);
}


__device__ __forceinline__ double gram_z(const GramArgs& g, double sx, double sy, int64_t i, int k) {
    return k < g.dx ? g.x[i * g.x_rs + k * g.x_cs] * sx : g.y[i * g.y_rs + (k - g.dx) * g.y_cs] * sy;
}

// z = [x·sx, y·sy] (fp64) -> tf32 hi/lo split into the operand rows A = [hi|lo|hi], B = [hi|hi|lo];
// one thread per (sample, feature) with the feature index fastest, so the row writes coalesce
__global__ void gram_tc_prep_kernel(GramArgs g, double sx, double sy, int dt, int dp, int kp, float* __restrict__ xa,
                                    float* __restrict__ xb) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= g.n * dt) return;
    const int64_t i = t / dt;
    const int k = static_cast<int>(t - i * dt);
    const double z = gram_z(g, sx, sy, i, k);
    const float hi = tf32_round(static_cast<float>(z));
    const float lo = tf32_round(static_cast<float>(z - static_cast<double>(hi)));
    float* a = xa + i * kp;
    float* b = xb + i * kp;
    a[k] = hi, a[dp + k] = lo, a[2 * dp + k] = hi;
    b[k] = hi, b[dp + k] = hi, b[2 * dp + k] = lo;
}

// sq_i = ‖z_i‖² accumulated in fp64 (one thread per sample: column-major reads coalesce)
__global__ void gram_tc_norms_kernel(GramArgs g, double sx, double sy, int dt, float* __restrict__ sq) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= g.n) return;
    double s2 = 0.0;
    for (int k = 0; k < dt; ++k) {
        const double z = gram_z(g, sx, sy, i, k);
        s2 += z * z;
    }
    sq[i] = static_cast<float>(s2);
}

}  // namespace

bool gram_tc_supported(const GramArgs& g) {
    return g.f32_compute && g.row0 % GT == 0 && g.ld % 8 == 0 && g.dx + (g.y ? g.dy : 0) <= 128;
}

namespace {
void gram_tc_shape(const GramArgs& g, int* dp, int* kp, int64_t* npad) {
    const int dt = g.dx + (g.y ? g.dy : 0);
    *dp = (dt + 7) / 8 * 8;
    *kp = (3 * *dp + KS - 1) / KS * KS;
    *npad = (g.n + GT - 1) / GT * GT;
}
}  // namespace

size_t gram_tc_scratch_bytes(const GramArgs& g) {
    int dp, kp;
    int64_t npad;
    gram_tc_shape(g, &dp, &kp, &npad);
    return (2 * static_cast<size_t>(npad) * kp + npad) * sizeof(float);  // [xa | xb] [npad][kp], sq [npad]
}

cudaError_t launch_gram_tc(const GramArgs& g, __half* hi, __half* lo, void* scratch_v, cudaStream_t stream) {
    const int dt = g.dx + (g.y ? g.dy : 0);
    int dp, kp;
    int64_t npad;
    gram_tc_shape(g, &dp, &kp, &npad);
    const size_t bytes = gram_tc_scratch_bytes(g);
    float* scratch = static_cast<float*>(scratch_v);
    cudaError_t e = cudaSuccess;
    float* xa = scratch;
    float* xb = xa + npad * kp;
    float* sq = xb + npad * kp;
    e = cudaMemsetAsync(scratch, 0, bytes, stream);
    if (e == cudaSuccess) {
        const double sx = std::sqrt(g.inv_two_sigma2_x), sy = g.y ? std::sqrt(g.inv_two_sigma2_y) : 0.0;
        const int64_t elems = g.n * dt;
        gram_tc_prep_kernel<<<static_cast<unsigned>((elems + 255) / 256), 256, 0, stream>>>(g, sx, sy, dt, dp, kp, xa,
                                                                                           xb);
        gram_tc_norms_kernel<<<static_cast<unsigned>((g.n + 255) / 256), 256, 0, stream>>>(g, sx, sy, dt, sq);
        e = cudaGetLastError();
    }
    TensorMapEncodeFn enc = tensor_map_encoder();
    if (e == cudaSuccess && !enc) e = cudaErrorInvalidValue;
    CUtensorMap ma, mb;
    for (int s = 0; s < 2 && e == cudaSuccess; ++s) {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(kp), static_cast<cuuint64_t>(npad)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(kp) * 4};
        cuuint32_t box[2] = {KS, GT};
        cuuint32_t estr[2] = {1, 1};
        if (enc(s == 0 ? &ma : &mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, s == 0 ? xa : xb, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            e = cudaErrorInvalidValue;
    }
    CUtensorMap mhi, mlo;  // outputs: fp16 [rows][ld] planes, 128-row x 64-column boxes, 128B swizzle
    for (int s = 0; s < 2 && e == cudaSuccess; ++s) {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.n), static_cast<cuuint64_t>(g.rows)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.ld) * 2};
        cuuint32_t box[2] = {64, GT};
        cuuint32_t estr[2] = {1, 1};
        if (enc(s == 0 ? &mhi : &mlo, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, s == 0 ? static_cast<void*>(hi) : lo, dims,
                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            e = cudaErrorInvalidValue;
    }
    if (e == cudaSuccess) e = ensure_smem_attr(reinterpret_cast<const void*>(gram_tc_kernel), kGSmem);
    if (e == cudaSuccess) {
        GtArgs a;
        a.nb = npad / GT;
        a.rect = (g.row0 != 0 || g.rows != g.n) ? 1 : 0;
        a.row0 = g.row0;
        a.row_end = g.row0 + g.rows;
        a.tiles = a.rect ? (g.rows + GT - 1) / GT * a.nb : a.nb * (a.nb + 1) / 2;
        a.ksub = kp / KS;
        a.n = g.n, a.ld = g.ld;
        a.sq = sq;
        a.hi = hi, a.lo = lo;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t grid = std::min<int64_t>(sms, a.tiles);
        if (grid > 0) {
            gram_tc_kernel<<<static_cast<unsigned>(grid), kGThreads, kGSmem, stream>>>(ma, mb, mhi, mlo, a);
            e = cudaGetLastError();
        }
    }
    return e;
}

}  // namespace rb
