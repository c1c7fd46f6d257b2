// Matrix-free block product (config 5; SURVEY §8(a5) "matrix-free variant", §7 step 6):
//   Y_i = Σ_j K(x_i, x_j) · V_j,   K = exp(−(|x_i|² + |x_j|² − 2 x_i·x_j) / (2σ²)),  K_ii = 1,
// with the kernel entries recomputed from bf16 X on the tensor cores and never stored
// (the reference materialises A: proj/src/kernel.cpp:35-72 + ops.cpp:98-107).
//
// FlashAttention-shaped, without the softmax bookkeeping (kernel values are already in (0, 1]):
//   S  = X_i · X_jᵀ            tcgen05.mma kind::f16 (bf16 in, fp32 accumulate) → TMEM
//   P  = exp2(2c·S − b_i − b_j) exp warps: TMEM → registers → MUFU ex2 → fp16 → SW128 smem
//   O += P · V_j               tcgen05.mma kind::f16 (fp16 in, fp32 accumulate) → TMEM
// where b = c·|x|², c = log2(e)/(2σ²). One CTA owns 128 rows (UMMA M); j-blocks of 128.
// Warp roles: 0 TMA (X_i once per row block, X_j + V_j ring), 1 MMA issuer, 2-5 exp,
// 6-9 O drain (fp32 register accumulation every kc j-blocks — the tensor core's long-K
// accumulation is lossy, see block_av_tc.cu). S and O are double-buffered in TMEM, P in smem.
// Persistent stream-K over (row block, j-block) with the same partial-slot protocol and pass
// epilogue as the materialised path.
#include <algorithm>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace rb {

namespace {

constexpr int MB = 128;  // rows per CTA (UMMA M)
constexpr int JB = 128;  // j-block: S tile N and P·V K
constexpr int kMfThreads = 320;
constexpr int kBiasBytes = JB * 4;

template <int DP, int NPAD>
struct MfCfg {
    static constexpr int kXTile = MB * DP * 2;      // X tile, bf16, [128][DP] as DP/64 SW128 sub-tiles
    static constexpr int kXSub = MB * 64 * 2;       // one 64-feature sub-tile (16 KB)
    static constexpr int kVTile = NPAD * JB * 2;    // V_j tile, fp16, [NPAD][128] as two SW128 sub-tiles
    static constexpr int kVSub = NPAD * 64 * 2;
    static constexpr int kPTile = MB * JB * 2;      // P tile, fp16, [128][128] as two SW128 sub-tiles
    static constexpr int kStage = kXTile + kVTile;  // X_j + V_j (1024-aligned); the j-block bias rides in a ring
    static constexpr int kStagesRaw = (226 * 1024 - kXTile - 2 * kPTile - 1024) / (kStage + kBiasBytes);
    static constexpr int kStages = kStagesRaw > 4 ? 4 : kStagesRaw;
    static constexpr int kSmem = kXTile + 2 * kPTile + kStages * (kStage + kBiasBytes) + 1024;
    static constexpr int kOCol = 2 * JB;  // O buffers after the two S buffers
    static constexpr int kHalf = NPAD / 2;  // O columns drained by each exp warpgroup
    static_assert(DP == 64 || DP == 128, "feature dimension is padded to 64 or 128");
    static_assert(NPAD % 16 == 0 && NPAD <= 128, "NPAD must be a multiple of 16 in [16,128]");
    static_assert(kStages >= 2, "need a double-buffered X_j/V_j ring");
    static_assert(kOCol + 2 * NPAD <= 512, "TMEM budget");
};

struct MfArgs {
    int64_t total_iters;  // row_blocks * j_blocks
    int j_blocks;
    int kc;               // j-blocks per O accumulation chunk
    int64_t row0;         // first global row of this rank
    int64_t n;            // samples
    int kt_chunk;         // j-blocks per V chunk (rpr / 128)
    float c2;             // 2c = log2(e)/σ²
    const float* nbias;   // −b = −c·|x|², [n_pad], zero padded
    float* partial;       // [slots][NPAD][128]
};

__device__ __forceinline__ uint64_t desc_sw128_k(uint32_t addr) { return umma_desc_sw128(addr); }

__device__ __forceinline__ uint32_t pack_f16x2_clamp1(float lo, float hi) {
    // fp16 pair, clamped to <= 1 (K <= 1; guards exp2 of a rounding-positive argument)
    uint32_t r;
    asm("{\n\t.reg .b32 one;\n\tmov.b32 one, 0x3C003C00;\n\tcvt.rn.f16x2.f32 %0, %1, %2;\n\tmin.f16x2 %0, %0, one;\n\t}"
        : "=r"(r)
        : "f"(hi), "f"(lo));
    return r;
}

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

// 8 kernel values of one row: p = exp2(2c·s − b_i − b_j), packed to fp16 (16 bytes of P)
template <bool DIAG>
__device__ __forceinline__ void exp8(const float* sv, float2 c2v, float2 nbv, float4 b0, float4 b1, int col0,
                                     int row, uint32_t* pk) {
    const float bj[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        float2 a = __ffma2_rn(make_float2(sv[2 * e], sv[2 * e + 1]), c2v, nbv);
        a = __fadd2_rn(a, make_float2(bj[2 * e], bj[2 * e + 1]));
        float p0 = ex2(a.x), p1 = ex2(a.y);
        if (DIAG) {  // K_ii = 1 exactly (proj/src/ops.cpp:12)
            if (col0 + 2 * e == row) p0 = 1.0f;
            if (col0 + 2 * e + 1 == row) p1 = 1.0f;
        }
        pk[e] = pack_f16x2_clamp1(p0, p1);
    }
}

template <int DP, int NPAD>
__global__ void __launch_bounds__(kMfThreads, 1)
    block_av_mf_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_v,
                       MfArgs args) {
    using C = MfCfg<DP, NPAD>;
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t xi_full, xi_empty;
    __shared__ __align__(8) uint64_t st_full[C::kStages], st_empty[C::kStages];
    __shared__ __align__(8) uint64_t s_full[2], s_empty[2], p_full[2], p_empty[2], o_full[2], o_empty[2];
    __shared__ uint32_t tmem_base_smem;

    const int warp = threadIdx.x / kWarp;
    const int lane = threadIdx.x % kWarp;
    const int G = gridDim.x, cta = blockIdx.x;
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
    const uint32_t xi_smem = base_u32;
    const uint32_t p_smem = xi_smem + C::kXTile;                // two P buffers
    const uint32_t st_smem = p_smem + 2 * C::kPTile;            // ring of X_j + V_j
    const uint32_t bias_smem = st_smem + C::kStages * C::kStage;  // ring of −b_j (128 floats per stage)
    const int64_t it_begin = (args.total_iters * cta) / G;
    const int64_t it_end = (args.total_iters * (cta + 1)) / G;
    const int JBn = args.j_blocks;
    constexpr uint32_t kExpThreads = 8 * kWarp;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&map_x);
        prefetch_tmap(&map_v);
        mbar_init(&xi_full, 1);
        mbar_init(&xi_empty, 1);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&st_full[s], 1);
            mbar_init(&st_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&s_empty[b], kExpThreads);
            mbar_init(&p_full[b], kExpThreads);
            mbar_init(&p_empty[b], 1);
            mbar_init(&o_full[b], 1);
            mbar_init(&o_empty[b], kExpThreads);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&tmem_base_smem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_smem;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();  // X, V and b are re-read by every row block
            int stage = 0;
            uint32_t phase = 0, seg = 0;
            int64_t it = it_begin;
            while (it < it_end) {
                const int64_t r = it / JBn;
                const int64_t seg_end = min(it_end, (r + 1) * JBn);
                mbar_wait(&xi_empty, (seg & 1u) ^ 1u);
                mbar_arrive_expect_tx(&xi_full, C::kXTile);
                for (int h = 0; h < DP / 64; ++h)
                    tma_load_2d(base + h * C::kXSub, &map_x, &xi_full, h * 64, static_cast<int>(args.row0 + r * MB),
                                pol);
                for (; it < seg_end; ++it) {
                    const int jb = static_cast<int>(it - r * JBn);
                    mbar_wait(&st_empty[stage], phase ^ 1u);
                    uint8_t* st = base + (st_smem - base_u32) + stage * C::kStage;
                    mbar_arrive_expect_tx(&st_full[stage], C::kStage + kBiasBytes);
                    for (int h = 0; h < DP / 64; ++h)
                        tma_load_2d(st + h * C::kXSub, &map_x, &st_full[stage], h * 64, jb * JB, pol);
                    const int vz = jb / args.kt_chunk, vx = (jb - vz * args.kt_chunk) * JB;
                    for (int h = 0; h < 2; ++h)
                        tma_load_3d(st + C::kXTile + h * C::kVSub, &map_v, &st_full[stage], vx + h * 64, 0, vz, pol);
                    bulk_load_1d(base + (bias_smem - base_u32) + stage * kBiasBytes, args.nbias + jb * JB,
                                 kBiasBytes, &st_full[stage], pol);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                ++seg;
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            constexpr uint32_t idesc_s = umma_idesc_bf16_f32(MB, JB);
            constexpr uint32_t idesc_o = umma_idesc_f16_f32(MB, NPAD);
            int stage = 0;
            uint32_t phase = 0, seg = 0, jc = 0, chunk = 0, in_chunk = 0;
            int prev_stage = -1;
            auto pv = [&](int st_idx, uint32_t jprev, bool last_of_segment) {
                const uint32_t pb = jprev & 1u;
                mbar_wait(&p_full[pb], (jprev >> 1) & 1u);
                tc_fence_after();
                const uint32_t ob = chunk & 1u;
                if (in_chunk == 0) {
                    mbar_wait(&o_empty[ob], ((chunk >> 1) & 1u) ^ 1u);
                    tc_fence_after();
                }
                const uint32_t d = tmem + C::kOCol + ob * NPAD;
                const uint32_t pa = p_smem + pb * C::kPTile;
                const uint32_t vb = st_smem + st_idx * C::kStage + C::kXTile;
#pragma unroll
                for (int k = 0; k < JB / 16; ++k) {
                    const uint32_t off = (k & 3) * 32;  // 16 K-elements = 32 bytes inside a 128-byte row
                    umma_f16(d, desc_sw128_k(pa + (k >> 2) * (MB * 128) + off),
                             desc_sw128_k(vb + (k >> 2) * C::kVSub + off), idesc_o, (in_chunk > 0 || k > 0) ? 1u : 0u);
                }
                umma_commit(&p_empty[pb]);
                umma_commit(&st_empty[st_idx]);
                ++in_chunk;
                if (in_chunk == static_cast<uint32_t>(args.kc) || last_of_segment) {
                    umma_commit(&o_full[ob]);
                    ++chunk;
                    in_chunk = 0;
                }
            };
            int64_t it = it_begin;
            while (it < it_end) {
                const int64_t r = it / JBn;
                const int64_t seg_end = min(it_end, (r + 1) * JBn);
                mbar_wait(&xi_full, seg & 1u);
                tc_fence_after();
                for (; it < seg_end; ++it) {
                    mbar_wait(&st_full[stage], phase);
                    const uint32_t sb = jc & 1u;
                    mbar_wait(&s_empty[sb], ((jc >> 1) & 1u) ^ 1u);
                    tc_fence_after();
                    const uint32_t xj = st_smem + stage * C::kStage;
#pragma unroll
                    for (int k = 0; k < DP / 16; ++k) {
                        const uint32_t off = (k >> 2) * C::kXSub + (k & 3) * 32;
                        umma_f16(tmem + sb * JB, desc_sw128_k(xi_smem + off), desc_sw128_k(xj + off), idesc_s,
                                 k > 0 ? 1u : 0u);
                    }
                    umma_commit(&s_full[sb]);
                    if (it + 1 == seg_end) umma_commit(&xi_empty);  // X_i free once the segment's S MMAs finish
                    if (prev_stage >= 0) pv(prev_stage, jc - 1, false);
                    prev_stage = stage;
                    ++jc;
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                pv(prev_stage, jc - 1, true);  // last P·V of the segment closes the O chunk
                prev_stage = -1;
                ++seg;
            }
        }
    } else {
        // ---------------- exp + O drain: two warpgroups, columns [64h, 64h+64) of S / P ----------------
        // Each thread owns one row (its TMEM lane) and half of the j-block's columns; it also drains
        // half of the O columns into fp32 registers (lazily, one j-block after the chunk closes, so
        // the exp work of the next j-block overlaps the last P·V of the chunk).
        const int h = (warp - 2) >> 2;
        const int q = warp & 3;  // TMEM lane quarter
        const int row = q * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        const float2 c2v = make_float2(args.c2, args.c2);
        float acc[C::kHalf];
#pragma unroll
        for (int j = 0; j < C::kHalf; ++j) acc[j] = 0.f;
        auto drain = [&](uint32_t c) {
            const uint32_t ob = c & 1u;
            mbar_wait(&o_full[ob], (c >> 1) & 1u);
            tc_fence_after();
            const uint32_t t0 = tmem + lane_off + C::kOCol + ob * NPAD + h * C::kHalf;
#pragma unroll
            for (int j0 = 0; j0 + 16 <= C::kHalf; j0 += 16) {
                float m[16];
                tmem_ld16(t0 + j0, m);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[j0 + i] += m[i];
            }
            if constexpr (C::kHalf % 16 != 0) {
                float m[8];
                tmem_ld8(t0 + C::kHalf - 8, m);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[C::kHalf - 8 + i] += m[i];
            }
            tc_fence_before();
            mbar_arrive(&o_empty[ob]);
        };
        uint32_t jc = 0, chunk = 0, phase = 0;
        int stage = 0;
        int64_t it = it_begin;
        while (it < it_end) {
            const int64_t r = it / JBn;
            const int64_t seg_end = min(it_end, (r + 1) * JBn);
            const int64_t g0 = args.row0 + r * MB;  // first global row of the block (a multiple of 128)
            const float2 nbv = make_float2(__ldg(args.nbias + g0 + row), __ldg(args.nbias + g0 + row));
            const int64_t diag_jb = g0 / JB;
            uint32_t in_chunk = 0, pend = 0;
            bool pending = false;
            for (; it < seg_end; ++it, ++jc) {
                const int64_t jb = it - r * JBn;
                const uint32_t sb = jc & 1u;
                mbar_wait(&s_full[sb], (jc >> 1) & 1u);
                tc_fence_after();
                float sv[64];
                tmem_ld32(tmem + lane_off + sb * JB + h * 64, sv);
                tmem_ld32(tmem + lane_off + sb * JB + h * 64 + 32, sv + 32);
                tmem_ld_wait();
                tc_fence_before();
                mbar_arrive(&s_empty[sb]);  // S buffer free for the MMA of j+2
                mbar_wait(&st_full[stage], phase);  // −b_j landed (already implied by s_full)
                mbar_wait(&p_empty[sb], ((jc >> 1) & 1u) ^ 1u);
                const uint32_t bsm = bias_smem + stage * kBiasBytes + h * 64 * 4;
                const uint32_t prow = p_smem + sb * C::kPTile + h * (MB * 128) + row * 128;
                const bool diag = jb == diag_jb;
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const float4 b0 = ld_shared_f4(bsm + g * 32);
                    const float4 b1 = ld_shared_f4(bsm + g * 32 + 16);
                    uint32_t pk[4];
                    if (diag)
                        exp8<true>(sv + 8 * g, c2v, nbv, b0, b1, h * 64 + 8 * g, row, pk);
                    else
                        exp8<false>(sv + 8 * g, c2v, nbv, b0, b1, h * 64 + 8 * g, row, pk);
                    st_shared_v4(prow + ((g ^ (row & 7)) << 4), pk[0], pk[1], pk[2], pk[3]);
                }
                fence_proxy_async_smem();  // P visible to the tensor core
                mbar_arrive(&p_full[sb]);
                if (++stage == C::kStages) {
                    stage = 0;
                    phase ^= 1u;
                }
                if (pending) {
                    drain(pend);
                    pending = false;
                }
                if (++in_chunk == static_cast<uint32_t>(args.kc) || it + 1 == seg_end) {
                    if (it + 1 == seg_end) {
                        drain(chunk);
                    } else {
                        pending = true;
                        pend = chunk;
                    }
                    ++chunk;
                    in_chunk = 0;
                }
            }
            const int64_t slot = r + cta;
            float* dst = args.partial + (slot * NPAD + h * C::kHalf) * MB + row;
#pragma unroll
            for (int j = 0; j < C::kHalf; ++j) {
                dst[j * MB] = acc[j];
                acc[j] = 0.f;
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

template <int DP, int NPAD>
cudaError_t launch_mf(const MfMatrixView& a, const SplitPanelView& v, const StreamKPlan& plan, float* partial,
                      cudaStream_t stream) {
    using C = MfCfg<DP, NPAD>;
    EncodeFn enc = encoder();
    if (!enc) return cudaErrorInvalidValue;
    CUtensorMap mx, mv;
    {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.dp), static_cast<cuuint64_t>(a.n)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.dp) * 2};
        cuuint32_t box[2] = {64, MB};
        cuuint32_t estr[2] = {1, 1};
        if (enc(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(a.x), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    {
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(v.rpr), static_cast<cuuint64_t>(v.cols),
                              static_cast<cuuint64_t>(v.world)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(v.rpr) * 2, static_cast<cuuint64_t>(v.rpr) * v.cols * 2};
        cuuint32_t box[3] = {64, NPAD, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        if (enc(&mv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<__half*>(v.v), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    if (v.rpr % JB != 0) return cudaErrorInvalidValue;
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(block_av_mf_kernel<DP, NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    MfArgs args;
    args.total_iters = plan.total_iters;
    args.j_blocks = plan.k_tiles;
    args.kc = plan.kc;
    args.row0 = a.row0;
    args.n = a.n;
    args.kt_chunk = static_cast<int>(v.rpr / JB);
    args.c2 = static_cast<float>(a.c2);
    args.nbias = a.bias;
    args.partial = partial;
    block_av_mf_kernel<DP, NPAD><<<plan.grid, kMfThreads, C::kSmem, stream>>>(mx, mv, args);
    return cudaGetLastError();
}

__global__ void mf_prepare_kernel(const double* __restrict__ x, int64_t n, int d, int64_t rs, int64_t cs, int dp,
                                  double c, __nv_bfloat16* __restrict__ xb, float* __restrict__ bias) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float sq = 0.f;
    for (int k = 0; k < dp; ++k) {
        const __nv_bfloat16 v = __float2bfloat16_rn(k < d ? static_cast<float>(x[i * rs + k * cs]) : 0.f);
        xb[i * dp + k] = v;
        const float f = __bfloat162float(v);
        sq = fmaf(f, f, sq);
    }
    bias[i] = static_cast<float>(-c * static_cast<double>(sq));  // −b
}

}  // namespace

StreamKPlan make_mf_plan(int64_t rows, int64_t n, int grid, int kc) {
    StreamKPlan p;
    p.row_blocks = static_cast<int>((rows + MB - 1) / MB);
    p.k_tiles = static_cast<int>((n + JB - 1) / JB);  // j-blocks
    p.total_iters = static_cast<int64_t>(p.row_blocks) * p.k_tiles;
    p.grid = grid;
    if (p.total_iters < grid) p.grid = static_cast<int>(p.total_iters > 0 ? p.total_iters : 1);
    p.kc = kc;
    p.slots = p.row_blocks + p.grid;
    p.rows_per_block = MB;
    p.cluster = 1;
    return p;
}

cudaError_t launch_block_av_mf(const MfMatrixView& a, const SplitPanelView& v, const StreamKPlan& plan,
                               float* partial, cudaStream_t stream) {
    const int npad = tc_npad(v.cols);
#define RB_MF_CASE(N)                                                                          \
    case N:                                                                                    \
        return a.dp == 64 ? launch_mf<64, N>(a, v, plan, partial, stream)                      \
                          : launch_mf<128, N>(a, v, plan, partial, stream);
    switch (npad) {
        RB_MF_CASE(16)
        RB_MF_CASE(32)
        RB_MF_CASE(48)
        RB_MF_CASE(64)
        RB_MF_CASE(80)
        RB_MF_CASE(96)
        RB_MF_CASE(112)
        RB_MF_CASE(128)
        default: return cudaErrorInvalidValue;
    }
#undef RB_MF_CASE
}

cudaError_t launch_mf_prepare(const double* x, int64_t n, int d, int64_t rs, int64_t cs, int dp, double c,
                              __nv_bfloat16* xb, float* bias, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    mf_prepare_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(x, n, d, rs, cs, dp, c, xb, bias);
    return cudaGetLastError();
}

}  // namespace rb
