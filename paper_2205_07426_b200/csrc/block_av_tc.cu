// Y = A · V, the hot block product (reference seam: ops::matmul_panel,
// proj/src/ops.cpp:98-107, called from proj/src/poly.cpp:155-163 and
// proj/src/hutchpp.cpp:90).
//
// B200 design:
//   * A lives in HBM as two fp16 planes (hi, lo) of A·n·2^14: the same 4 bytes
//     per entry as fp32, split so the 5th-gen tensor cores consume it directly.
//     The iterate V is stored the same way (hi, lo fp16 planes), column-major,
//     with a per-column power-of-two scale chosen by the previous pass's
//     epilogue; the fp32 recurrence state itself stays in the epilogue.
//   * Y ≈ A_hi·V_hi + A_lo·V_hi + A_hi·V_lo (the dropped lo·lo term is 2^-22
//     relative) as two tcgen05.mma (kind::f16, fp32 accumulate) per K=16 step:
//     A_hi·[V_hi | V_lo] with N' = 2N (A_hi is read from shared memory once)
//     and A_lo·V_hi into the first N accumulator columns; the drain adds the
//     two halves. The opt-in "fast" operand mode drops V_lo (A_hi·V_hi +
//     A_lo·V_hi, one V plane); see DESIGN.md for its measured error.
//   * Each CTA owns 256 rows (two UMMA M=128 tiles sharing one staged V tile),
//     so V is re-read from L2 once per 256 rows: L2 traffic 1.16x the A stream.
//   * CTA pairs (thread-block clusters of 2) own adjacent 256-row blocks and walk
//     the same k-tiles in lockstep: each CTA TMA-loads half of the V tile and
//     multicasts it to both, so V leaves L2 once per 512 rows (L2 traffic
//     ~1.08x the A stream in fast mode, ~1.16x in split mode). A stage is
//     released only when both CTAs' MMAs are done (multicast commit, count 2).
//   * Persistent stream-K schedule over pairs: one CTA per SM, each pair owning
//     one contiguous range of (row-block-pair, k-tile) iterations, so every SM
//     streams the same number of A bytes. A range that ends inside a row block
//     writes an fp32 partial to slot = 2·(pair_block + pair) + rank (unique
//     along the monotone staircase); the pass epilogue sums a row block's slots
//     in pair order (deterministic).
//   * The tensor core's fp32 accumulation is lossy over long K (measured on
//     B200: 1e-4 rms at K=1e5 with Gaussian operands), so TMEM accumulation
//     is chunked (kc k-tiles) and drained into fp32 registers with
//     round-to-nearest adds; two accumulator sets double-buffer the drain.
//   * Warp roles: warp 0 = TMA producer, warp 1 = MMA issuer (+TMEM owner),
//     warps 2..9 = TMEM drain (4 per M=128 tile) and partial writers.
#include <algorithm>
#include <cstdio>
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace rb {

namespace {

constexpr int BM = 256;  // rows per CTA (two UMMA M=128 tiles)
constexpr int TM = 128;  // UMMA M
constexpr int BK = 32;   // K per stage: one 64-byte swizzle row of fp16
constexpr int kThreads = 320;
#ifndef RB_SMEM_BUDGET_KB
#define RB_SMEM_BUDGET_KB 220
#endif
constexpr int kSmemBudget = RB_SMEM_BUDGET_KB;  // KB of dynamic smem for the TMA ring

template <int NPAD, bool VSPLIT>
struct TcCfg {
    static constexpr int kAPlane = BM * BK * 2;  // one plane, both tiles
    static constexpr int kATile = TM * BK * 2;   // one plane, one tile
    static constexpr int kVPlane = NPAD * BK * 2;
    static constexpr int kVBytes = (VSPLIT ? 2 : 1) * kVPlane;
    static constexpr int kStageBytes = 2 * kAPlane + kVBytes;
    static constexpr int kStagesRaw = (kSmemBudget * 1024) / kStageBytes;
    static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
    static constexpr int kAccCols = (VSPLIT ? 2 : 1) * NPAD;              // accumulator width per tile
    static constexpr int kBufs = (2 * 2 * kAccCols <= 512) ? 2 : 1;         // double-buffer the drain if it fits
    static constexpr int kTmemNeed = kBufs * 2 * kAccCols;
    static constexpr int kTmemCols = (kTmemNeed <= 32) ? 32 : (kTmemNeed <= 64) ? 64 : (kTmemNeed <= 128) ? 128
                                                         : (kTmemNeed <= 256) ? 256 : 512;
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024;
    static_assert(NPAD % 16 == 0 && NPAD >= 16 && NPAD <= 128, "NPAD must be a multiple of 16 in [16,128]");
    static_assert(kStages >= 3, "need a deep enough TMA ring");
    static_assert(kVPlane % 512 == 0, "64-byte swizzle atoms are 512 bytes");
};

struct TcArgs {
    int64_t total_iters;  // row_blocks * k_tiles
    int k_tiles;          // k tiles per row block
    int kt_chunk;         // k tiles per V chunk (rpr / BK)
    int kc;               // k tiles per TMEM chunk
    float* partial;       // [slots][NPAD][BM]
    int a_policy;         // 0: evict_first for the A stream, 1: evict_normal
};

// UMMA shared-memory descriptor: K-major, 64-byte swizzle (rows of 64 bytes, 8-row atoms of 512 bytes).
__device__ __forceinline__ uint64_t desc_sw64(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);  // start address
    d |= static_cast<uint64_t>(1) << 16;                      // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(512 >> 4) << 32;               // SBO: stride between 8-row atoms
    d |= static_cast<uint64_t>(1) << 46;                      // descriptor version (sm100)
    d |= static_cast<uint64_t>(4) << 61;                      // SWIZZLE_64B
    return d;
}

template <int NPAD, bool VSPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    block_av_tc_kernel(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                       const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_vlo,
                       TcArgs args) {
    using C = TcCfg<NPAD, VSPLIT>;
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t full_bar[C::kStages];
    __shared__ __align__(8) uint64_t empty_bar[C::kStages];
    __shared__ __align__(8) uint64_t tmem_full_bar[2];
    __shared__ __align__(8) uint64_t tmem_empty_bar[2];
    __shared__ uint32_t tmem_base_smem;

    const int warp = threadIdx.x / kWarp;
    const int lane = threadIdx.x % kWarp;
    const int G = gridDim.x / 2;  // CTA pairs
    const int pair = blockIdx.x / 2;
    const int rank = static_cast<int>(cluster_ctarank());

    const uint32_t smem_base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* smem_base = smem_raw + (smem_base_u32 - smem_u32(smem_raw));

    // iterations are (row-block-pair, k-tile); this CTA serves row block 2*rp + rank
    const int64_t it_begin = (args.total_iters * pair) / G;
    const int64_t it_end = (args.total_iters * (pair + 1)) / G;
    const int KT = args.k_tiles;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&map_ahi);
        prefetch_tmap(&map_alo);
        prefetch_tmap(&map_v);
        if (VSPLIT) prefetch_tmap(&map_vlo);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 2);  // released by both CTAs' MMAs
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tmem_full_bar[b], 1);
            mbar_init(&tmem_empty_bar[b], 8 * kWarp);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&tmem_base_smem, C::kTmemCols);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // peer barriers are initialised before any multicast lands
    tc_fence_after();
    const uint32_t tmem_base = tmem_base_smem;

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            const uint64_t pol_stream = args.a_policy ? policy_evict_normal() : policy_evict_first();
            const uint64_t pol_keep = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t it = it_begin; it < it_end; ++it) {
                const int rp = static_cast<int>(it / KT);
                const int k = static_cast<int>(it - static_cast<int64_t>(rp) * KT);
                const int r = 2 * rp + rank;
                mbar_wait(&empty_bar[stage], phase ^ 1u);  // both CTAs released this stage
                uint8_t* st = smem_base + stage * C::kStageBytes;
                mbar_arrive_expect_tx(&full_bar[stage], C::kStageBytes);
                tma_load_2d(st, &map_ahi, &full_bar[stage], k * BK, r * BM, pol_stream);
                tma_load_2d(st + C::kAPlane, &map_alo, &full_bar[stage], k * BK, r * BM, pol_stream);
                const int vz = k / args.kt_chunk;               // V chunk (shard) holding these K rows
                const int vx = (k - vz * args.kt_chunk) * BK;   // offset inside the chunk
                if (VSPLIT) {  // rank 0 multicasts V_hi, rank 1 V_lo
                    tma_load_3d_mc(st + 2 * C::kAPlane + rank * C::kVPlane, rank ? &map_vlo : &map_v,
                                   &full_bar[stage], vx, 0, vz, 0x3, pol_keep);
                } else {  // each rank multicasts half of the V rows
                    tma_load_3d_mc(st + 2 * C::kAPlane + rank * (C::kVPlane / 2), &map_v, &full_bar[stage], vx,
                                   rank * (NPAD / 2), vz, 0x3, pol_keep);
                }
                if (++stage == C::kStages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc_f16_f32(TM, NPAD);
            constexpr uint32_t idesc2 = umma_idesc_f16_f32(TM, VSPLIT ? 2 * NPAD : NPAD);
            int stage = 0;
            uint32_t phase = 0;
            uint32_t chunk = 0;
            int64_t it = it_begin;
            while (it < it_end) {
                const int64_t rp = it / KT;
                const int64_t seg_end = min(it_end, (rp + 1) * KT);
                while (it < seg_end) {
                    const int64_t cend = min(seg_end, it + args.kc);
                    const uint32_t buf = chunk % C::kBufs;
                    const uint32_t use = chunk / C::kBufs;
                    mbar_wait(&tmem_empty_bar[buf], (use & 1u) ^ 1u);
                    tc_fence_after();
                    const uint32_t d0 = tmem_base + buf * (2 * C::kAccCols);
                    const int64_t cstart = it;
                    for (; it < cend; ++it) {
                        mbar_wait(&full_bar[stage], phase);
                        tc_fence_after();
                        const uint32_t st = smem_base_u32 + stage * C::kStageBytes;
                        const uint32_t v = st + 2 * C::kAPlane;
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk) {
                            const uint32_t off = kk * 32;  // 16 fp16 along K = 32 bytes
                            const uint64_t dv = desc_sw64(v + off);
#pragma unroll
                            for (int t = 0; t < BM / TM; ++t) {
                                const uint32_t acc = (it > cstart || kk > 0) ? 1u : 0u;
                                const uint32_t d = d0 + t * C::kAccCols;
                                // A_hi x [V_hi | V_lo]: the two V planes are adjacent in smem (N' = 2N rows)
                                umma_f16(d, desc_sw64(st + t * C::kATile + off), dv, VSPLIT ? idesc2 : idesc, acc);
                                umma_f16(d, desc_sw64(st + C::kAPlane + t * C::kATile + off), dv, idesc, 1u);
                            }
                        }
                        umma_commit_mc(&empty_bar[stage], 0x3);  // release the stage in both CTAs
                        if (++stage == C::kStages) {
                            stage = 0;
                            phase ^= 1u;
                        }
                    }
                    umma_commit(&tmem_full_bar[buf]);
                    ++chunk;
                }
            }
        }
    } else {
        // ---------------- TMEM drain (warps 2..9: tile (warp-2)/4, lane quarter warp%4) ----------------
        const int tile = (warp - 2) / 4;
        const int quarter = warp & 3;  // TMEM lane quarter this warp may access
        const int row_local = tile * TM + quarter * 32 + lane;
        const uint32_t lane_base = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + tile * C::kAccCols;
        float acc[NPAD];
#pragma unroll
        for (int j = 0; j < NPAD; ++j) acc[j] = 0.f;
        uint32_t chunk = 0;
        int64_t it = it_begin;
        while (it < it_end) {
            const int64_t rp = it / KT;
            const int64_t seg_end = min(it_end, (rp + 1) * KT);
            while (it < seg_end) {
                const int64_t cend = min(seg_end, it + args.kc);
                const uint32_t buf = chunk % C::kBufs;
                const uint32_t use = chunk / C::kBufs;
                mbar_wait(&tmem_full_bar[buf], use & 1u);
                tc_fence_after();
                const uint32_t t0 = lane_base + buf * (2 * C::kAccCols);
#pragma unroll
                for (int j0 = 0; j0 < NPAD; j0 += 16) {
                    float m[16];
                    tmem_ld16(t0 + j0, m);
                    if (VSPLIT) {
                        float c[16];
                        tmem_ld16(t0 + NPAD + j0, c);  // A_hi·V_lo half
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; ++i) acc[j0 + i] += m[i] + c[i];
                    } else {
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 16; ++i) acc[j0 + i] += m[i];
                    }
                }
                tc_fence_before();
                mbar_arrive(&tmem_empty_bar[buf]);
                it = cend;
                ++chunk;
            }
            // segment finished: publish the partial for row block 2*rp + rank
            const int64_t slot = 2 * (rp + pair) + rank;
            float* dst = args.partial + (slot * NPAD) * BM + row_local;
#pragma unroll
            for (int j = 0; j < NPAD; ++j) {
                dst[j * BM] = acc[j];
                acc[j] = 0.f;
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // no CTA leaves while its peer may still multicast into it
    if (warp == 1) tmem_dealloc(tmem_base, C::kTmemCols);
}

bool make_map_f16(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_bytes,
                  uint32_t box_inner, uint32_t box_outer,
                  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
    TensorMapEncodeFn enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {pitch_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, promo,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_map_v3(CUtensorMap* m, const void* base, uint64_t rpr, uint64_t cols, uint64_t world, uint32_t box_rows) {
    TensorMapEncodeFn enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {rpr, cols, world};
    cuuint64_t strides[2] = {rpr * 2ull, rpr * cols * 2ull};
    cuuint32_t box[3] = {BK, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int NPAD, bool VSPLIT>
cudaError_t launch_tc(const SplitMatrixView& a, const SplitPanelView& v, const StreamKPlan& plan, float* partial,
                      cudaStream_t stream) {
    using C = TcCfg<NPAD, VSPLIT>;
    CUtensorMap m_ahi, m_alo, m_v, m_vlo;
    // split: one CTA of the pair loads V_hi, the other V_lo; fast: each loads half of V's rows
    const uint32_t vbox = VSPLIT ? NPAD : NPAD / 2;
    // measured on B200 (r1): 256-byte L2 promotion + evict_first for the A stream beats no/128-byte
    // promotion and evict_normal by 1-2%
    const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    bool ok = make_map_f16(&m_ahi, a.hi, a.cols, a.rows, a.ld * 2ull, BK, BM, promo) &&
              make_map_f16(&m_alo, a.lo, a.cols, a.rows, a.ld * 2ull, BK, BM, promo) &&
              make_map_v3(&m_v, v.v, v.rpr, v.cols, v.world, vbox) &&
              make_map_v3(&m_vlo, VSPLIT ? v.vlo : v.v, v.rpr, v.cols, v.world, vbox);
    if (v.rpr % BK != 0) return cudaErrorInvalidValue;
    if (!ok) return cudaErrorInvalidValue;
    if (cudaError_t e =
            ensure_smem_attr(reinterpret_cast<const void*>(block_av_tc_kernel<NPAD, VSPLIT>), C::kSmemBytes);
        e != cudaSuccess)
        return e;
    TcArgs args;
    args.total_iters = plan.total_iters;
    args.k_tiles = plan.k_tiles;
    args.kt_chunk = static_cast<int>(v.rpr / BK);
    args.kc = plan.kc;
    args.partial = partial;
    args.a_policy = 0;
    block_av_tc_kernel<NPAD, VSPLIT><<<2 * plan.grid, kThreads, C::kSmemBytes, stream>>>(m_ahi, m_alo, m_v, m_vlo,
                                                                                       args);
    return cudaGetLastError();
}

}  // namespace

int tc_block_rows() { return BM; }
int tc_block_k() { return BK; }

StreamKPlan make_streamk_plan(int64_t rows, int64_t cols, int grid, int kc) {
    // grid = CTAs (rounded down to pairs); iterations are (row-block-pair, k-tile)
    StreamKPlan p;
    p.row_blocks = static_cast<int>((rows + BM - 1) / BM);
    p.k_tiles = static_cast<int>((cols + BK - 1) / BK);
    const int64_t pair_blocks = (p.row_blocks + 1) / 2;
    p.total_iters = pair_blocks * p.k_tiles;
    int pairs = std::max(1, grid / 2);
    if (p.total_iters < pairs) pairs = static_cast<int>(p.total_iters > 0 ? p.total_iters : 1);
    p.grid = pairs;  // stream-K participants (pairs)
    p.cluster = 2;
    p.kc = kc;
    p.slots = static_cast<int>(2 * (pair_blocks + pairs));
    p.rows_per_block = BM;
    return p;
}

int tc_npad(int cols) { return ((cols + 15) / 16) * 16; }

cudaError_t launch_block_av_tc(const SplitMatrixView& a, const SplitPanelView& v, const StreamKPlan& plan,
                               float* partial, cudaStream_t stream) {
    const int npad = tc_npad(v.cols);
#define RB_TC_CASE(N)                                                                              \
    case N:                                                                                        \
        return v.vlo ? launch_tc<N, true>(a, v, plan, partial, stream)                             \
                     : launch_tc<N, false>(a, v, plan, partial, stream);
    switch (npad) {
        RB_TC_CASE(16)
        RB_TC_CASE(32)
        RB_TC_CASE(48)
        RB_TC_CASE(64)
        RB_TC_CASE(80)
        RB_TC_CASE(96)
        RB_TC_CASE(112)
        RB_TC_CASE(128)
        default: return cudaErrorInvalidValue;
    }
#undef RB_TC_CASE
}

}  // namespace rb
