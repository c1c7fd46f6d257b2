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
#include <cmath>
#include <cstdio>
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace rb {

namespace {

constexpr int BM = 256;  // rows per CTA (two UMMA M=128 tiles)
constexpr int TM = 128;  // UMMA M
#ifndef RB_TC_BK
#define RB_TC_BK 32
#endif
constexpr int BK = RB_TC_BK;  // K per stage: one 64-byte (32) or 128-byte (64) swizzle row of fp16
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
    static_assert(kStages >= (BK == 32 ? 3 : 2), "need a deep enough TMA ring");
    static_assert(kVPlane % (BK * 16) == 0, "swizzle atoms are 8 rows");
};

struct TcArgs {
    int64_t total_iters;  // row_blocks * k_tiles
    int k_tiles;          // k tiles per row block (of this launch's K window)
    int k_off, k_total;   // K window: tile k of the launch is global tile (k_off + k) mod k_total
    int kt_chunk;         // k tiles per V chunk (rpr / BK)
    int64_t g_rows;       // grouped stacked matrices: operand offset of row block r's group (0: none)
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

// descriptor of the single-matrix kernel's K-major tiles (64- or 128-byte swizzle rows)
__device__ __forceinline__ uint64_t desc_tc(uint32_t smem_addr) {
    return BK == 64 ? umma_desc_sw128(smem_addr) : desc_sw64(smem_addr);
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
                const int kg = k + args.k_off < args.k_total ? k + args.k_off : k + args.k_off - args.k_total;
                mbar_wait(&empty_bar[stage], phase ^ 1u);  // both CTAs released this stage
                uint8_t* st = smem_base + stage * C::kStageBytes;
                mbar_arrive_expect_tx(&full_bar[stage], C::kStageBytes);
                tma_load_2d(st, &map_ahi, &full_bar[stage], kg * BK, r * BM, pol_stream);
                tma_load_2d(st + C::kAPlane, &map_alo, &full_bar[stage], kg * BK, r * BM, pol_stream);
                const int vz = kg / args.kt_chunk;              // V chunk (shard) holding these K rows
                int vx = (kg - vz * args.kt_chunk) * BK;        // offset inside the chunk
                if (args.g_rows > 0)  // the group's own operand rows (a CTA pair never straddles groups)
                    vx += static_cast<int>((static_cast<int64_t>(r) * BM / args.g_rows) * args.g_rows);
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
                            const uint64_t dv = desc_tc(v + off);
#pragma unroll
                            for (int t = 0; t < BM / TM; ++t) {
                                const uint32_t acc = (it > cstart || kk > 0) ? 1u : 0u;
                                const uint32_t d = d0 + t * C::kAccCols;
                                // A_hi x [V_hi | V_lo]: the two V planes are adjacent in smem (N' = 2N rows)
                                umma_f16(d, desc_tc(st + t * C::kATile + off), dv, VSPLIT ? idesc2 : idesc, acc);
                                umma_f16(d, desc_tc(st + C::kAPlane + t * C::kATile + off), dv, idesc, 1u);
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
                  CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_64B) {
    TensorMapEncodeFn enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {pitch_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swz, promo,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_map_v3(CUtensorMap* m, const void* base, uint64_t rpr, uint64_t cols, uint64_t world, uint32_t box_rows,
                 uint32_t box_k = BK, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_64B, uint64_t slice = 0) {
    TensorMapEncodeFn enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[3] = {rpr, cols, world};
    cuuint64_t strides[2] = {rpr * 2ull, (slice ? slice : rpr * cols) * 2ull};
    cuuint32_t box[3] = {box_k, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
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
    constexpr CUtensorMapSwizzle swz_tc = BK == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    bool ok = make_map_f16(&m_ahi, a.hi, a.cols, a.rows, a.ld * 2ull, BK, BM, promo, swz_tc) &&
              make_map_f16(&m_alo, a.lo, a.cols, a.rows, a.ld * 2ull, BK, BM, promo, swz_tc) &&
              make_map_v3(&m_v, v.v, v.rpr, v.cols, v.world, vbox, BK, swz_tc, v.slice) &&
              make_map_v3(&m_vlo, VSPLIT ? v.vlo : v.v, v.rpr, v.cols, v.world, vbox, BK, swz_tc, v.slice);
    if (v.rpr % BK != 0) return cudaErrorInvalidValue;
    if (!ok) return cudaErrorInvalidValue;
    if (cudaError_t e =
            ensure_smem_attr(reinterpret_cast<const void*>(block_av_tc_kernel<NPAD, VSPLIT>), C::kSmemBytes);
        e != cudaSuccess)
        return e;
    TcArgs args;
    args.total_iters = plan.total_iters;
    args.k_tiles = plan.k_tiles;
    args.k_off = plan.k_off;
    args.k_total = plan.k_total > 0 ? plan.k_total : plan.k_tiles;
    args.kt_chunk = static_cast<int>(v.rpr / BK);
    args.g_rows = v.group_rows;
    args.kc = plan.kc;
    args.partial = partial;
    args.a_policy = 0;
    block_av_tc_kernel<NPAD, VSPLIT><<<2 * plan.grid, kThreads, C::kSmemBytes, stream>>>(m_ahi, m_alo, m_v, m_vlo,
                                                                                       args);
    return cudaGetLastError();
}


// ------------------------------------------------------------------ fused mutual-information pass
// One pass over A and B computes the products of all three MI terms (proj/src/measures.cpp:36-46):
//   Y_A = A·V_A,   Y_B = B·V_B,   Y_J = J·V_J,   J = n·(A∘B) with J_ii = 1/n (proj/src/kernel.cpp:74-108),
// J formed tile by tile from the staged A and B planes and never stored: 8 B of HBM per entry instead
// of 12 B for three separate passes over A, B and a materialised J.
// CTA pairs (cluster of 2, tcgen05 cta_group::2): each CTA owns 128 rows; the leader issues M = 256
// MMAs whose A operands (A, B and J hi/lo planes) come from each CTA's TMEM and whose B operand (the
// iterate) is split by rows between the two CTAs' shared memory.
//   warp 0       TMA: A_hi, A_lo, B_hi, B_lo tiles of this CTA's rows (128 x 64, SWIZZLE_128B, local ring)
//   warp 1       MMA issuer (leader): per K=16 group and operand hi·hi, lo·hi, hi·lo into one accumulator
//   warp 2       TMA: this CTA's half of the six V planes (completing on the leader's barriers)
//   warps 4-11   operand builders (lane quarter warp%4, K half (warp-4)/4): shared memory -> registers ->
//                A, B planes and J = n·(A∘B) (packed half2 split arithmetic) into a ring of TMEM slots
//   warps 12-23  TMEM drains: operand (warp-12)/4, fp32 register accumulation every 256 columns
// setmaxnreg moves registers from warpgroup 0 and the builders to the drains.
constexpr int TBM = 128;
constexpr int TBK = 64;  // k per stage: one 128-byte (SWIZZLE_128B) row of fp16 per TMA request
constexpr int kTriConv = 8;    // two warpgroups: lane quarter warp%4, K half (warp-4)/4
constexpr int kTriDrain = 12;  // three warpgroups: operand (warp-12)/4
constexpr int kTriConv0 = 4, kTriDrain0 = 12;
#ifndef RB_TRI_SMEM_KB
#define RB_TRI_SMEM_KB 220
#endif
#ifndef RB_TRI_AB_STAGES
#define RB_TRI_AB_STAGES 2
#endif
constexpr int kTriThreads = 32 * 24;  // warpgroup 0: TMA (warp 0), MMA (warp 1); setmaxnreg per role

template <int NPAD, bool VSPLIT>
struct TriCfg {
    static constexpr int kAPlane = TBM * TBK * 2;             // 16 KB: one fp16 plane of 128 rows x 64
    static constexpr int kABStage = 4 * kAPlane;              // A_hi, A_lo, B_hi, B_lo
    static constexpr int kVPer = VSPLIT ? 2 : 1;               // V planes per operand
    static constexpr int kVHalf = (NPAD / 2) * TBK * 2;       // this CTA's half of one V plane's rows
    static constexpr int kVStage = 3 * kVPer * kVHalf;
    static constexpr int kABStages = RB_TRI_AB_STAGES;
    static constexpr int kVStagesRaw = (RB_TRI_SMEM_KB * 1024 - kABStages * kABStage) / kVStage;
    static constexpr int kVStages = kVStagesRaw > 8 ? 8 : kVStagesRaw;
    static constexpr int kOpCols = 6 * 8;                     // one K=16 slot: A, B, J hi/lo planes (8 cols each)
    static constexpr int kBufs = (2 * 3 * NPAD + 4 * kOpCols <= 512) ? 2 : 1;  // accumulator buffers
    static constexpr int kOpCol0 = kBufs * 3 * NPAD;          // operand slots after the accumulators
    static constexpr int kSlotsRaw = (512 - kOpCol0) / kOpCols;
    static constexpr int kSlots = kSlotsRaw > 8 ? 8 : kSlotsRaw;  // half-stage operand slots in flight
    static constexpr int kSmemBytes = kABStages * kABStage + kVStages * kVStage + 1024;
    static_assert(NPAD % 16 == 0 && NPAD >= 16 && NPAD <= 80, "fused MI pass: NPAD in [16, 80]");
    static_assert(kSlots >= 4 && kOpCol0 + kSlots * kOpCols <= 512, "TMEM budget");
    static_assert(kVStages >= 1, "need a V ring");
    static_assert(kVHalf % 1024 == 0, "128-byte swizzle atoms");
};

struct TriArgs {
    int64_t total_iters;  // pair_blocks * k_tiles
    int k_tiles;          // k tiles of this launch's K window
    int k_off, k_total;   // K window: tile k of the launch is global tile (k_off + k) mod k_total
    int kt_chunk;         // k tiles per V chunk (rpr / BK)
    int kc;               // k tiles per TMEM chunk
    int64_t dp_blocks;    // pair blocks owned whole (waves of pairs); stream-K over the rest
    float* partial[3];    // [slots][NPAD][128] per operand (A, B, J)
    int64_t row0;         // global index of this rank's first row (J diagonal)
    uint32_t scale_a;     // fp16x2 2^ea, 2^eb with ea + eb = log2(stored J / (stored A · stored B))
    uint32_t scale_b;
    float diag;           // stored J_ii
    int a_policy;         // 0: evict_first for the A/B stream, 1: evict_normal
};

// The (pair block, k range) segments of one CTA pair: whole pair blocks in data-parallel waves (all
// pairs walk the same k tiles at about the same time, so the three V tiles of a k tile leave HBM once
// per wave and are served from L2 to the other pairs), then an even stream-K share of the tail.
struct TriSegs {
    int64_t waves, grid, pair, KT, dp, it, it_end, w = 0;
    __device__ TriSegs(const TriArgs& a, int p, int P) : grid(P), pair(p), KT(a.k_tiles), dp(a.dp_blocks) {
        waves = dp / P;
        const int64_t tail = a.total_iters - dp * KT;
        it = tail * p / P;
        it_end = tail * (p + 1) / P;
    }
    __device__ bool next(int64_t& r, int& k0, int& k1) {
        if (w < waves) {
            r = w * grid + pair;
            k0 = 0;
            k1 = static_cast<int>(KT);
            ++w;
            return true;
        }
        if (it >= it_end) return false;
        const int64_t rt = it / KT;
        const int64_t e = min(it_end, (rt + 1) * KT);
        r = dp + rt;
        k0 = static_cast<int>(it - rt * KT);
        k1 = static_cast<int>(e - rt * KT);
        it = e;
        return true;
    }
    // partial slot of 128-row block 2r + rank (same layout as the matrix-free path's epilogue)
    __device__ int64_t slot(int64_t r, int rank) const { return r < dp ? 2 * r + rank : 2 * (r + pair) + rank; }
};

__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.b32 %0, 1, 0, e;\n\t}" : "=r"(p));
    return p != 0;
}

__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// a·b − c with the negation folded into the FMA's operand modifier (no separate sign-flip instruction)
__device__ __forceinline__ uint32_t hfma2_negc(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("{\n\t.reg .b32 nc;\n\tneg.f16x2 nc, %3;\n\tfma.rn.f16x2 %0, %1, %2, nc;\n\t}" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// 2 entries of J from packed (hi, lo) fp16 pairs of A and B, as a (hi, lo) fp16 split, in packed
// half2 arithmetic: with a = a_h + a_l and b = b_h + b_l prescaled by exact powers of two,
//   j_h = fl16(a_h b_h),  r = a_h b_h - j_h (exact: an 11x11-bit product minus its rounding),
//   j_l = fl16(a_h b_l + fl16(a_l b_h + r))   (a_l b_l ~ 2^-22 relative is dropped, as in the split product)
// so J is carried to ~21 bits like the materialised split of hadamard_split_kernel (22 bits).
__device__ __forceinline__ void joint_pair(uint32_t ah, uint32_t al, uint32_t bh, uint32_t bl, uint32_t sa,
                                           uint32_t sb, uint32_t& jh, uint32_t& jl) {
    ah = hmul2(ah, sa), al = hmul2(al, sa), bh = hmul2(bh, sb), bl = hmul2(bl, sb);
    jh = hmul2(ah, bh);
    const uint32_t r = hfma2_negc(ah, bh, jh);
    jl = hfma2(ah, bl, hfma2(al, bh, r));
}

__device__ __forceinline__ uint32_t f2h(float2 f) {
    const __half2 h = __float22half2_rn(f);
    uint32_t u;
    memcpy(&u, &h, 4);
    return u;
}

template <int NPAD, bool VSPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTriThreads, 1)
    block_av_tri_kernel(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                        const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                        const __grid_constant__ CUtensorMap map_va, const __grid_constant__ CUtensorMap map_valo,
                        const __grid_constant__ CUtensorMap map_vb, const __grid_constant__ CUtensorMap map_vblo,
                        const __grid_constant__ CUtensorMap map_vj, const __grid_constant__ CUtensorMap map_vjlo,
                        TriArgs args) {
    using C = TriCfg<NPAD, VSPLIT>;
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t ab_full[C::kABStages], ab_empty[C::kABStages];
    __shared__ __align__(8) uint64_t v_full[C::kVStages], v_empty[C::kVStages];
    __shared__ __align__(8) uint64_t op_full[C::kSlots], op_empty[C::kSlots];
    __shared__ __align__(8) uint64_t acc_full[C::kBufs], acc_empty[C::kBufs];
    __shared__ uint32_t tmem_base_smem;

    const int warp = threadIdx.x / kWarp;
    const int lane = threadIdx.x % kWarp;
    const int G = gridDim.x / 2;
    const int pair = blockIdx.x / 2;
    const uint32_t rank = cluster_ctarank();  // 0 = leader: issues the pair's MMAs
    const bool leader = rank == 0;
    constexpr uint16_t kBoth = 0b11;

    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
    const uint32_t v_u32 = base_u32 + C::kABStages * C::kABStage;  // V ring after the A/B ring

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&map_ahi), prefetch_tmap(&map_alo), prefetch_tmap(&map_bhi), prefetch_tmap(&map_blo);
        prefetch_tmap(&map_va), prefetch_tmap(&map_vb), prefetch_tmap(&map_vj);
        if (VSPLIT) prefetch_tmap(&map_valo), prefetch_tmap(&map_vblo), prefetch_tmap(&map_vjlo);
        for (int s = 0; s < C::kABStages; ++s) {
            mbar_init(&ab_full[s], 1);
            mbar_init(&ab_empty[s], kTriConv);  // every builder warp has read the tiles
        }
        for (int s = 0; s < C::kVStages; ++s) {
            mbar_init(&v_full[s], 1);   // leader: both CTAs' V halves landed
            mbar_init(&v_empty[s], 1);  // the pair's MMAs are done with the stage
        }
        for (int b = 0; b < C::kSlots; ++b) {
            mbar_init(&op_full[b], 2 * (kTriConv / 2));  // leader: both CTAs' converters of this K half
            mbar_init(&op_empty[b], 1);
        }
        for (int b = 0; b < C::kBufs; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 2 * kTriDrain);  // leader: both CTAs' drains
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_2sm(&tmem_base_smem, 512);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = tmem_base_smem;

    // registers move only between warpgroups of the CTA: 4x(80-40) + 8x(80-64) = 12x(104-80) per thread
    // (drains: 80 fp32 accumulators + a 16-column TMEM load in flight)
    if (warp < kTriConv0) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (warp == 0 || warp == 2) {
        // ---------------- TMA: A/B tiles of this CTA's rows (warp 0, local ring); its half of the V planes
        // (warp 2, completing on the leader's barriers). Separate issuers: neither ring's back-pressure
        // delays the other's loads.
        if (lane == 0) {
            const uint64_t pol_stream = args.a_policy ? policy_evict_normal() : policy_evict_first();
            const uint64_t pol_keep = policy_evict_last();
            const CUtensorMap* vmap[3][2] = {{&map_va, &map_valo}, {&map_vb, &map_vblo}, {&map_vj, &map_vjlo}};
            int as = 0, vs = 0;
            uint32_t aph = 0, vph = 0;
            TriSegs sg(args, pair, G);
            int64_t rp;
            int k0, k1;
            while (sg.next(rp, k0, k1)) {
                const int r = static_cast<int>(2 * rp + rank);
                for (int k = k0; k < k1; ++k) {
                    const int kg = k + args.k_off < args.k_total ? k + args.k_off : k + args.k_off - args.k_total;
                    if (warp == 0) {
                        mbar_wait(&ab_empty[as], aph ^ 1u);
                        uint8_t* st = base + as * C::kABStage;
                        mbar_arrive_expect_tx(&ab_full[as], C::kABStage);
                        tma_load_2d(st, &map_ahi, &ab_full[as], kg * TBK, r * TBM, pol_stream);
                        tma_load_2d(st + C::kAPlane, &map_alo, &ab_full[as], kg * TBK, r * TBM, pol_stream);
                        tma_load_2d(st + 2 * C::kAPlane, &map_bhi, &ab_full[as], kg * TBK, r * TBM, pol_stream);
                        tma_load_2d(st + 3 * C::kAPlane, &map_blo, &ab_full[as], kg * TBK, r * TBM, pol_stream);
                        if (++as == C::kABStages) as = 0, aph ^= 1u;
                    } else {
                        mbar_wait(&v_empty[vs], vph ^ 1u);
                        if (leader) mbar_arrive_expect_tx(&v_full[vs], 2 * C::kVStage);
                        const uint32_t bar = mapa_shared(&v_full[vs], 0);
                        uint8_t* vt = base + (v_u32 - base_u32) + vs * C::kVStage;
                        const int vz = kg / args.kt_chunk;
                        const int vx = (kg - vz * args.kt_chunk) * TBK;
#pragma unroll
                        for (int q = 0; q < 3 * C::kVPer; ++q)  // rows [rank·NPAD/2, +NPAD/2) of every plane
                            tma_load_3d_2sm(vt + q * C::kVHalf, vmap[q / C::kVPer][q % C::kVPer], bar, vx,
                                            static_cast<int>(rank) * (NPAD / 2), vz, pol_keep);
                        if (++vs == C::kVStages) vs = 0, vph ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader): M = 256 over the pair, A operands from TMEM ----------------
        if (leader) {
            constexpr uint32_t idesc = umma_idesc_f16_f32(2 * TBM, NPAD);
            const uint64_t dv0 = umma_desc_sw128(v_u32);
            int vs = 0;
            uint32_t vph = 0, u = 0, chunk = 0;
            TriSegs sg(args, pair, G);
            int64_t rp;
            int k0, k1;
            while (sg.next(rp, k0, k1)) {
                int it = k0;
                while (it < k1) {
                    const int cend = min(k1, it + args.kc);
                    const uint32_t buf = chunk % C::kBufs;
                    mbar_wait(&acc_empty[buf], ((chunk / C::kBufs) & 1u) ^ 1u);
                    tc_fence_after();
                    const uint32_t d0 = tmem + buf * (3 * NPAD);
                    const int cstart = it;
                    for (; it < cend; ++it, ++u) {
                        mbar_wait(&v_full[vs], vph);
                        const uint64_t dv = dv0 + static_cast<uint64_t>((vs * C::kVStage) >> 4);
                        const uint32_t cont = it > cstart ? 1u : 0u;
#pragma unroll
                        for (int kk = 0; kk < TBK / 16; ++kk) {  // K group kk of the tile: its own operand slot
                            const uint32_t q = (TBK / 16) * u + kk, slot = q % C::kSlots;
                            mbar_wait(&op_full[slot], (q / C::kSlots) & 1u);
                            tc_fence_after();
                            const uint32_t ta = tmem + C::kOpCol0 + slot * C::kOpCols;
                            if (elect_one()) {
#pragma unroll
                                for (int o = 0; o < 3; ++o) {
                                    const uint32_t d = d0 + o * NPAD;
                                    const uint32_t th = ta + o * 16;  // operand o: hi at +0, lo at +8
                                    const uint64_t vh = dv + (((o * C::kVPer) * C::kVHalf + kk * 32) >> 4);
                                    umma2_f16_ts(d, th, vh, idesc, cont | (kk > 0));             // hi·hi
                                    umma2_f16_ts(d, th + 8, vh, idesc, 1u);                      // lo·hi
                                    if (VSPLIT) umma2_f16_ts(d, th, vh + (C::kVHalf >> 4), idesc, 1u);  // hi·lo
                                }
                                umma2_commit_mc(&op_empty[slot], kBoth);
                            }
                            __syncwarp();
                        }
                        if (elect_one()) umma2_commit_mc(&v_empty[vs], kBoth);
                        __syncwarp();
                        if (++vs == C::kVStages) vs = 0, vph ^= 1u;
                    }
                    if (elect_one()) umma2_commit_mc(&acc_full[buf], kBoth);
                    __syncwarp();
                    ++chunk;
                }
            }
        }
    } else if (warp >= kTriConv0 && warp < kTriConv0 + kTriConv) {
        // ---------------- operand builders: A, B and J = n·(A∘B) into TMEM ----------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 64;\n" ::: "memory");
        // K groups {half, half + 2} (16 columns each) of the tile: the two halves build groups 0 and 1
        // side by side, then 2 and 3 -- the order the MMA issuer consumes them in
        const int half = (warp - kTriConv0) / 4;
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        const int sw = row & 7;  // 128-byte swizzle: 16-byte chunk c of row r sits at c ^ (r & 7)
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t op_full_l = mapa_shared(&op_full[0], 0);
        const uint32_t dh = f2h(make_float2(args.diag, args.diag));
        int as = 0;
        uint32_t aph = 0, u = 0;
        TriSegs sg(args, pair, G);
        int64_t rp;
        int k0, k1;
        while (sg.next(rp, k0, k1)) {
            const int64_t grow = args.row0 + (2 * rp + rank) * TBM + row;  // global row (J diagonal)
            const int64_t wrow = grow - lane;                                  // the warp's first row
            for (int k = k0; k < k1; ++k, ++u) {
                const int kg = k + args.k_off < args.k_total ? k + args.k_off : k + args.k_off - args.k_total;
                mbar_wait(&ab_full[as], aph);
                const uint8_t* src = base + as * C::kABStage + row * 128;
#pragma unroll
                for (int sub = 0; sub < 2; ++sub) {
                    const int g = half + 2 * sub;  // K group: columns [16g, 16g + 16) of the tile
                    uint32_t pa_h[8], pa_l[8], pb_h[8], pb_l[8], jh[8], jl[8];
#pragma unroll
                    for (int c2 = 0; c2 < 2; ++c2) {
                        const int po = ((2 * g + c2) ^ sw) * 16;
                        const uint4 x0 = *reinterpret_cast<const uint4*>(src + po);
                        const uint4 x1 = *reinterpret_cast<const uint4*>(src + C::kAPlane + po);
                        const uint4 x2 = *reinterpret_cast<const uint4*>(src + 2 * C::kAPlane + po);
                        const uint4 x3 = *reinterpret_cast<const uint4*>(src + 3 * C::kAPlane + po);
                        pa_h[4 * c2] = x0.x, pa_h[4 * c2 + 1] = x0.y, pa_h[4 * c2 + 2] = x0.z, pa_h[4 * c2 + 3] = x0.w;
                        pa_l[4 * c2] = x1.x, pa_l[4 * c2 + 1] = x1.y, pa_l[4 * c2 + 2] = x1.z, pa_l[4 * c2 + 3] = x1.w;
                        pb_h[4 * c2] = x2.x, pb_h[4 * c2 + 1] = x2.y, pb_h[4 * c2 + 2] = x2.z, pb_h[4 * c2 + 3] = x2.w;
                        pb_l[4 * c2] = x3.x, pb_l[4 * c2 + 1] = x3.y, pb_l[4 * c2 + 2] = x3.z, pb_l[4 * c2 + 3] = x3.w;
                    }
                    if (sub == 1) {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&ab_empty[as]);  // this warp is done with the A/B stage
                    }
#pragma unroll
                    for (int t = 0; t < 8; ++t)
                        joint_pair(pa_h[t], pa_l[t], pb_h[t], pb_l[t], args.scale_a, args.scale_b, jh[t], jl[t]);
                    // J_ii = 1/n (kernel.cpp:98-99). Branch-free per-register selects: a conditional write to
                    // jh[e / 2] is compiled into a dynamically indexed local-memory array (spilled to the stack
                    // every K group: ~40 GB of local stores per config-4 launch, round-2 ncu)
                    // Only the few K groups whose 16 columns meet this warp's 32 rows take the branch
                    // (warp-uniform test: rows [wrow, wrow + 32) vs columns [c0, c0 + 16)).
                    const int64_t c0 = static_cast<int64_t>(kg) * TBK + 16 * g;
                    if (wrow < c0 + 16 && c0 < wrow + 32) {
                        const int64_t e = grow - c0;
                        const int qd = (e >= 0 && e < 16) ? static_cast<int>(e) : -2;
                        const uint32_t dmask = (qd & 1) ? 0xFFFF0000u : 0x0000FFFFu;
#pragma unroll
                        for (int t = 0; t < 8; ++t) {
                            const uint32_t sel = (t == (qd >> 1)) ? dmask : 0u;
                            jh[t] = (jh[t] & ~sel) | (dh & sel);
                            jl[t] &= ~sel;
                        }
                    }
                    const uint32_t q = (TBK / 16) * u + g, slot = q % C::kSlots;
                    mbar_wait(&op_empty[slot], ((q / C::kSlots) & 1u) ^ 1u);  // earlier MMAs are done with the slot
                    tc_fence_after();
                    const uint32_t ta = tmem + lane_off + C::kOpCol0 + slot * C::kOpCols;
                    tmem_st8(ta, pa_h);
                    tmem_st8(ta + 8, pa_l);
                    tmem_st8(ta + 16, pb_h);
                    tmem_st8(ta + 24, pb_l);
                    tmem_st8(ta + 32, jh);
                    tmem_st8(ta + 40, jl);
                    tmem_st_wait();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(op_full_l + slot * 8);
                }
                if (++as == C::kABStages) as = 0, aph ^= 1u;
            }
        }
    } else if (warp >= kTriDrain0) {
        // ---------------- TMEM drains: operand (warp-12)/4, lane quarter warp%4 ----------------
        asm volatile("setmaxnreg.inc.sync.aligned.u32 104;\n" ::: "memory");
        const int op = (warp - kTriDrain0) / 4;
        const int quarter = warp & 3;
        const int row_local = quarter * 32 + lane;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + op * NPAD;
        const uint32_t acc_empty_l = mapa_shared(&acc_empty[0], 0);
        float acc[NPAD];
#pragma unroll
        for (int j = 0; j < NPAD; ++j) acc[j] = 0.f;
        uint32_t chunk = 0;
        TriSegs sg(args, pair, G);
        int64_t rp;
        int k0, k1;
        while (sg.next(rp, k0, k1)) {
            for (int it = k0; it < k1; it += args.kc) {
                const uint32_t buf = chunk % C::kBufs;
                mbar_wait(&acc_full[buf], (chunk / C::kBufs) & 1u);
                tc_fence_after();
                const uint32_t t0 = lane_base + buf * (3 * NPAD);
                // 16 columns per TMEM load round trip (the MMA issuer waits for this drain at every
                // chunk boundary: the accumulator is single-buffered)
#pragma unroll
                for (int j0 = 0; j0 < NPAD; j0 += 16) {
                    float m[16];
                    tmem_ld16(t0 + j0, m);
                    tmem_ld_wait();
#pragma unroll
                    for (int i = 0; i < 16; ++i) acc[j0 + i] += m[i];
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(acc_empty_l + buf * 8);
                ++chunk;
            }
            const int64_t slot = sg.slot(rp, static_cast<int>(rank));
            float* dst = args.partial[op] + (slot * NPAD) * TBM + row_local;
#pragma unroll
            for (int j = 0; j < NPAD; ++j) {
                dst[j * TBM] = acc[j];
                acc[j] = 0.f;
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer is done with the pair's TMEM and barriers
    if (warp == 1) tmem_dealloc_2sm(tmem, 512);
}

template <int NPAD, bool VSPLIT>
cudaError_t launch_tri(const SplitMatrixView& a, const SplitMatrixView& b, const SplitPanelView* v,
                       const StreamKPlan& plan, float* const* partial, int64_t row0, float factor, float diag,
                       cudaStream_t stream) {
    using C = TriCfg<NPAD, VSPLIT>;
    CUtensorMap ma[4], mv[6];
    const uint32_t vbox = NPAD / 2;  // each CTA of the pair stages half of every V plane's rows
    // measured on B200: 128-byte L2 promotion + evict_first for the A/B stream beats 256 B / none and
    // evict_normal by 2-4 % (profiles/r1_microbench.md)
    // (round 2, aligned pitch: 128 B 19.5 ms, none 19.7 ms, 256 B 20.2 ms per config-4 pass, same box)
    const CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    constexpr CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B;
    bool ok = make_map_f16(&ma[0], a.hi, a.cols, a.rows, a.ld * 2ull, TBK, TBM, promo, swz) &&
              make_map_f16(&ma[1], a.lo, a.cols, a.rows, a.ld * 2ull, TBK, TBM, promo, swz) &&
              make_map_f16(&ma[2], b.hi, b.cols, b.rows, b.ld * 2ull, TBK, TBM, promo, swz) &&
              make_map_f16(&ma[3], b.lo, b.cols, b.rows, b.ld * 2ull, TBK, TBM, promo, swz);
    for (int o = 0; o < 3 && ok; ++o) {
        if (VSPLIT != (v[o].vlo != nullptr) || v[o].rpr % TBK != 0) return cudaErrorInvalidValue;
        ok = make_map_v3(&mv[2 * o], v[o].v, v[o].rpr, v[o].cols, v[o].world, vbox, TBK, swz, v[o].slice) &&
             make_map_v3(&mv[2 * o + 1], VSPLIT ? v[o].vlo : v[o].v, v[o].rpr, v[o].cols, v[o].world, vbox, TBK,
                         swz, v[o].slice);
    }
    if (!ok) return cudaErrorInvalidValue;
    if (cudaError_t e =
            ensure_smem_attr(reinterpret_cast<const void*>(block_av_tri_kernel<NPAD, VSPLIT>), C::kSmemBytes);
        e != cudaSuccess)
        return e;
    TriArgs args;
    args.total_iters = plan.total_iters;
    args.k_tiles = plan.k_tiles;
    args.k_off = plan.k_off;
    args.k_total = plan.k_total > 0 ? plan.k_total : plan.k_tiles;
    args.kt_chunk = static_cast<int>(v[0].rpr / TBK);
    args.kc = plan.kc;
    args.dp_blocks = plan.dp_blocks;
    for (int o = 0; o < 3; ++o) args.partial[o] = partial[o];
    args.row0 = row0;
    int e = 0;
    if (!(factor > 0.0f) || std::frexp(factor, &e) != 0.5f) return cudaErrorInvalidValue;  // 2^(e-1)
    const int ea = (e - 1) / 2, eb = (e - 1) - ea;  // each prescale a normal fp16 power of two
    if (ea < -14 || eb < -14 || ea > 15 || eb > 15) return cudaErrorInvalidValue;
    const __half ha = __float2half(std::ldexp(1.0f, ea)), hb = __float2half(std::ldexp(1.0f, eb));
    const uint32_t ua = __half_as_ushort(ha), ub = __half_as_ushort(hb);
    args.scale_a = ua | (ua << 16);
    args.scale_b = ub | (ub << 16);
    args.diag = diag;
    args.a_policy = 0;
    block_av_tri_kernel<NPAD, VSPLIT><<<2 * plan.grid, kTriThreads, C::kSmemBytes, stream>>>(
        ma[0], ma[1], ma[2], ma[3], mv[0], mv[1], mv[2], mv[3], mv[4], mv[5], args);
    return cudaGetLastError();
}

}  // namespace

int tc_block_rows() { return BM; }
int tc_block_k() { return BK; }

// k tiles of a window: [col0 / tile, ceil(min(col0 + cols, n) / tile)), the end wrapping past n
void apply_window(StreamKPlan& p, int64_t n, int tile, KWindow w) {
    const int total = static_cast<int>((n + tile - 1) / tile);
    if (w.cols < 0 || (w.col0 == 0 && w.cols >= n)) {
        p.k_tiles = total;
        p.k_off = 0, p.k_total = 0;
        return;
    }
    const int64_t c0 = w.col0 % n;
    const int off = static_cast<int>(c0 / tile);
    const int64_t end = c0 + w.cols;  // may pass n: the window wraps
    const int cnt = end <= n ? static_cast<int>((end + tile - 1) / tile) - off
                             : (total - off) + static_cast<int>((end - n + tile - 1) / tile);
    p.k_tiles = std::max(0, std::min(cnt, total));
    p.k_off = off, p.k_total = total;
}

StreamKPlan make_streamk_plan(int64_t rows, int64_t cols, int grid, int kc, KWindow w) {
    // grid = CTAs (rounded down to pairs); iterations are (row-block-pair, k-tile)
    StreamKPlan p;
    p.row_blocks = static_cast<int>((rows + BM - 1) / BM);
    apply_window(p, cols, BK, w);
    const int64_t pair_blocks = (p.row_blocks + 1) / 2;
    p.total_iters = pair_blocks * p.k_tiles;
    int pairs = std::max(1, grid / 2);
    if (p.total_iters < pairs) pairs = static_cast<int>(p.total_iters > 0 ? p.total_iters : 1);
    p.grid = pairs;  // stream-K participants (pairs)
    p.cluster = 2;
    p.kc = std::max(1, kc * 32 / BK);  // kc counts 32-column tiles
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

StreamKPlan make_tri_plan(int64_t rows, int64_t cols, int grid, int kc, KWindow w) {
    // 128-row blocks, CTA pairs walking the same k tiles (iterations: (row-block-pair, k-tile))
    StreamKPlan p;
    p.row_blocks = static_cast<int>((rows + TBM - 1) / TBM);
    apply_window(p, cols, TBK, w);
    const int64_t pair_blocks = (p.row_blocks + 1) / 2;
    p.total_iters = pair_blocks * p.k_tiles;
    int pairs = std::max(1, grid / 2);
    if (p.total_iters < pairs) pairs = static_cast<int>(p.total_iters > 0 ? p.total_iters : 1);
    p.grid = pairs;
    p.cluster = 2;
    // half the split product's TMEM accumulation length: all three split products land in one accumulator,
    // whose truncation bias grows with the chunk (config 4 vars entropy: +5e-6 from 256 to 512 columns,
    // +1.6e-5 more at 1024; the drain cost is invisible in the pass time)
    p.kc = std::max(1, kc * 32 / TBK / 2);
    p.slots = static_cast<int>(2 * (pair_blocks + pairs));
    p.rows_per_block = TBM;
    p.dp_blocks = static_cast<int>((pair_blocks / pairs) * pairs);  // whole waves; the remainder stream-K
    return p;
}

int tri_max_cols() { return 80; }

cudaError_t launch_block_av_tri(const SplitMatrixView& a, const SplitMatrixView& b, const SplitPanelView* v,
                                const StreamKPlan& plan, float* const* partial, int64_t row0, double factor,
                                double diag, cudaStream_t stream) {
    const int npad = tc_npad(v[0].cols);
    if (v[1].cols != v[0].cols || v[2].cols != v[0].cols) return cudaErrorInvalidValue;
    const float f = static_cast<float>(factor), dg = static_cast<float>(diag);
#define RB_TRI_CASE(N)                                                                               \
    case N:                                                                                          \
        return v[0].vlo ? launch_tri<N, true>(a, b, v, plan, partial, row0, f, dg, stream)           \
                        : launch_tri<N, false>(a, b, v, plan, partial, row0, f, dg, stream);
    switch (npad) {
        RB_TRI_CASE(16)
        RB_TRI_CASE(32)
        RB_TRI_CASE(48)
        RB_TRI_CASE(64)
        RB_TRI_CASE(80)
        default: return cudaErrorInvalidValue;
    }
#undef RB_TRI_CASE
}

}  // namespace rb
