// Matrix-free block product (config 5; SURVEY §8(a5) "matrix-free variant", §7 step 6):
//   Y_i = Σ_j K(x_i, x_j) · V_j,   K = exp(−|x_i − x_j|² / (2σ²)),  K_ii = 1,
// with the kernel entries recomputed from bf16 X on the tensor cores and never stored
// (the reference materialises A: proj/src/kernel.cpp:35-72 + ops.cpp:98-107).
//
// FlashAttention-shaped, without the softmax bookkeeping (kernel values are already in (0, 1]):
//   S  = [X_i | a_i] · [X_j | a'_j]ᵀ = x_i·x_j − |x_i|²/2 − |x_j|²/2 = −|x_i − x_j|²/2
//        tcgen05.mma kind::f16 (bf16 in, fp32 accumulate) → TMEM. The squared norms ride in 16
//        augmented K columns: a_i = [h_i, m_i, l_i, 1, 1, 1, 0…], a'_j = [1, 1, 1, h_j, m_j, l_j, 0…]
//        with h + m + l = −|x|²/2 split over three bf16 (24-bit significand), so the exp warps
//        do no bias arithmetic at all.
//   P  = exp2(c2·S)             exp warps: TMEM → registers → MUFU ex2 → fp16 → back into TMEM
//                               (over the S columns just read; c2 = log2(e)/σ²)
//   O += P · V_j                tcgen05.mma kind::f16 with A = P from TMEM, B = V_j from smem
//
// CTA pairs (tcgen05 cta_group::2): a cluster of two CTAs owns 256 rows (128 each, UMMA M=256);
// the leader issues every MMA for the pair. Each CTA stages only HALF of the shared operands —
// 64 of the 128 j-rows of X_j / a'_j and NPAD/2 of the V_j columns — so the L2→SMEM traffic and
// the shared-memory operand reads per row are halved against one CTA per 128 rows.
// Warp roles per CTA: 0 TMA (X_i, X_j half), 1 S issuer and 3 P·V issuer (leader only; two issuing
// threads so neither chain's barrier waits stall the other's MMAs), 2 TMA (V_j half), 4-19 four exp
// warpgroups (columns [32h, 32h+32) of each S tile) that also drain a quarter of O each into fp32
// registers every kc j-blocks (the tensor core's long-K accumulation is lossy, see block_av_tc.cu).
// S/P are triple-buffered in TMEM, O double-buffered for NPAD <= 64.
// Persistent schedule: whole 256-row blocks in data-parallel waves of pairs (L2 reuse of X_j /
// V_j across the wave) plus a stream-K split of the tail; partial slots and the pass epilogue
// are shared with the materialised path (cluster = 2).
#include <algorithm>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace rb {

namespace {

constexpr int MB = 128;   // rows per CTA (the pair's UMMA M is 256)
constexpr int JB = 128;   // j-block: S tile N and P·V K
constexpr int kAug = 16;  // augmented K columns carrying −|x|²/2
constexpr int kEG = 4;               // exp/drain warpgroups; group h owns S columns [h·CW, (h+1)·CW)
constexpr int CW = JB / kEG;         // S columns per exp thread and j-block
constexpr uint32_t kExpWarps = 4 * kEG;
constexpr int kMfThreads = 32 * (4 + kExpWarps);  // warps 0-3: TMA(X), S issuer, TMA(V), P·V issuer

template <int DP, int NPAD>
struct MfCfg {
    static constexpr int kXTile = MB * DP * 2;          // X_i, bf16, [128][DP] as DP/64 SW128 sub-tiles
    static constexpr int kXSub = MB * 64 * 2;           // 16 KB
    static constexpr int kATile = MB * kAug * 2;        // a_i, bf16 [128][16], SW32
    static constexpr int kFixed = kXTile + kATile;
    static constexpr int kXjTile = (JB / 2) * DP * 2;   // this CTA's half of X_j: [64][DP]
    static constexpr int kXjSub = (JB / 2) * 64 * 2;    // 8 KB
    static constexpr int kAjTile = (JB / 2) * kAug * 2; // half of a'_j: [64][16]
    static constexpr int kXSlot = kXjTile + kAjTile;    // 1024-aligned
    static constexpr int kNH = NPAD / 2;                // V_j columns staged by this CTA
    static constexpr int kVTile = kNH * JB * 2;         // [kNH][128] as two SW128 sub-tiles
    static constexpr int kVSub = kNH * 64 * 2;
    static constexpr int kBudget = 226 * 1024 - 1024 - kFixed;
    static constexpr int kVStages = 4;
    static constexpr int kXStagesRaw = (kBudget - kVStages * kVTile) / kXSlot;
    static constexpr int kXStages = kXStagesRaw > 4 ? 4 : kXStagesRaw;
    static constexpr int kSmem = kFixed + kXStages * kXSlot + kVStages * kVTile + 1024;
    static constexpr int kNS = 3;           // S/P buffers in TMEM (S(j+3) never waits on P·V(j))
    static constexpr int kOCol = kNS * JB;  // O buffers after the S/P buffers
    static constexpr int kNO = (512 - kOCol) / NPAD >= 2 ? 2 : 1;
    static constexpr int kOW = NPAD / kEG;  // O columns drained by each exp warpgroup
    static_assert(DP == 64 || DP == 128, "feature dimension is padded to 64 or 128");
    static_assert(NPAD % 16 == 0 && NPAD <= 128, "NPAD must be a multiple of 16 in [16,128]");
    static_assert(kXStages >= 2, "need a double-buffered X_j ring");
    static_assert(kXSlot % 1024 == 0 && kVTile % 1024 == 0 && kFixed % 1024 == 0, "SW128 alignment");
    static_assert(kOCol + kNO * NPAD <= 512, "TMEM budget");
    static_assert(kOW % 4 == 0, "O drain granularity");
};

struct MfArgs {
    int64_t total_iters;  // pair_blocks * j_blocks
    int j_blocks;         // j-blocks of this launch's window
    int j_off, j_total;   // window: j-block jb of the launch is global block (j_off + jb) mod j_total
    __device__ int global_jb(int jb) const { return jb + j_off < j_total ? jb + j_off : jb + j_off - j_total; }
    int kc;               // j-blocks per O accumulation chunk
    int64_t row0;         // first global row of this rank
    int kt_chunk;         // j-blocks per V chunk (rpr / 128)
    float c2;             // log2(e)/σ²
    int64_t dp_blocks;    // 256-row blocks owned whole (waves of pairs); stream-K over the rest
    float* partial;       // [slots][NPAD][128]
    unsigned long long* trace;  // RB_MF_TRACE builds only: clock64 stamps of CTA 0's first 256 j-blocks
};

#ifdef RB_MF_TRACE
__device__ __forceinline__ unsigned long long clock_now() {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    return c;
}
#define MF_STAMP(slot, j) \
    if (args.trace && blockIdx.x == 0 && (j) < 256) args.trace[(j) * 16 + (slot)] = clock_now();
#else
#define MF_STAMP(slot, j)
#endif

// The (256-row block, j-range) segments one CTA pair processes: whole blocks in data-parallel
// waves (all pairs walk the same j-blocks at about the same time, so X_j / V_j are fetched from
// HBM once per wave and served from L2 to the other pairs), then an even stream-K share of the tail.
struct MfSegments {
    int64_t waves, grid, pair, J, dp_rows, it, it_end, w = 0;
    __device__ MfSegments(const MfArgs& a, int p, int P) : grid(P), pair(p), J(a.j_blocks), dp_rows(a.dp_blocks) {
        waves = a.dp_blocks / P;
        const int64_t tail = a.total_iters - a.dp_blocks * J;
        it = tail * p / P;
        it_end = tail * (p + 1) / P;
    }
    __device__ bool next(int64_t& r, int& j0, int& j1) {
        if (w < waves) {
            r = w * grid + pair;
            j0 = 0;
            j1 = static_cast<int>(J);
            ++w;
            return true;
        }
        if (it >= it_end) return false;
        const int64_t rt = it / J;
        const int64_t e = min(it_end, (rt + 1) * J);
        r = dp_rows + rt;
        j0 = static_cast<int>(it - rt * J);
        j1 = static_cast<int>(e - rt * J);
        it = e;
        return true;
    }
    // partial slot of 128-row block 2r + rank (epilogue: panel.cu, cluster = 2)
    __device__ int64_t slot(int64_t r, uint32_t rank) const {
        return r < dp_rows ? 2 * r + rank : 2 * (r + pair) + rank;
    }
};

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

// exp2 of a pair on the FMA pipe (offloads the MUFU): 2^x = 2^n · 2^f, n = rint(x), f ∈ [-½, ½],
// 2^f by a degree-4 near-minimax polynomial (max relative error 2.7e-6, far below the fp16
// rounding of P), 2^n added into the exponent bits.
__device__ __forceinline__ float2 exp2_poly(float2 a) {
    const float2 x = make_float2(fmaxf(a.x, -125.f), fmaxf(a.y, -125.f));  // keeps 2^n·p a normal float
    const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5·2^23: rint into the low mantissa bits
    const float2 t = __fadd2_rn(x, magic);
    const float2 n = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
    const float2 f = __ffma2_rn(n, make_float2(-1.f, -1.f), x);
    float2 p = __ffma2_rn(make_float2(0.0095701f, 0.0095701f), f, make_float2(0.05591786f, 0.05591786f));
    p = __ffma2_rn(p, f, make_float2(0.24024744f, 0.24024744f));
    p = __ffma2_rn(p, f, make_float2(0.6931218f, 0.6931218f));
    p = __ffma2_rn(p, f, make_float2(0.9999993f, 0.9999993f));
    return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                       __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}

constexpr int kEmuPairs = 0;  // of every 8 pairs, this many go to the FMA pipe (0: measured fastest on B200)

// 16 kernel values of one row: p = exp2(c2·s), packed to 8 fp16 pairs (K order)
template <bool DIAG>
__device__ __forceinline__ void exp16(const float* sv, float2 c2v, int col0, int row, uint32_t* pk) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const float2 a = __fmul2_rn(make_float2(sv[2 * e], sv[2 * e + 1]), c2v);
        float p0, p1;
        if (e % 4 >= 4 - kEmuPairs / 2) {
            const float2 q = exp2_poly(a);
            p0 = q.x, p1 = q.y;
        } else {
            p0 = ex2(a.x), p1 = ex2(a.y);
        }
        if (DIAG) {  // K_ii = 1 exactly (proj/src/ops.cpp:12)
            if (col0 + 2 * e == row) p0 = 1.0f;
            if (col0 + 2 * e + 1 == row) p1 = 1.0f;
        }
        pk[e] = pack_f16x2_clamp1(p0, p1);
    }
}

// 32 columns of S (TMEM, two pipelined x16 reads) -> 16 fp16 pairs of P written back to TMEM at wr
template <bool DIAG>
__device__ __forceinline__ void exp_store32(uint32_t rd, uint32_t wr, float2 c2v, int col0, int row) {
    float sv[32];
    uint32_t pk[16];
    tmem_ld32(rd, sv);  // one 32-column read
    tmem_ld_wait();
    exp16<DIAG>(sv, c2v, col0, row, pk);
    exp16<DIAG>(sv + 16, c2v, col0 + 16, row, pk + 8);
    tmem_st16(wr, pk);  // one 16-column write of the fp16 pairs, over columns already read
}

// One thread's CW columns of S -> P (P over the first CW/2 of the columns it read)
template <bool DIAG>
__device__ __forceinline__ void exp_cols(uint32_t taddr, float2 c2v, int col0, int row) {
#pragma unroll
    for (int c = 0; c < CW; c += 32) exp_store32<DIAG>(taddr + c, taddr + c / 2, c2v, col0 + c, row);
}

template <int DP, int NPAD>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kMfThreads, 1)
    block_av_mf_kernel(const __grid_constant__ CUtensorMap map_xi, const __grid_constant__ CUtensorMap map_xj,
                       const __grid_constant__ CUtensorMap map_ar, const __grid_constant__ CUtensorMap map_ac,
                       const __grid_constant__ CUtensorMap map_v, MfArgs args) {
    using C = MfCfg<DP, NPAD>;
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t xi_full, xi_empty;
    __shared__ __align__(8) uint64_t x_full[C::kXStages], x_empty[C::kXStages];
    __shared__ __align__(8) uint64_t v_full[C::kVStages], v_empty[C::kVStages];
    __shared__ __align__(8) uint64_t s_full[C::kNS], s_empty[C::kNS], p_full[C::kNS];
    __shared__ __align__(8) uint64_t o_full[C::kNO], o_empty[C::kNO];
    __shared__ uint32_t tmem_base_smem;

    const int warp = threadIdx.x / kWarp;
    const int lane = threadIdx.x % kWarp;
    const uint32_t rank = cluster_ctarank();  // 0 = leader (issues the pair's MMAs)
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, P = gridDim.x >> 1;
    const uint32_t base_u32 = (smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t* base = smem_raw + (base_u32 - smem_u32(smem_raw));
    const uint32_t xi_smem = base_u32;                            // X_i | a_i
    const uint32_t xs_smem = xi_smem + C::kFixed;                 // ring of X_j half | a'_j half
    const uint32_t vs_smem = xs_smem + C::kXStages * C::kXSlot;   // ring of V_j halves
    constexpr uint16_t kBoth = 0b11, kLead = 0b01;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&map_xi);
        prefetch_tmap(&map_xj);
        prefetch_tmap(&map_ar);
        prefetch_tmap(&map_ac);
        prefetch_tmap(&map_v);
        mbar_init(&xi_full, 1);
        mbar_init(&xi_empty, 1);
        for (int s = 0; s < C::kXStages; ++s) {
            mbar_init(&x_full[s], 1);
            mbar_init(&x_empty[s], 1);
        }
        for (int s = 0; s < C::kVStages; ++s) {
            mbar_init(&v_full[s], 1);
            mbar_init(&v_empty[s], 1);
        }
        for (int b = 0; b < C::kNS; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&s_empty[b], 1);
            mbar_init(&p_full[b], 2 * kExpWarps);  // one arrival per exp warp of both CTAs
        }
        for (int b = 0; b < C::kNO; ++b) {
            mbar_init(&o_full[b], 1);
            mbar_init(&o_empty[b], 2 * kExpWarps);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc_2sm(&tmem_base_smem, 512);
    tc_fence_before();
    cluster_sync_all();  // both CTAs' barriers initialised and the pair's TMEM allocated
    tc_fence_after();
    const uint32_t tmem = tmem_base_smem;

    if (warp == 0) {
        // ---------------- TMA producer: X_i | a_i (own rows), X_j | a'_j (own half) ----------------
        if (lane == 0) {
            const uint64_t pol = policy_evict_normal();  // the wave re-reads X_j / a'_j from L2 (LRU)
            const uint32_t xi_full_l = mapa_shared(&xi_full, 0);
            int stage = 0;
            uint32_t phase = 0, seg = 0;
            MfSegments sg(args, pair, P);
            int64_t r;
            int j0, j1;
            while (sg.next(r, j0, j1)) {
                const int gi0 = static_cast<int>(args.row0 + (2 * r + rank) * MB);
                mbar_wait(&xi_empty, (seg & 1u) ^ 1u);
                if (leader) mbar_arrive_expect_tx(&xi_full, 2 * C::kFixed);
                for (int h = 0; h < DP / 64; ++h)
                    tma_load_2d_2sm(base + h * C::kXSub, &map_xi, xi_full_l, h * 64, gi0, pol);
                tma_load_2d_2sm(base + C::kXTile, &map_ar, xi_full_l, 0, gi0, pol);
                for (int jb = j0; jb < j1; ++jb) {
                    const int jr = args.global_jb(jb) * JB + static_cast<int>(rank) * (JB / 2);
                    mbar_wait(&x_empty[stage], phase ^ 1u);
                    if (leader) mbar_arrive_expect_tx(&x_full[stage], 2 * C::kXSlot);
                    const uint32_t bar = mapa_shared(&x_full[stage], 0);
                    uint8_t* st = base + (xs_smem - base_u32) + stage * C::kXSlot;
                    for (int h = 0; h < DP / 64; ++h) tma_load_2d_2sm(st + h * C::kXjSub, &map_xj, bar, h * 64, jr, pol);
                    tma_load_2d_2sm(st + C::kXjTile, &map_ac, bar, 0, jr, pol);
                    if (++stage == C::kXStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
                ++seg;
            }
        }
    } else if (warp == 2) {
        // ---------------- TMA producer: V_j, columns [rank·NPAD/2, +NPAD/2) ----------------
        if (lane == 0) {
            const uint64_t pol = policy_evict_normal();
            int stage = 0;
            uint32_t phase = 0;
            MfSegments sg(args, pair, P);
            int64_t r;
            int j0, j1;
            while (sg.next(r, j0, j1)) {
                for (int jb = j0; jb < j1; ++jb) {
                    mbar_wait(&v_empty[stage], phase ^ 1u);
                    if (leader) mbar_arrive_expect_tx(&v_full[stage], 2 * C::kVTile);
                    const uint32_t bar = mapa_shared(&v_full[stage], 0);
                    uint8_t* st = base + (vs_smem - base_u32) + stage * C::kVTile;
                    const int jg = args.global_jb(jb);
                    const int vz = jg / args.kt_chunk, vx = (jg - vz * args.kt_chunk) * JB;
                    for (int h = 0; h < 2; ++h)
                        tma_load_3d_2sm(st + h * C::kVSub, &map_v, bar, vx + h * 64, static_cast<int>(rank) * C::kNH,
                                        vz, pol);
                    if (++stage == C::kVStages) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- S issuer (leader CTA only): S(j) = [X_i|a_i]·[X_j|a'_j]ᵀ ----------------
        // S and P·V are issued from two threads so that neither chain's barrier waits stall the
        // other's MMAs (tcgen05.commit tracks the MMAs of the issuing thread only).
        if (leader && lane == 0) {
            constexpr uint32_t idesc_s = umma_idesc_bf16_f32(2 * MB, JB);
            int xs = 0;
            uint32_t xph = 0, seg = 0, jc = 0;
            MfSegments sg(args, pair, P);
            int64_t r;
            int j0, j1;
            while (sg.next(r, j0, j1)) {
                mbar_wait(&xi_full, seg & 1u);
                tc_fence_after();
                for (int jb = j0; jb < j1; ++jb, ++jc) {
                    const uint32_t sb = jc % C::kNS;
                    MF_STAMP(0, jc)
                    mbar_wait(&s_empty[sb], ((jc / C::kNS) & 1u) ^ 1u);  // P·V of j-3 done with this buffer
                    MF_STAMP(1, jc)
                    mbar_wait(&x_full[xs], xph);
                    MF_STAMP(2, jc)
                    tc_fence_after();
                    const uint32_t xj = xs_smem + xs * C::kXSlot;
                    const uint32_t d = tmem + sb * JB;
#pragma unroll
                    for (int k = 0; k < DP / 16; ++k)
                        umma2_f16(d, umma_desc_sw128(xi_smem + (k >> 2) * C::kXSub + (k & 3) * 32),
                                  umma_desc_sw128(xj + (k >> 2) * C::kXjSub + (k & 3) * 32), idesc_s, k > 0 ? 1u : 0u);
                    umma2_f16(d, umma_desc_kmajor(xi_smem + C::kXTile, 6, 256),
                              umma_desc_kmajor(xj + C::kXjTile, 6, 256), idesc_s, 1u);
                    umma2_commit_mc(&s_full[sb], kBoth);
                    umma2_commit_mc(&x_empty[xs], kBoth);  // X_j halves consumed
                    MF_STAMP(3, jc)
                    if (++xs == C::kXStages) {
                        xs = 0;
                        xph ^= 1u;
                    }
                }
                umma2_commit_mc(&xi_empty, kBoth);  // X_i free after the segment's S MMAs
                ++seg;
            }
        }
    } else if (warp == 3) {
        // ---------------- P·V issuer (leader CTA only): O += P(j)·V_j ----------------
        if (leader && lane == 0) {
            constexpr uint32_t idesc_o = umma_idesc_f16_f32(2 * MB, NPAD);
            int vs = 0;
            uint32_t vph = 0, jc = 0, chunk = 0;
            MfSegments sg(args, pair, P);
            int64_t r;
            int j0, j1;
            while (sg.next(r, j0, j1)) {
                uint32_t in_chunk = 0;
                for (int jb = j0; jb < j1; ++jb, ++jc) {
                    const uint32_t pb = jc % C::kNS;
                    const uint32_t ob = chunk % C::kNO;
                    MF_STAMP(4, jc)
                    if (in_chunk == 0) mbar_wait(&o_empty[ob], ((chunk / C::kNO) & 1u) ^ 1u);
                    mbar_wait(&v_full[vs], vph);
                    MF_STAMP(5, jc)
                    mbar_wait(&p_full[pb], (jc / C::kNS) & 1u);
                    MF_STAMP(6, jc)
                    tc_fence_after();
                    const uint32_t d = tmem + C::kOCol + ob * NPAD;
                    // P of exp group g (K in [g·CW, (g+1)·CW)) sits at columns [g·CW, g·CW + CW/2)
                    const uint32_t pa = tmem + pb * JB;
                    const uint32_t vb = vs_smem + vs * C::kVTile;
#pragma unroll
                    for (int k = 0; k < JB / 16; ++k)
                        umma2_f16_ts(d, pa + (k / (CW / 16)) * CW + (k % (CW / 16)) * 8,
                                     umma_desc_sw128(vb + (k >> 2) * C::kVSub + (k & 3) * 32), idesc_o,
                                     (in_chunk > 0 || k > 0) ? 1u : 0u);
                    umma2_commit_mc(&s_empty[pb], kLead);  // S/P buffer reusable
                    umma2_commit_mc(&v_empty[vs], kBoth);  // V_j halves consumed
                    MF_STAMP(7, jc)
                    if (++vs == C::kVStages) {
                        vs = 0;
                        vph ^= 1u;
                    }
                    if (++in_chunk == static_cast<uint32_t>(args.kc) || jb + 1 == j1) {
                        umma2_commit_mc(&o_full[ob], kBoth);
                        ++chunk;
                        in_chunk = 0;
                    }
                }
            }
        }
    } else if (warp >= 4) {
        // ---------------- exp + O drain: two warpgroups, columns [64h, 64h+64) of S ----------------
        // Each thread owns one row (its TMEM lane) and half of the j-block's columns; it writes its
        // P values back over the S columns it has just read (so the two halves never race) and
        // drains half of the O columns into fp32 registers, lazily one j-block after the chunk
        // closes so the exp work of the next j-block overlaps the chunk's last P·V.
        const int h = (warp - 4) >> 2;  // exp warpgroup: S columns [h·CW, (h+1)·CW), O columns [h·OW, (h+1)·OW)
        const int q = warp & 3;  // TMEM lane quarter
        const int row = q * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        const float2 c2v = make_float2(args.c2, args.c2);
        float acc[C::kOW];
#pragma unroll
        for (int j = 0; j < C::kOW; ++j) acc[j] = 0.f;
        auto drain = [&](uint32_t c) {
            const uint32_t ob = c % C::kNO;
            mbar_wait(&o_full[ob], (c / C::kNO) & 1u);
            tc_fence_after();
            const uint32_t t0 = tmem + lane_off + C::kOCol + ob * NPAD + h * C::kOW;
            constexpr int n16 = C::kOW / 16, r8 = (C::kOW % 16) / 8, r4 = (C::kOW % 8) / 4;
#pragma unroll
            for (int j0 = 0; j0 < 16 * n16; j0 += 16) {
                float m[16];
                tmem_ld16(t0 + j0, m);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 16; ++i) acc[j0 + i] += m[i];
            }
            if constexpr (r8) {
                float m[8];
                tmem_ld8(t0 + 16 * n16, m);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 8; ++i) acc[16 * n16 + i] += m[i];
            }
            if constexpr (r4) {
                float m[4];
                tmem_ld4(t0 + 16 * n16 + 8 * r8, m);
                tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 4; ++i) acc[16 * n16 + 8 * r8 + i] += m[i];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(&o_empty[ob], 0));
        };
        uint32_t jc = 0, chunk = 0;
        MfSegments sg(args, pair, P);
        int64_t r;
        int j0, j1;
        while (sg.next(r, j0, j1)) {
            const int64_t diag_jb = (args.row0 + (2 * r + rank) * MB) / JB;  // blocks start at multiples of 128
            uint32_t in_chunk = 0, pend = 0;
            bool pending = false;
            for (int jb = j0; jb < j1; ++jb, ++jc) {
                const uint32_t sb = jc % C::kNS;
                if (warp == 4 && lane == 0) { MF_STAMP(8, jc) }
                mbar_wait(&s_full[sb], (jc / C::kNS) & 1u);
                if (warp == 4 && lane == 0) { MF_STAMP(9, jc) }
                tc_fence_after();
                const uint32_t taddr = tmem + lane_off + sb * JB + h * CW;
                if (args.global_jb(jb) == diag_jb)
                    exp_cols<true>(taddr, c2v, h * CW, row);
                else
                    exp_cols<false>(taddr, c2v, h * CW, row);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(mapa_shared(&p_full[sb], 0));
                if (warp == 4 && lane == 0) { MF_STAMP(10, jc) }
                if (pending) {  // chunk closed one j-block ago; its last P·V has had time to finish
                    drain(pend);
                    pending = false;
                }
                if (++in_chunk == static_cast<uint32_t>(args.kc) || jb + 1 == j1) {
                    if (jb + 1 == j1) {
                        drain(chunk);
                    } else {
                        pending = true;
                        pend = chunk;
                    }
                    ++chunk;
                    in_chunk = 0;
                }
            }
            const int64_t slot = sg.slot(r, rank);
            float* dst = args.partial + (slot * NPAD + h * C::kOW) * MB + row;
#pragma unroll
            for (int j = 0; j < C::kOW; ++j) {
                dst[j * MB] = acc[j];
                acc[j] = 0.f;
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer is done with the pair's TMEM and barriers
    if (warp == 1) tmem_dealloc_2sm(tmem, 512);
}

template <int DP, int NPAD>
cudaError_t launch_mf(const MfMatrixView& a, const SplitPanelView& v, const StreamKPlan& plan, float* partial,
                      cudaStream_t stream) {
    using C = MfCfg<DP, NPAD>;
    TensorMapEncodeFn enc = tensor_map_encoder();
    if (!enc) return cudaErrorInvalidValue;
    if (v.rpr % JB != 0) return cudaErrorInvalidValue;
    CUtensorMap mxi, mxj, mar, mac, mv;
    const cuuint32_t estr[3] = {1, 1, 1};
    for (int t = 0; t < 2; ++t) {
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.dp), static_cast<cuuint64_t>(a.n)};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.dp) * 2};
        cuuint32_t box[2] = {64, t == 0 ? static_cast<cuuint32_t>(MB) : static_cast<cuuint32_t>(JB / 2)};
        if (enc(t == 0 ? &mxi : &mxj, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<__nv_bfloat16*>(a.x), dims,
                strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    for (int side = 0; side < 2; ++side) {
        cuuint64_t dims[2] = {kAug, static_cast<cuuint64_t>(a.npad)};
        cuuint64_t strides[1] = {kAug * 2};
        cuuint32_t box[2] = {kAug, side == 0 ? static_cast<cuuint32_t>(MB) : static_cast<cuuint32_t>(JB / 2)};
        if (enc(side == 0 ? &mar : &mac, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                const_cast<__nv_bfloat16*>(a.xa) + static_cast<size_t>(side) * a.npad * kAug, dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    {
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(v.rpr), static_cast<cuuint64_t>(v.cols),
                              static_cast<cuuint64_t>(v.world)};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(v.rpr) * 2,
                                 static_cast<cuuint64_t>(v.slice ? v.slice : v.rpr * v.cols) * 2};
        cuuint32_t box[3] = {64, static_cast<cuuint32_t>(C::kNH), 1};
        if (enc(&mv, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<__half*>(v.v), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return cudaErrorInvalidValue;
    }
    if (cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(block_av_mf_kernel<DP, NPAD>), C::kSmem);
        e != cudaSuccess)
        return e;
    MfArgs args;
    args.total_iters = plan.total_iters;
    args.j_blocks = plan.k_tiles;
    args.j_off = plan.k_off;
    args.j_total = plan.k_total > 0 ? plan.k_total : plan.k_tiles;
    args.kc = plan.kc;
    args.row0 = a.row0;
    args.kt_chunk = static_cast<int>(v.rpr / JB);
    args.c2 = static_cast<float>(a.c2);
    args.dp_blocks = plan.dp_blocks;
    args.partial = partial;
    args.trace = nullptr;
#ifdef RB_MF_TRACE
    static unsigned long long* trace = nullptr;
    if (!trace) cudaMalloc(&trace, 256 * 16 * 8);
    cudaMemsetAsync(trace, 0, 256 * 16 * 8, stream);
    args.trace = trace;
#endif
    block_av_mf_kernel<DP, NPAD><<<2 * plan.grid, kMfThreads, C::kSmem, stream>>>(mxi, mxj, mar, mac, mv, args);
#ifdef RB_MF_TRACE
    if (NPAD == 128) {
        cudaStreamSynchronize(stream);
        static unsigned long long h[256 * 16];
        cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
        const unsigned long long t0 = h[100 * 16];
        for (int j = 100; j < 116; ++j) {
            fprintf(stderr, "j=%3d", j);
            for (int k = 0; k < 15; ++k) fprintf(stderr, " %7lld", static_cast<long long>(h[j * 16 + k] - t0));
            fprintf(stderr, "\n");
        }
    }
#endif
    return cudaGetLastError();
}

// x (fp64) -> bf16 samples [n][dp] and the augmented columns [2][npad][16]:
// row side a = [h, m, l, 1, 1, 1, 0…], column side a' = [1, 1, 1, h, m, l, 0…], h + m + l = −|bf16(x)|²/2
__global__ void mf_prepare_kernel(const double* __restrict__ x, int64_t n, int d, int64_t rs, int64_t cs, int dp,
                                  int64_t npad, __nv_bfloat16* __restrict__ xb, __nv_bfloat16* __restrict__ xa) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double sq = 0.0;
    for (int k = 0; k < dp; ++k) {
        const __nv_bfloat16 v = __float2bfloat16_rn(k < d ? static_cast<float>(x[i * rs + k * cs]) : 0.f);
        xb[i * dp + k] = v;
        const double f = static_cast<double>(__bfloat162float(v));
        sq += f * f;
    }
    double v = -0.5 * sq;
    __nv_bfloat16 part[3];
    for (int t = 0; t < 3; ++t) {
        part[t] = __double2bfloat16(v);
        v -= static_cast<double>(__bfloat162float(part[t]));
    }
    const __nv_bfloat16 one = __float2bfloat16_rn(1.f), zero = __float2bfloat16_rn(0.f);
    __nv_bfloat16* ar = xa + i * kAug;
    __nv_bfloat16* ac = xa + (npad + i) * kAug;
    for (int k = 0; k < kAug; ++k) {
        ar[k] = k < 3 ? part[k] : (k < 6 ? one : zero);
        ac[k] = k < 3 ? one : (k < 6 ? part[k - 3] : zero);
    }
}

}  // namespace

StreamKPlan make_mf_plan(int64_t rows, int64_t n, int grid, int kc, KWindow w) {
    // CTA pairs over 256-row blocks; the epilogue reads 128-row blocks with cluster = 2
    StreamKPlan p;
    const int64_t pair_blocks = (rows + 2 * MB - 1) / (2 * MB);
    p.row_blocks = static_cast<int>((rows + MB - 1) / MB);
    apply_window(p, n, JB, w);  // k tiles = j-blocks
    p.total_iters = pair_blocks * p.k_tiles;
    int pairs = std::max(1, grid / 2);
    if (p.total_iters < pairs) pairs = static_cast<int>(p.total_iters > 0 ? p.total_iters : 1);
    p.grid = pairs;
    p.kc = kc;
    p.cluster = 2;
    p.slots = static_cast<int>(2 * (pair_blocks + pairs));
    p.rows_per_block = MB;
    p.dp_blocks = static_cast<int>((pair_blocks / pairs) * pairs);  // whole waves; the remainder goes stream-K
    return p;
}

int mf_aug_cols() { return kAug; }

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

cudaError_t launch_mf_prepare(const double* x, int64_t n, int d, int64_t rs, int64_t cs, int dp, int64_t npad,
                              __nv_bfloat16* xb, __nv_bfloat16* xa, cudaStream_t stream) {
    if (n <= 0) return cudaSuccess;
    mf_prepare_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(x, n, d, rs, cs, dp, npad, xb, xa);
    return cudaGetLastError();
}

}  // namespace rb
