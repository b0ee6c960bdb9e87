// efta_attn_pair.cuh — CTA-pair (cta_group::2) variant of the fused EFTA forward.
//
// Why a pair: with one 128-row query tile per SM, every SM streams the full K_j / V_j
// tiles of its head from L2 each block. A cluster of two CTAs on one TPC computes an
// M=256 tile with tcgen05.mma.cta_group::2: each CTA keeps its own 128 query rows (A)
// and holds only HALF of each B operand in its shared memory, so per-SM ingress halves.
//
// B-operand split (CUTLASS 2x1SM traits: CTA v owns B rows [v*N/2, (v+1)*N/2)):
//   S  = Q . [K_j ; KC1_j]^T  N = 128 (+16): leader K rows 0..63 (0..71),
//                                             peer   K rows 64..127 (72..127 + c1_hi, c1_lo)
//        Only the c1 checksum rows (hi/lo) ride in the score MMA; c2, needed only to locate
//        a fault once c1 flagged one, is recomputed on the CUDA cores in the rare path
//        (pair_score_c2), so the checksum MMA work is +12.5% instead of +25%.
//   O += P . [V_j | VC_j]    N = d (+32), B = [V_j^T ; VC_j^T] K-major (keys contiguous),
//                            written by the encode prepass; each CTA loads (d+32)/2 rows.
//
// TMEM (512 columns): S[0] | S[1] (SW = 144 / 128 each) | O (d + 32 / d) | P (64, fp16x2).
// P has its own buffer, so the score MMA of block j+2 can overwrite S[j&1] as soon as the
// row warpgroup has read S_j (s_free), long before P.V of block j ran: the two row
// warpgroups of the alternating schedule (efta_attn_alt.cuh) then never wait for scores.
// With one P buffer per warpgroup (when TMEM allows) block j's P only waits for P.V(j-2);
// the protected d=128 layout shares one buffer: block j's P is stored after P.V(j-1).
//
// The leader (cluster rank 0) issues every MMA and multicasts its commits to both CTAs'
// barriers; both CTAs' TMA loads signal the leader's full barriers; both CTAs' row
// warpgroups signal the leader's s_free / p_ready barriers.
#pragma once
#include "efta_attn_kernel.cuh"

#ifndef EFTA_TMA_STORE_D128
#define EFTA_TMA_STORE_D128 0  // d=128 O store through 16-row TMA boxes (A/B variant, default off)
#endif

namespace efta_sm100 {

template <int D, bool PROT>
struct PairLayout {
    static constexpr int NSUB = D / 64;
    static constexpr int SW = PROT ? 144 : 128;          // score MMA N (TMEM columns per S buffer)
    static constexpr int HN_S = SW / 2;                  // B rows per CTA, scores
    static constexpr int VROWS = PROT ? D + 32 : D;      // rows of the V^T (+VC^T) operand = O columns
    static constexpr int HN_V = VROWS / 2;               // B rows per CTA, P.V
    // 4-stage K / V rings, 3 where the double-buffered Q would not fit (protected d=128)
    // unprotected d=64: 6 stages (A/B: +2-3% at S=2048 / 512; the protected d=64 kernel is row-bound
    // and measured -0.3% / +-0 with 6, profiles/r02/s3/ab_ring_d64.log)
    static constexpr int KS = (D == 128 && PROT) ? 3 : ((D == 64 && !PROT) ? 6 : 4), VS = KS;
    static constexpr uint32_t Q_BYTES = NSUB * 16384;  // one Q buffer (two: the next tile's Q loads early)
    static constexpr uint32_t K_CHUNK = HN_S * 128;      // one 64-column chunk of the K half
    static constexpr uint32_t K_STAGE = NSUB * K_CHUNK;
    static constexpr uint32_t V_CHUNK = HN_V * 128;      // one 64-key chunk of the V^T half
    static constexpr uint32_t V_STAGE = 2 * V_CHUNK;
    static constexpr uint32_t OFF_Q = 0;
    static constexpr uint32_t OFF_K = OFF_Q + 2 * Q_BYTES;
    static constexpr uint32_t OFF_V = OFF_K + KS * K_STAGE;
    static constexpr uint32_t OFF_BAR = OFF_V + VS * V_STAGE;
    // q_full, k_full/empty[KS], v_full/empty[VS], s_full[2], s_free[2], p_ready[2],
    // o_done[2], o_final, chain barriers mx_early[2 tile parity][2][4], mx_late[2][2][4], q_empty[2],
    // o_free, fin[2][4], second q_full, tile ring full[4] / empty[4], tile-boundary ack[2][4]
    static constexpr int NBAR = 1 + 2 * KS + 2 * VS + 2 + 2 + 2 + 2 + 1 + 32 + 2 + 1 + 8 + 1 + 8 + 8;
    static constexpr uint32_t OFF_TMEM = OFF_BAR + NBAR * 8;
    static constexpr uint32_t OFF_RED = (OFF_TMEM + 16 + 15) & ~15u;
    static constexpr uint32_t RED_BYTES = 128 * 24 + 256;  // per row warpgroup
    static constexpr uint32_t OFF_XCH = OFF_RED + 2 * RED_BYTES;
    static constexpr uint32_t OFF_TINFO = OFF_XCH + 2 * 7168;  // chain exchange x tile parity; tile ring: int[4]
    // epilogue O staging: d=64 holds each warp's 32 output rows (8 KB, 128-byte swizzle) for an
    // asynchronous TMA store; d=128 stages 16-row boxes through two (protected) or one 2 KB
    // buffer per warp (what the K / V rings leave)
    // (the d=128 TMA variant, EFTA_TMA_STORE_D128=1, needs 1 KB-aligned buffers: two per warp
    // protected, one unprotected; the default d=128 build keeps the coalesced path's 2 KB per warp)
    static constexpr bool kTma = D == 64 || EFTA_TMA_STORE_D128 != 0;
    static constexpr int OBUF_N = D == 64 ? 4 : ((EFTA_TMA_STORE_D128 != 0 && PROT) ? 2 : 1);  // per warp: 2 KB buffers
    static constexpr uint32_t OSTG_BYTES = 4 * 2048 * OBUF_N;
    static constexpr uint32_t OFF_OSTG = kTma ? ((OFF_TINFO + 16 + 1023) & ~1023u) : OFF_TINFO + 16;
    static constexpr uint32_t SMEM_BYTES = OFF_OSTG + OSTG_BYTES + 1024;
    // TMEM columns
    static constexpr uint32_t COL_S0 = 0, COL_O = 2 * SW, COL_P = COL_O + VROWS, TMEM_COLS = 512;
    // one P buffer per row warpgroup when it fits (unprotected d=128, every d=64 variant);
    // protected d=128 (2*144 + 160 + 64 = 512) shares one
    static constexpr int NPB = (COL_P + 128 <= TMEM_COLS) ? 2 : 1;
    static_assert(COL_P + 64 * NPB <= TMEM_COLS, "TMEM budget");
    static_assert(K_CHUNK % 1024 == 0 && V_CHUNK % 1024 == 0, "swizzle atoms must stay 1 KB aligned");
    static_assert(RED_BYTES == AttnLayout<D>::RED_BYTES, "row scratch size");
    static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
};
constexpr int kPairThreads = 384;  // warps 0-3: TMA K / score MMA / P.V MMA / TMA Q,V; 4-7, 8-11: row warpgroups

// ---- dynamic tile schedule: an in-order atomic tile counter, fetched one tile ahead by the
// leader's Q/V producer and broadcast to both CTAs through a 4-slot ring (keeps the set of
// heads in flight compact, so the K/V blocks of a head are read from HBM once: a static
// round-robin schedule lets clusters drift apart and spread over more heads than L2 holds)
constexpr int kTileRing = 4;
constexpr int kTileConsumers = 21;  // leader warps 0,1,2,4-11 + peer warps 0,3,4-11
__device__ __forceinline__ void st_cluster_s32(const void* smem_local, uint32_t cta, int v) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\tst.shared::cluster.s32 [ra], %2;\n\t}" ::"r"(
            smem_u32(smem_local)),
        "r"(cta), "r"(v)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_rel_cluster(uint64_t* bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
        "r"(cta)
        : "memory");
}
// consumer release of a tile-ring slot: relaxed (a release at cluster scope costs a GPU-scope
// MEMBAR + ERRBAR per warp and tile; the slot's value is already in a register, and the
// producer rewrites the slot only kTileRing tiles later)
__device__ __forceinline__ void mbar_arrive_relaxed_cluster(uint64_t* bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
        "r"(cta)
        : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
// consumer side: tile of this cluster's k-th step (-1: done); one arrival per calling warp
__device__ __forceinline__ int pair_next_tile(const int* tinfo, uint64_t* tfull, uint64_t* tempty, int k,
                                              bool warp_wide) {
    const int slot = k & (kTileRing - 1);
    mbar_wait_acq_cluster(&tfull[slot], static_cast<uint32_t>(k / kTileRing) & 1u);
    const int u = *reinterpret_cast<const volatile int*>(&tinfo[slot]);
    if (warp_wide) __syncwarp();
    if (!warp_wide || (threadIdx.x & 31) == 0) mbar_arrive_relaxed_cluster(&tempty[slot], 0);
    return u;
}

}  // namespace efta_sm100

#include "efta_attn_alt.cuh"

namespace efta_sm100 {

// tm_ka: K rows [0, HN_S) (or [64r, 64r+64) unprotected), tm_kb: K rows 72..127 (protected),
// tm_kc: KC rows in 8-row boxes (protected), tm_vt: [V^T ; VC^T] rows of each block, box rows HN_V.
// INJ: the fault-tap build (reference op sequence, eager rescale, taps at every FaultSite;
// efta_attn_alt.cuh) — the `debug` variant of the same schedule.
template <int D, int MODE, bool INJ, bool CAUSAL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
efta_attn_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_ka,
                      const __grid_constant__ CUtensorMap tm_kb, const __grid_constant__ CUtensorMap tm_kc,
                      const __grid_constant__ CUtensorMap tm_vt, const __grid_constant__ CUtensorMap tm_o,
                      const AttnParams p) {
    constexpr bool PROT = MODE != EFTA_MODE_NONE;
    using L = PairLayout<D, PROT>;
    constexpr int KS = L::KS, VS = L::VS, NSUB = L::NSUB;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = k_full + KS;
    uint64_t* v_full = k_empty + KS;
    uint64_t* v_empty = v_full + VS;
    uint64_t* s_full = v_empty + VS;   // [2] by block parity
    uint64_t* s_free = s_full + 2;     // [2] row warpgroup w has read S_j (leader)
    uint64_t* p_ready = s_free + 2;    // [2] P_j stored / O rescaled (leader)
    uint64_t* o_done = p_ready + 2;    // [2] P.V of block j complete
    uint64_t* o_final = o_done + 2;
    uint64_t* mx_early = o_final + 1;  // [tile parity][warpgroup][warp quarter]
    uint64_t* mx_late = mx_early + 16; // [2][2][4]
    uint64_t* q_empty = mx_late + 16;  // [2] every score MMA of the tile using Q buffer b done
    uint64_t* o_free = q_empty + 2;    // the epilogue read O (leader; 4 warps x 2 CTAs)
    uint64_t* fin_bar = o_free + 1;    // [tile parity][4] warpgroup 0's sums of the tile (per warp quarter)
    uint64_t* q_full2 = fin_bar + 8;   // q_full of Q buffer 1 (q_full is buffer 0's)
    uint64_t* t_full = q_full2 + 1;    // [4] tile ring slot published (this CTA)
    uint64_t* t_empty = t_full + 4;    // [4] tile ring slot consumed by all 21 warps (leader)
    uint64_t* ack_bar = t_empty + 4;   // [tile parity][4] warpgroup 1 consumed the tile's chain / fin slots
    int* tinfo = reinterpret_cast<int*>(smem + L::OFF_TINFO);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

    const int warp = warp_id(), lane = lane_id();
    const uint32_t rank = cluster_rank();
    const int n = p.nblk;
    // persistent clusters: tile u = (head, query pair), handed out in order by an atomic counter
    const int npq = n / 2, total = p.n_heads_flat * npq;
    int* tile_counter = reinterpret_cast<int*>(p.scratch);  // zeroed by the host before the launch

    if (warp == 0 && lane == 0) {
        mbar_init(q_full, 1);
        for (int s = 0; s < KS; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
        for (int s = 0; s < VS; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&s_full[b], 1);
            mbar_init(&s_free[b], 8);   // 4 row warps x 2 CTAs
            mbar_init(&p_ready[b], 8);
            mbar_init(&o_done[b], 1);
        }
        mbar_init(o_final, 1);
        for (int i = 0; i < 32; ++i) mbar_init(&mx_early[i], 32);  // early and late, both parities
        mbar_init(&q_empty[0], 1);
        mbar_init(&q_empty[1], 1);
        mbar_init(q_full2, 1);
        for (int i = 0; i < kTileRing; ++i) { mbar_init(&t_full[i], 1); mbar_init(&t_empty[i], kTileConsumers); }
        mbar_init(o_free, 8);
        for (int i = 0; i < 8; ++i) { mbar_init(&fin_bar[i], 32); mbar_init(&ack_bar[i], 32); }
        fence_barrier_init();
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_ka);
        tma_prefetch_desc(&tm_vt);
        if (PROT) { tma_prefetch_desc(&tm_kb); tma_prefetch_desc(&tm_kc); }
    }
    if (warp == 1) tmem_alloc2(tmem_slot, L::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / TMA
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t q_smem = smem_u32(smem + L::OFF_Q);
    const uint32_t k_smem = smem_u32(smem + L::OFF_K);
    const uint32_t v_smem = smem_u32(smem + L::OFF_V);

    if (warp == 0) {
        // -------------------------------------------------------- K (+KC1) half producer
        setmaxnreg_dec<40>();
        if (lane == 0) {
            int g = 0;
            for (int k = 0;; ++k) {
                const int u = pair_next_tile(tinfo, t_full, t_empty, k, false);
                if (u < 0) break;
                const PairTile tt = pair_tile<CAUSAL>(p, u);
                const int head = tt.head;
                const int kvh = kv_head(p, head);  // GQA: the K / checksum operands of the head's group
                const int seq_row0 = kvh * p.seq_len;
                for (int j = 0; j < tt.nblk; ++j, ++g) {
                    const int s = g % KS;
                    mbar_wait(&k_empty[s], ((g / KS) & 1) ^ 1);
                    uint8_t* dst = smem + L::OFF_K + s * L::K_STAGE;
                    if (rank == 0) mbar_arrive_expect_tx(&k_full[s], 2 * L::K_STAGE);
                    const int krow = seq_row0 + j * kBlock;
                    const int crow = (kvh * n + j) * 32;
#pragma unroll
                    for (int sub = 0; sub < NSUB; ++sub) {
                        uint8_t* c = dst + sub * L::K_CHUNK;
                        if (!PROT) {
                            tma_load_2d_pair(c, &tm_ka, &k_full[s], sub * 64, krow + 64 * rank, kEvictLast);
                        } else if (rank == 0) {
                            tma_load_2d_pair(c, &tm_ka, &k_full[s], sub * 64, krow, kEvictLast);
                        } else {
                            tma_load_2d_pair(c, &tm_kb, &k_full[s], sub * 64, krow + 72, kEvictLast);
                            tma_load_2d_pair(c + 56 * 128, &tm_kc, &k_full[s], sub * 64, crow, kEvictLast);  // c1_hi
                            tma_load_2d_pair(c + 64 * 128, &tm_kc, &k_full[s], sub * 64, crow + 16,
                                             kEvictLast);  // c1_lo
                        }
                    }
                }
            }
        }
    } else if (warp == 3) {
        // -------------------------------------------------------- Q, V^T (+VC^T) half producer
        setmaxnreg_dec<40>();
        if (lane == 0) {
            // leader: fetch tiles in order, one ahead, and publish them to both CTAs
            auto publish = [&](int k, int u) {
                const int slot = k & (kTileRing - 1);
                mbar_wait_acq_cluster(&t_empty[slot], (static_cast<uint32_t>(k / kTileRing) & 1u) ^ 1u);
                tinfo[slot] = u;
                st_cluster_s32(&tinfo[slot], 1, u);
                mbar_arrive_rel_cluster(&t_full[slot], 0);
                mbar_arrive_rel_cluster(&t_full[slot], 1);
            };
            auto fetch = [&]() {
                const int u = atomicAdd(tile_counter, 1);
                return u < total ? u : -1;
            };
            int u_next = 0;
            if (rank == 0) {
                u_next = fetch();
                publish(0, u_next);
            }
            int g = 0;
            for (int k = 0;; ++k) {
                int u;
                if (rank == 0) {
                    u = u_next;
                    if (u < 0) break;
                    u_next = fetch();
                    publish(k + 1, u_next);
                } else {
                    u = pair_next_tile(tinfo, t_full, t_empty, k, false);
                    if (u < 0) break;
                }
                const PairTile tt = pair_tile<CAUSAL>(p, u);
                const int head = tt.head, qt = 2 * tt.pair + static_cast<int>(rank);
                const int seq_row0 = head * p.seq_len;
                // Q buffer k&1 was last read by the score MMAs of tile k-2
                const int qb = k & 1;
                uint64_t* qf = qb ? q_full2 : q_full;
                if (k >= 2) mbar_wait(&q_empty[qb], ((k - 2) >> 1) & 1);
                if (rank == 0) mbar_arrive_expect_tx(qf, 2 * L::Q_BYTES);
#pragma unroll
                for (int sub = 0; sub < NSUB; ++sub)
                    tma_load_2d_pair(smem + L::OFF_Q + qb * L::Q_BYTES + sub * 16384, &tm_q, qf, sub * 64,
                                     seq_row0 + qt * kBlock, kEvictFirst);
                for (int j = 0; j < tt.nblk; ++j, ++g) {
                    const int s = g % VS;
                    mbar_wait(&v_empty[s], ((g / VS) & 1) ^ 1);
                    uint8_t* dst = smem + L::OFF_V + s * L::V_STAGE;
                    if (rank == 0) mbar_arrive_expect_tx(&v_full[s], 2 * L::V_STAGE);
                    const int vrow = (kv_head(p, head) * n + j) * L::VROWS + L::HN_V * rank;
#pragma unroll
                    for (int c = 0; c < 2; ++c)
                        tma_load_2d_pair(dst + c * L::V_CHUNK, &tm_vt, &v_full[s], c * 64, vrow, kEvictLast);
                }
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- score MMA issuer (pair leader)
        // S_j = Q . [K_j ; KC1_j]^T into S[j&1]; S_{j+2} once both CTAs' warpgroup read S_j.
        // Two issuer threads: a single one idles the tensor pipe while it waits on the
        // other operand's barriers (the tcgen05 queue is shallow, tools/mma2_bench.cu).
        setmaxnreg_dec<40>();
        if (rank == 0) {  // the whole warp runs the loop; one elected lane issues
            constexpr uint32_t ID_S = idesc_f16_f32(256, L::SW, 0, 0);
            const uint64_t dq = smem_desc_sw128(q_smem, 16, 1024);
            const uint64_t dk0 = smem_desc_sw128(k_smem, 16, 1024);
            int g = 0;
            for (int k = 0;; ++k) {
                const int u = pair_next_tile(tinfo, t_full, t_empty, k, true);
                if (u < 0) break;
                const int nb = pair_tile<CAUSAL>(p, u).nblk;
                const int qb = k & 1;
                mbar_wait(qb ? q_full2 : q_full, (k >> 1) & 1);
                tc_fence_after();
                const uint64_t dqb = dq + ((qb * L::Q_BYTES) >> 4);
                for (int j = 0; j < nb; ++j, ++g) {
                    if (g >= 2) {
                        mbar_wait(&s_free[g & 1], ((g - 2) >> 1) & 1);
                        EFTA_TS(7, g - 2);
                    }
                    const int s = g % KS;
                    mbar_wait(&k_full[s], (g / KS) & 1);
                    tc_fence_after();
                    const uint64_t dk = dk0 + ((s * L::K_STAGE) >> 4);
                    const uint32_t d_s = tmem + L::COL_S0 + (g & 1) * L::SW;
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            const uint32_t offq = (kk >> 2) * 16384 + (kk & 3) * 32;
                            const uint32_t offk = (kk >> 2) * L::K_CHUNK + (kk & 3) * 32;
                            mma2_ss(d_s, dqb + (offq >> 4), dk + (offk >> 4), ID_S, kk > 0);
                        }
                        commit2_both(&k_empty[s]);
                        commit2_both(&s_full[g & 1]);
                        if (j == nb - 1) commit2_both(&q_empty[qb]);
                    }
                    __syncwarp();
                    EFTA_TS(11, g - 2);
                }
            }
        }
    } else if (warp == 2) {
        // -------------------------------------------------------- P.V MMA issuer (pair leader)
        setmaxnreg_dec<40>();
        if (rank == 0) {
            constexpr uint32_t ID_PV = idesc_f16_f32(256, L::VROWS, 0, 0);
            const uint64_t dv0 = smem_desc_sw128(v_smem, 16, 1024);
            const uint32_t d_o = tmem + L::COL_O;
            int g = 0;
            for (int k = 0;; ++k) {
                const int u = pair_next_tile(tinfo, t_full, t_empty, k, true);
                if (u < 0) break;
                const int nb = pair_tile<CAUSAL>(p, u).nblk;
                for (int j = 0; j < nb; ++j, ++g) {
                    EFTA_TS(10, g);
                    mbar_wait(&p_ready[g & 1], (g >> 1) & 1);
                    EFTA_TS(12, g);
                    tc_fence_after();
                    const int s = g % VS;
                    mbar_wait(&v_full[s], (g / VS) & 1);
                    EFTA_TS(14, g);
                    if (j == 0 && k > 0) mbar_wait(o_free, (k - 1) & 1);  // the last epilogue read O
                    tc_fence_after();
                    const uint64_t dv = dv0 + ((s * L::V_STAGE) >> 4);
                    const uint32_t a_p = tmem + L::COL_P + (L::NPB == 2 ? (g & 1) * 64 : 0);
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < kBlock / 16; ++kk) {
                            const uint32_t offv = (kk >> 2) * L::V_CHUNK + (kk & 3) * 32;
                            mma2_ts(d_o, a_p + kk * 8, dv + (offv >> 4), ID_PV, (j > 0 || kk > 0) ? 1u : 0u);
                        }
                        commit2_both(&v_empty[s]);
                        commit2_both(&o_done[g & 1]);
                        if (j == nb - 1) commit2_both(o_final);
                    }
                    __syncwarp();
                    EFTA_TS(13, g);
                }
            }
        }
        __syncwarp();
    } else {
        setmaxnreg_inc<232>();
        row_alt<D, PROT, INJ, CAUSAL>(p, smem + L::OFF_RED, reinterpret_cast<AltXch*>(smem + L::OFF_XCH),
                              reinterpret_cast<float*>(smem + L::OFF_OSTG), &tm_o, s_full,
                              s_free, p_ready, o_done, o_final, mx_early, mx_late, fin_bar, ack_bar, o_free, tmem,
                              warp, lane, n, tinfo, t_full, t_empty, rank);
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer may still be reading our shared memory / TMEM via the MMAs
    tc_fence_after();
    if (warp == 1) tmem_dealloc2(tmem, L::TMEM_COLS);
}

// Prepass for the pair kernel: KC (as before) + [V_j^T ; VC_j^T] per (head, block):
//   VT[(head*n + j) * VROWS + r][key] = V[j*128 + key][r]                         r < D
//   VT[(head*n + j) * VROWS + D + x / 8+x / 16+x / 24+x][key] = c1_hi / c2_hi / c1_lo / c2_lo
// HBM-bound: every global access is a 16-byte vector (8 halves), V is transposed through
// shared memory, the strided sums run in fp32 in ascending l / g (the reference order).
template <int D, bool PROT>
__global__ void __launch_bounds__(256) efta_encode_pair_kernel(const __half* __restrict__ k,
                                                               const __half* __restrict__ v,
                                                               __half* __restrict__ kc, __half* __restrict__ vt,
                                                               int seq_len, int nblk) {
    constexpr int VROWS = PROT ? D + 32 : D;
    constexpr int G_O = D / 8;
    // V block in shared memory, row `key` at key*SP + (key/8)*8 halves: 16-byte aligned rows, and
    // the column reads of the transpose (keys 8 apart across a warp) spread over 8 banks
    constexpr int SP = D + 8;
    __shared__ __align__(16) __half sv[128 * SP + 16 * 8];
    auto sidx = [](int key, int c) { return key * SP + (key >> 3) * 8 + c; };
    const int j = blockIdx.x, head = blockIdx.y;
    const size_t row0 = static_cast<size_t>(head) * seq_len + static_cast<size_t>(j) * 128;
    for (int idx = threadIdx.x; idx < 128 * D / 8; idx += blockDim.x) {
        const int r = idx / (D / 8), c8 = idx % (D / 8);
        *reinterpret_cast<uint4*>(&sv[sidx(r, c8 * 8)]) = reinterpret_cast<const uint4*>(v + (row0 + r) * D)[c8];
    }
    if (PROT) {
        // KC rows: thread = (group x, 8 consecutive dims); 16 vector loads of K rows x + 8l
        const size_t crow0 = (static_cast<size_t>(head) * nblk + j) * 32;
        for (int t = threadIdx.x; t < 8 * (D / 8); t += blockDim.x) {
            const int x = t / (D / 8), d8 = t % (D / 8);
            float c1[8], c2[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) { c1[i] = 0.0f; c2[i] = 0.0f; }
#pragma unroll
            for (int l = 0; l < 16; ++l) {
                const uint4 raw = reinterpret_cast<const uint4*>(k + (row0 + x + 8 * l) * D)[d8];
                const __half* hv = reinterpret_cast<const __half*>(&raw);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float val = __half2float(hv[i]);
                    c1[i] = __fadd_rn(c1[i], val);
                    c2[i] = __fadd_rn(c2[i], __fmul_rn(static_cast<float>(l + 1), val));
                }
            }
            __align__(16) __half h1[8], h2[8], l1[8], l2[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                h1[i] = __float2half_rn(c1[i]);
                h2[i] = __float2half_rn(c2[i]);
                l1[i] = __float2half_rn(__fsub_rn(c1[i], __half2float(h1[i])));
                l2[i] = __float2half_rn(__fsub_rn(c2[i], __half2float(h2[i])));
            }
            reinterpret_cast<uint4*>(kc + (crow0 + x) * D)[d8] = *reinterpret_cast<const uint4*>(h1);
            reinterpret_cast<uint4*>(kc + (crow0 + 8 + x) * D)[d8] = *reinterpret_cast<const uint4*>(h2);
            reinterpret_cast<uint4*>(kc + (crow0 + 16 + x) * D)[d8] = *reinterpret_cast<const uint4*>(l1);
            reinterpret_cast<uint4*>(kc + (crow0 + 24 + x) * D)[d8] = *reinterpret_cast<const uint4*>(l2);
        }
    }
    __syncthreads();
    __half* dst = vt + (static_cast<size_t>(head) * nblk + j) * VROWS * 128;
    // transpose: thread = (dim r, 8 consecutive keys) -> one 16-byte store
    for (int t = threadIdx.x; t < D * 16; t += blockDim.x) {
        const int r = t / 16, k8 = t % 16;
        __align__(16) __half h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) h[i] = sv[sidx(k8 * 8 + i, r)];
        reinterpret_cast<uint4*>(dst + r * 128)[k8] = *reinterpret_cast<const uint4*>(h);
    }
    if (PROT) {
        // VC rows: thread = (group x, 8 consecutive keys)
        for (int t = threadIdx.x; t < 8 * 16; t += blockDim.x) {
            const int x = t / 16, k8 = t % 16;
            __align__(16) __half h1[8], h2[8], l1[8], l2[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int key = k8 * 8 + i;
                float c1 = 0.0f, c2 = 0.0f;
#pragma unroll
                for (int g = 0; g < G_O; ++g) {
                    const float val = __half2float(sv[sidx(key, x + 8 * g)]);
                    c1 = __fadd_rn(c1, val);
                    c2 = __fadd_rn(c2, __fmul_rn(static_cast<float>(g + 1), val));
                }
                h1[i] = __float2half_rn(c1);
                h2[i] = __float2half_rn(c2);
                l1[i] = __float2half_rn(__fsub_rn(c1, __half2float(h1[i])));
                l2[i] = __float2half_rn(__fsub_rn(c2, __half2float(h2[i])));
            }
            reinterpret_cast<uint4*>(dst + (D + x) * 128)[k8] = *reinterpret_cast<const uint4*>(h1);
            reinterpret_cast<uint4*>(dst + (D + 8 + x) * 128)[k8] = *reinterpret_cast<const uint4*>(h2);
            reinterpret_cast<uint4*>(dst + (D + 16 + x) * 128)[k8] = *reinterpret_cast<const uint4*>(l1);
            reinterpret_cast<uint4*>(dst + (D + 24 + x) * 128)[k8] = *reinterpret_cast<const uint4*>(l2);
        }
    }
}

}  // namespace efta_sm100
