// efta_attn_pair.cuh — CTA-pair (cta_group::2) variant of the fused EFTA forward.
//
// Why: with one 128-row query tile per SM, every SM streams the full K_j / V_j tiles
// of its head each iteration. A cluster of two CTAs on one TPC computes an M=256 tile
// with tcgen05.mma.cta_group::2: each CTA keeps its own 128 query rows (A) and holds
// only HALF of each B operand in its shared memory, so per-SM ingress halves.
//
// Shared-memory bandwidth (128 B/clk/SM, tools/mma2_bench.cu): an SS score MMA with Q
// in shared memory reads A (4 KB) + the CTA's B half (2 KB) + serves the peer's view of
// that half (2 KB) every 64 clk — the whole budget, before any TMA write lands. So Q
// lives in TMEM (staged once by the row warps) and both GEMMs are TS MMAs that read
// only B from shared memory (~64 B/clk each, leaving room for the K/V stream).
//
// TMEM columns (512): S[b] = b*NS (NS = 144 protected / 128), O = 2*NS (D + 32 / D),
// Q = O + OW (D/2 columns of fp16 pairs: the TS A operand of the score MMA).
// The score MMA carries the c1 checksum columns only (hi 8 + lo 8: N = 144, the
// exp-stage product check needs c1 alone); c2 of a score row, used only by the rare
// linear repair, is computed on the CUDA cores from Q and KC (pair_score_c2).
//
// B-operand split (CTA v owns B rows [v*N/2, (v+1)*N/2)):
//   S  = Q . [K_j ; KC1_j]^T  N = 128 (+16):  leader K rows 0..63 (0..71),
//                                            peer   K rows 64..127 (72..127 + c1_hi, c1_lo)
//   O += P . [V_j | VC_j]    N = d (+32), B = [V_j^T ; VC_j^T] K-major (keys contiguous),
//                            written by the encode prepass; each CTA loads (d+32)/2 rows.
// The leader (cluster rank 0) issues every MMA and multicasts its commits to both CTAs'
// barriers; both CTAs' TMA loads signal the leader's full barriers; both CTAs' row warps
// signal the leader's q_ready / p_ready. Row work: the split-row schedule (row_split).
#pragma once
#include "efta_attn_split.cuh"

namespace efta_sm100 {

// warps: 0 TMA producer, 1 score-MMA issuer, 2 P.V-MMA issuer, 3..10 row warps
// (two row warpgroups: warps 3-6 = half 0, 7-10 = half 1; warp w reads TMEM lanes 32*(w%4))
constexpr int kPairThreads = 352;

template <int D, bool PROT>
struct PairLayout {
    static constexpr int NSUB = D / 64;
    static constexpr int NS = PROT ? 144 : 128;           // score MMA N (scores + c1 hi/lo)
    static constexpr int HN_S = NS / 2;                    // B rows per CTA, scores
    static constexpr int VROWS = PROT ? D + 32 : D;        // rows of the V^T (+VC^T) operand
    static constexpr int HN_V = VROWS / 2;                 // B rows per CTA, P.V
    static constexpr int KS = 4, VS = 4;
    static constexpr uint32_t K_CHUNK = HN_S * 128;        // one 64-column chunk of the K half
    static constexpr uint32_t K_STAGE = NSUB * K_CHUNK;
    static constexpr uint32_t V_CHUNK = HN_V * 128;        // one 64-key chunk of the V^T half
    static constexpr uint32_t V_STAGE = 2 * V_CHUNK;
    static constexpr uint32_t OFF_K = 0;
    static constexpr uint32_t OFF_V = OFF_K + KS * K_STAGE;
    static constexpr uint32_t OFF_BAR = OFF_V + VS * V_STAGE;
    static constexpr int NBAR = 1 + 2 * KS + 2 * VS + 2 + 3 + 2 + 1;
    static constexpr uint32_t OFF_TMEM = OFF_BAR + NBAR * 8;
    static constexpr uint32_t OFF_RED = (OFF_TMEM + 16 + 15) & ~15u;
    static constexpr uint32_t RED_BYTES = 128 * 24 + 256;
    static constexpr uint32_t OFF_XCH = (OFF_RED + RED_BYTES + 15) & ~15u;  // split-row exchange
    static constexpr uint32_t SMEM_BYTES = OFF_XCH + SplitXch::BYTES + 1024;
    static_assert(SMEM_BYTES <= 232448, "shared memory budget");
    static_assert(K_CHUNK % 1024 == 0 && V_CHUNK % 1024 == 0, "swizzle atoms must stay 1 KB aligned");
    // TMEM plan
    static constexpr uint32_t COL_S0 = 0, S_STRIDE = NS;
    static constexpr uint32_t COL_O = 2 * NS;
    static constexpr uint32_t COL_Q = COL_O + (PROT ? D + 32 : D);
    static constexpr uint32_t TMEM_COLS = 512;
    static_assert(COL_Q + D / 2 <= TMEM_COLS, "TMEM budget");
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* smem_dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void mma2_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
// arrive on this barrier in both CTAs of the pair once the issued MMAs complete
__device__ __forceinline__ void commit2_both(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}
// TMA into this CTA's shared memory, completion signalled on the pair leader's barrier
__device__ __forceinline__ void tma_load_2d_pair(void* smem_dst, const void* tmap, uint64_t* bar, int c0,
                                                 int c1, uint64_t hint) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar) & 0xFEFFFFFFu), "r"(c0), "r"(c1),
        "l"(hint)
        : "memory");
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p)), "r"(bytes)
                 : "memory");
}

// Persistent pair kernel: grid = 2 x (clusters), each cluster walks the work items
// it = cluster, cluster + C, ... ; item = (head, pair of 128-row query tiles), the CTA of
// rank r owns query tile 2*(it % (n/2)) + r. Ring stages and barrier phases run on a
// global key-block counter g = t*n + j (t = the cluster's item ordinal), so the producers
// stream the next item's K/V while the row warps finish the current one, and the next
// item's first score MMAs overlap the current item's epilogue.
// tm_ka: K rows [0, HN_S) of each block (leader; [64r, 64r+64) unprotected), tm_kb: K rows
// 72..127 (peer, protected), tm_kc: KC rows in 8-row boxes (protected), tm_vt: [V^T ; VC^T]
// rows of each block, box rows HN_V.
template <int D, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1)
efta_attn_pair_kernel(const __grid_constant__ CUtensorMap tm_ka, const __grid_constant__ CUtensorMap tm_kb,
                      const __grid_constant__ CUtensorMap tm_kc, const __grid_constant__ CUtensorMap tm_vt,
                      const __grid_constant__ AttnParams p) {
    constexpr bool PROT = MODE != EFTA_MODE_NONE;
    using L = PairLayout<D, PROT>;
    constexpr int KS = L::KS, VS = L::VS, NSUB = L::NSUB;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
    uint64_t* q_ready = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = k_full + KS;
    uint64_t* v_full = k_empty + KS;
    uint64_t* v_empty = v_full + VS;
    uint64_t* s_full = v_empty + VS;
    // p_ready[g&1]: row warps of different slices / CTAs are not in lockstep, so a fast
    // warp may arrive for block g+1 before block g's phase completed; alternating barriers
    // keep the counts apart (a warp cannot reach g+2 before PV(g), hence p_ready[g&1], ran)
    uint64_t* p_ready = s_full + 2;
    uint64_t* o_done = p_ready + 2;
    uint64_t* pv_done = o_done + 1;  // [2]: PV(g) done, per S buffer g&1
    uint64_t* o_free = pv_done + 2;  // O read out of TMEM by both CTAs' row warps
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

    const int warp = warp_id(), lane = lane_id();
    const uint32_t rank = cluster_rank();
    const int n = p.nblk;
    const int pairs_per_head = n / 2;
    const int total = pairs_per_head * p.n_heads_flat;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    auto item_head = [&](int it) { return it / pairs_per_head; };
    auto item_qt = [&](int it) { return 2 * (it % pairs_per_head) + static_cast<int>(rank); };

    if (warp == 0 && lane == 0) {
        mbar_init(q_ready, 16);  // 8 row warps x 2 CTAs
        for (int s = 0; s < KS; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
        for (int s = 0; s < VS; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
        mbar_init(&s_full[0], 1);
        mbar_init(&s_full[1], 1);
        mbar_init(&p_ready[0], 16);  // 8 row warps x 2 CTAs
        mbar_init(&p_ready[1], 16);
        mbar_init(o_done, 1);
        mbar_init(&pv_done[0], 1);
        mbar_init(&pv_done[1], 1);
        mbar_init(o_free, 16);
        fence_barrier_init();
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
    const uint32_t k_smem = smem_u32(smem + L::OFF_K);
    const uint32_t v_smem = smem_u32(smem + L::OFF_V);

    if (warp == 0) {
        // -------------------------------------------------------- K (+KC1) / V^T (+VC^T) producer
        // one thread streams both rings in block order (K(g) is consumed before V(g))
        if (lane == 0) {
            for (int t = 0, it = cid; it < total; ++t, it += ncl) {
                const int head = item_head(it);
                const int seq_row0 = head * p.seq_len;
                for (int j = 0; j < n; ++j) {
                    const int g = t * n + j;
                    const int s = g % KS;
                    mbar_wait(&k_empty[s], ((g / KS) & 1) ^ 1);
                    if (j == (n > 8 ? n - 8 : 0) && it + ncl < total) {  // next item's Q rows -> L2
                        const int nit = it + ncl;
                        prefetch_l2_bulk(p.q + (static_cast<size_t>(item_head(nit)) * p.seq_len +
                                                static_cast<size_t>(item_qt(nit)) * kBlock) * D,
                                         kBlock * D * 2);
                    }
                    uint8_t* dst = smem + L::OFF_K + s * L::K_STAGE;
#ifdef EFTA_NO_TMA  // experiment build: MMAs on stale tiles, no K/V traffic
                    if (rank == 0) mbar_arrive(&k_full[s]);
#else
                    if (rank == 0) mbar_arrive_expect_tx(&k_full[s], 2 * L::K_STAGE);
                    const int krow = seq_row0 + j * kBlock;
#pragma unroll
                    for (int sub = 0; sub < NSUB; ++sub) {
                        uint8_t* c = dst + sub * L::K_CHUNK;
                        if (!PROT) {
                            tma_load_2d_pair(c, &tm_ka, &k_full[s], sub * 64, krow + 64 * rank, kEvictLast);
                        } else if (rank == 0) {
                            tma_load_2d_pair(c, &tm_ka, &k_full[s], sub * 64, krow, kEvictLast);
                        } else {
                            const int crow = (head * n + j) * 32;
                            tma_load_2d_pair(c, &tm_kb, &k_full[s], sub * 64, krow + 72, kEvictLast);
                            tma_load_2d_pair(c + 56 * 128, &tm_kc, &k_full[s], sub * 64, crow, kEvictLast);      // c1_hi
                            tma_load_2d_pair(c + 64 * 128, &tm_kc, &k_full[s], sub * 64, crow + 16, kEvictLast); // c1_lo
                        }
                    }
#endif
                    const int sv = g % VS;
                    mbar_wait(&v_empty[sv], ((g / VS) & 1) ^ 1);
                    uint8_t* vdst = smem + L::OFF_V + sv * L::V_STAGE;
#ifdef EFTA_NO_TMA
                    if (rank == 0) mbar_arrive(&v_full[sv]);
#else
                    if (rank == 0) mbar_arrive_expect_tx(&v_full[sv], 2 * L::V_STAGE);
                    const int vrow = (head * n + j) * L::VROWS + L::HN_V * rank;
#pragma unroll
                    for (int c = 0; c < 2; ++c)
                        tma_load_2d_pair(vdst + c * L::V_CHUNK, &tm_vt, &v_full[sv], c * 64, vrow, kEvictLast);
#endif
                }
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- score MMA issuer (pair leader)
        // tcgen05.mma issue from one thread is effectively unbuffered (tools/mma2_bench.cu:
        // every clock the issuing thread spends waiting is a tensor-pipe bubble), so the two
        // GEMMs have separate issuer threads: while one waits on a barrier the other's MMAs
        // keep the pipe busy.
        if (lane == 0 && rank == 0) {
            constexpr uint32_t ID_S = idesc_f16_f32(256, L::NS, 0, 0);
            const uint32_t a_q = tmem + L::COL_Q;
            for (int t = 0, it = cid; it < total; ++t, it += ncl) {
                for (int j = 0; j < n; ++j) {
                    const int g = t * n + j;
                    const int s = g % KS;
                    if (j == 0) {  // this item's Q staged in TMEM by both CTAs
                        mbar_wait(q_ready, t & 1);
                        tc_fence_after();
                    }
                    if (g >= 2) {  // S[g&1] holds P(g-2) until PV(g-2) has read it
                        mbar_wait(&pv_done[g & 1], ((g >> 1) + 1) & 1);
                        tc_fence_after();
                    }
                    mbar_wait(&k_full[s], (g / KS) & 1);
                    EFTA_TS(9, j);
                    tc_fence_after();
                    const uint32_t kb = k_smem + s * L::K_STAGE;
                    const uint32_t d_s = tmem + L::COL_S0 + (g & 1) * L::S_STRIDE;
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t offk = (kk >> 2) * L::K_CHUNK + (kk & 3) * 32;
                        mma2_ts(d_s, a_q + kk * 8, smem_desc_sw128(kb + offk, 16, 1024), ID_S, kk > 0);
                    }
                    commit2_both(&k_empty[s]);
                    commit2_both(&s_full[g & 1]);
                    EFTA_TS(11, j);
                }
            }
        }
        __syncwarp();
    } else if (warp == 2) {
        // -------------------------------------------------------- P.V MMA issuer (pair leader)
        if (lane == 0 && rank == 0) {
            constexpr uint32_t ID_PV = idesc_f16_f32(256, L::VROWS, 0, 0);
            for (int t = 0, it = cid; it < total; ++t, it += ncl) {
                for (int j = 0; j < n; ++j) {
                    const int g = t * n + j;
                    EFTA_TS(10, j);
                    mbar_wait(&p_ready[g & 1], (g >> 1) & 1);
                    EFTA_TS(12, j);
                    tc_fence_after();
                    const int s = g % VS;
                    mbar_wait(&v_full[s], (g / VS) & 1);
                    if (j == 0 && t > 0) mbar_wait(o_free, (t - 1) & 1);  // previous item's O read out
                    EFTA_TS(14, j);
                    tc_fence_after();
                    const uint32_t vb = v_smem + s * L::V_STAGE;
                    const uint32_t a_p = tmem + L::COL_S0 + (g & 1) * L::S_STRIDE;
#pragma unroll
                    for (int kk = 0; kk < kBlock / 16; ++kk) {
                        const uint32_t offv = (kk >> 2) * L::V_CHUNK + (kk & 3) * 32;
                        mma2_ts(tmem + L::COL_O, a_p + kk * 8, smem_desc_sw128(vb + offv, 16, 1024), ID_PV,
                                (j > 0 || kk > 0) ? 1u : 0u);
                    }
                    commit2_both(&v_empty[s]);
                    commit2_both(&pv_done[g & 1]);
                    commit2_both(o_done);
                    EFTA_TS(13, j);
                }
            }
        }
        __syncwarp();
    } else if (warp >= kRowWarp0) {
        RowScratch rs;
        rs.slots = reinterpret_cast<RowSlot*>(smem + L::OFF_RED);
        rs.ints = reinterpret_cast<int*>(smem + L::OFF_RED + 128 * sizeof(RowSlot));
        rs.dbl = reinterpret_cast<double*>(smem + L::OFF_RED + 128 * sizeof(RowSlot) + 16 * sizeof(int));
        if (cid < total) {
            stage_q_rows<D>(p, tmem + L::COL_Q, warp, lane, item_head(cid) * p.seq_len + item_qt(cid) * kBlock);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(q_ready, 0);
        }
        for (int t = 0, it = cid; it < total; ++t, it += ncl) {
            const int head = item_head(it), qt = item_qt(it);
            const int nit = it + ncl;
            const int next_q_row = nit < total ? item_head(nit) * p.seq_len + item_qt(nit) * kBlock : -1;
            row_split<D, MODE, true, L>(p, s_full, p_ready, o_done, o_free, tmem, warp, lane, head, qt, n,
                                        head * p.seq_len, t * n, rs, reinterpret_cast<float*>(smem + L::OFF_XCH),
                                        next_q_row, q_ready);
        }
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
template <int D, bool PROT>
__global__ void __launch_bounds__(256) efta_encode_pair_kernel(const __half* __restrict__ k,
                                                               const __half* __restrict__ v,
                                                               __half* __restrict__ kc, __half* __restrict__ vt,
                                                               int seq_len, int nblk) {
    constexpr int VROWS = PROT ? D + 32 : D;
    constexpr int G_O = D / 8;
    __shared__ __half sv[128 * (D + 8)];
    const int j = blockIdx.x, head = blockIdx.y;
    const size_t row0 = static_cast<size_t>(head) * seq_len + static_cast<size_t>(j) * 128;
    for (int idx = threadIdx.x; idx < 128 * D / 8; idx += blockDim.x) {
        const int r = idx / (D / 8), c8 = idx % (D / 8);
        *reinterpret_cast<uint4*>(&sv[r * (D + 8) + c8 * 8]) = reinterpret_cast<const uint4*>(v + (row0 + r) * D)[c8];
    }
    if (PROT) {
        const size_t crow0 = (static_cast<size_t>(head) * nblk + j) * 32;
        for (int t = threadIdx.x; t < 8 * D; t += blockDim.x) {
            const int x = t / D, dim = t % D;
            float c1 = 0.0f, c2 = 0.0f;
#pragma unroll
            for (int l = 0; l < 16; ++l) {
                const float val = __half2float(k[(row0 + x + 8 * l) * D + dim]);
                c1 = __fadd_rn(c1, val);
                c2 = __fadd_rn(c2, __fmul_rn(static_cast<float>(l + 1), val));
            }
            const __half h1 = __float2half_rn(c1), h2 = __float2half_rn(c2);
            kc[(crow0 + x) * D + dim] = h1;
            kc[(crow0 + 8 + x) * D + dim] = h2;
            kc[(crow0 + 16 + x) * D + dim] = __float2half_rn(__fsub_rn(c1, __half2float(h1)));
            kc[(crow0 + 24 + x) * D + dim] = __float2half_rn(__fsub_rn(c2, __half2float(h2)));
        }
    }
    __syncthreads();
    __half* dst = vt + (static_cast<size_t>(head) * nblk + j) * VROWS * 128;
    for (int t = threadIdx.x; t < D * 128; t += blockDim.x) {  // transpose: coalesced over keys
        const int r = t / 128, key = t % 128;
        dst[r * 128 + key] = sv[key * (D + 8) + r];
    }
    if (PROT) {
        for (int t = threadIdx.x; t < 8 * 128; t += blockDim.x) {
            const int x = t / 128, key = t % 128;
            float c1 = 0.0f, c2 = 0.0f;
#pragma unroll
            for (int g = 0; g < G_O; ++g) {
                const float val = __half2float(sv[key * (D + 8) + x + 8 * g]);
                c1 = __fadd_rn(c1, val);
                c2 = __fadd_rn(c2, __fmul_rn(static_cast<float>(g + 1), val));
            }
            const __half h1 = __float2half_rn(c1), h2 = __float2half_rn(c2);
            dst[(D + x) * 128 + key] = h1;
            dst[(D + 8 + x) * 128 + key] = h2;
            dst[(D + 16 + x) * 128 + key] = __float2half_rn(__fsub_rn(c1, __half2float(h1)));
            dst[(D + 24 + x) * 128 + key] = __float2half_rn(__fsub_rn(c2, __half2float(h2)));
        }
    }
}

}  // namespace efta_sm100
