// efta_attn_pair.cuh — CTA-pair (cta_group::2) variant of the fused EFTA forward.
//
// Why: with one 128-row query tile per SM, every SM streams the full K_j / V_j tiles
// of its head from L2 each iteration (64 KB, 88 KB protected, at d=128); the measured
// iteration time sits at the chip's L2->SM delivery limit while the tensor cores idle
// (tools/mma_bench.cu: every MMA flavour runs at its floor in isolation). A cluster of
// two CTAs on one TPC computes an M=256 tile with tcgen05.mma.cta_group::2: each CTA
// keeps its own 128 query rows (A) and holds only HALF of each B operand in its shared
// memory, so per-SM ingress halves (32 KB / 40 KB per iteration).
//
// B-operand split (CUTLASS 2x1SM traits: CTA v owns B rows [v*N/2, (v+1)*N/2)):
//   S  = Q . [K_j ; KC_j]^T  N = 128 (+32):  leader K rows 0..63 (0..79),
//                                            peer   K rows 64..127 (80..127 + KC 0..31)
//   O += P . [V_j | VC_j]    N = d (+32), B = [V_j^T ; VC_j^T] K-major (keys contiguous),
//                            written by the encode prepass; each CTA loads (d+32)/2 rows.
// The leader (cluster rank 0) issues every MMA and multicasts its commits to both CTAs'
// barriers; both CTAs' TMA loads signal the leader's full barriers; both row warpgroups
// signal the leader's p_ready. The row warpgroup code is the single-CTA one (row_wg).
#pragma once
#include "efta_attn_kernel.cuh"

namespace efta_sm100 {

template <int D, bool PROT>
struct PairLayout {
    static constexpr int NSUB = D / 64;
    static constexpr int HN_S = (PROT ? 160 : 128) / 2;  // B rows per CTA, scores
    static constexpr int VROWS = PROT ? D + 32 : D;      // rows of the V^T (+VC^T) operand
    static constexpr int HN_V = VROWS / 2;               // B rows per CTA, P.V
    static constexpr int KS = 4, VS = 4;
    static constexpr uint32_t Q_BYTES = NSUB * 16384;
    static constexpr uint32_t K_CHUNK = HN_S * 128;      // one 64-column chunk of the K half
    static constexpr uint32_t K_STAGE = NSUB * K_CHUNK;
    static constexpr uint32_t V_CHUNK = HN_V * 128;      // one 64-key chunk of the V^T half
    static constexpr uint32_t V_STAGE = 2 * V_CHUNK;
    static constexpr uint32_t OFF_Q = 0;
    static constexpr uint32_t OFF_K = OFF_Q + Q_BYTES;
    static constexpr uint32_t OFF_V = OFF_K + KS * K_STAGE;
    static constexpr uint32_t OFF_BAR = OFF_V + VS * V_STAGE;
    static constexpr int NBAR = 1 + 2 * KS + 2 * VS + 2 + 2;
    static constexpr uint32_t OFF_TMEM = OFF_BAR + NBAR * 8;
    static constexpr uint32_t OFF_RED = (OFF_TMEM + 16 + 15) & ~15u;
    static constexpr uint32_t RED_BYTES = 128 * 24 + 256;
    static constexpr uint32_t SMEM_BYTES = OFF_RED + RED_BYTES + 1024;
    static_assert(K_CHUNK % 1024 == 0 && V_CHUNK % 1024 == 0, "swizzle atoms must stay 1 KB aligned");
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
__device__ __forceinline__ void mma2_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
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

// tm_ka: K rows [0, HN_S) (or [64r, 64r+64) unprotected), tm_kb: K rows 80..127 (protected),
// tm_kc: KC (protected), tm_vt: [V^T ; VC^T] rows of each block, box rows HN_V.
template <int D, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
efta_attn_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_ka,
                      const __grid_constant__ CUtensorMap tm_kb, const __grid_constant__ CUtensorMap tm_kc,
                      const __grid_constant__ CUtensorMap tm_vt, const AttnParams p) {
    constexpr bool PROT = MODE != EFTA_MODE_NONE;
    using L = PairLayout<D, PROT>;
    using TL = AttnLayout<D>;  // TMEM column plan (shared with the single-CTA kernel)
    constexpr int KS = L::KS, VS = L::VS, NSUB = L::NSUB;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = k_full + KS;
    uint64_t* v_full = k_empty + KS;
    uint64_t* v_empty = v_full + VS;
    uint64_t* s_full = v_empty + VS;
    uint64_t* p_ready = s_full + 2;
    uint64_t* o_done = p_ready + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

    const int warp = warp_id(), lane = lane_id();
    const uint32_t rank = cluster_rank();
    const int qt = blockIdx.x, head = blockIdx.y, n = p.nblk;
    const int seq_row0 = head * p.seq_len;

    if (warp == 0 && lane == 0) {
        mbar_init(q_full, 1);
        for (int s = 0; s < KS; ++s) { mbar_init(&k_full[s], 1); mbar_init(&k_empty[s], 1); }
        for (int s = 0; s < VS; ++s) { mbar_init(&v_full[s], 1); mbar_init(&v_empty[s], 1); }
        mbar_init(&s_full[0], 1);
        mbar_init(&s_full[1], 1);
        mbar_init(p_ready, 8);  // 4 row warps x 2 CTAs
        mbar_init(o_done, 1);
        fence_barrier_init();
        tma_prefetch_desc(&tm_q);
        tma_prefetch_desc(&tm_ka);
        tma_prefetch_desc(&tm_vt);
        if (PROT) { tma_prefetch_desc(&tm_kb); tma_prefetch_desc(&tm_kc); }
    }
    if (warp == 1) tmem_alloc2(tmem_slot, TL::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / TMA
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t q_smem = smem_u32(smem + L::OFF_Q);
    const uint32_t k_smem = smem_u32(smem + L::OFF_K);
    const uint32_t v_smem = smem_u32(smem + L::OFF_V);

    if (warp == 0) {
        // -------------------------------------------------------- K (+KC) half producer
        if (lane == 0) {
            for (int j = 0; j < n; ++j) {
                const int s = j % KS;
                mbar_wait(&k_empty[s], ((j / KS) & 1) ^ 1);
                uint8_t* dst = smem + L::OFF_K + s * L::K_STAGE;
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
                        tma_load_2d_pair(c, &tm_kb, &k_full[s], sub * 64, krow + 80, kEvictLast);
                        tma_load_2d_pair(c + 48 * 128, &tm_kc, &k_full[s], sub * 64, (head * n + j) * 32,
                                         kEvictLast);
                    }
                }
            }
        }
    } else if (warp == 3) {
        // -------------------------------------------------------- Q, V^T (+VC^T) half producer
        if (lane == 0) {
            if (rank == 0) mbar_arrive_expect_tx(q_full, 2 * L::Q_BYTES);
#pragma unroll
            for (int sub = 0; sub < NSUB; ++sub)
                tma_load_2d_pair(smem + L::OFF_Q + sub * 16384, &tm_q, q_full, sub * 64, seq_row0 + qt * kBlock,
                                 kEvictFirst);
            for (int j = 0; j < n; ++j) {
                const int s = j % VS;
                mbar_wait(&v_empty[s], ((j / VS) & 1) ^ 1);
                uint8_t* dst = smem + L::OFF_V + s * L::V_STAGE;
                if (rank == 0) mbar_arrive_expect_tx(&v_full[s], 2 * L::V_STAGE);
                const int vrow = (head * n + j) * L::VROWS + L::HN_V * rank;
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    tma_load_2d_pair(dst + c * L::V_CHUNK, &tm_vt, &v_full[s], c * 64, vrow, kEvictLast);
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------- MMA issuer (pair leader only)
        if (lane == 0 && rank == 0) {
            constexpr uint32_t ID_S = idesc_f16_f32(256, PROT ? 160 : 128, 0, 0);
            constexpr uint32_t ID_PV = idesc_f16_f32(256, L::VROWS, 0, 0);
            mbar_wait(q_full, 0);
            tc_fence_after();
            auto issue_s = [&](int j) {
                const int s = j % KS;
                mbar_wait(&k_full[s], (j / KS) & 1);
                tc_fence_after();
                const uint32_t kb = k_smem + s * L::K_STAGE;
                const uint32_t d_s = tmem + TL::COL_S0 + (j & 1) * TL::S_STRIDE;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t offq = (kk >> 2) * 16384 + (kk & 3) * 32;
                    const uint32_t offk = (kk >> 2) * L::K_CHUNK + (kk & 3) * 32;
                    mma2_ss(d_s, smem_desc_sw128(q_smem + offq, 16, 1024), smem_desc_sw128(kb + offk, 16, 1024),
                            ID_S, kk > 0);
                }
                commit2_both(&k_empty[s]);
                commit2_both(&s_full[j & 1]);
            };
            issue_s(0);
            for (int j = 0; j < n; ++j) {
                EFTA_TS(10, j);
                if (j + 1 < n) issue_s(j + 1);
                EFTA_TS(11, j);
                mbar_wait(p_ready, j & 1);
                EFTA_TS(12, j);
                tc_fence_after();
                const int s = j % VS;
                mbar_wait(&v_full[s], (j / VS) & 1);
                EFTA_TS(14, j);
                tc_fence_after();
                const uint32_t vb = v_smem + s * L::V_STAGE;
                const uint32_t a_p = tmem + TL::COL_S0 + (j & 1) * TL::S_STRIDE;
#pragma unroll
                for (int kk = 0; kk < kBlock / 16; ++kk) {
                    const uint32_t offv = (kk >> 2) * L::V_CHUNK + (kk & 3) * 32;
                    mma2_ts(tmem + TL::COL_O, a_p + kk * 8, smem_desc_sw128(vb + offv, 16, 1024), ID_PV,
                            (j > 0 || kk > 0) ? 1u : 0u);
                }
                commit2_both(&v_empty[s]);
                commit2_both(o_done);
                EFTA_TS(13, j);
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        row_wg<D, MODE, false, true>(p, smem + L::OFF_RED, s_full, p_ready, o_done, tmem, warp, lane, head, qt,
                                     n, seq_row0);
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer may still be reading our shared memory / TMEM via the MMAs
    tc_fence_after();
    if (warp == 1) tmem_dealloc2(tmem, TL::TMEM_COLS);
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
